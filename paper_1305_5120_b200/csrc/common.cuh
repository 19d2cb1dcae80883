// Shared device helpers for the ChFSI B200 kernels (sm_100a).
//
// Everything on the hot path is complex128 stored as interleaved double2,
// column-major, exactly the numpy F-order layout the reference uses
// (reference pkg/src/chfsi/linalg.py:89-121). FP64 tensor-core math on
// sm_100a is the warp-level DMMA path (mma.sync ... f64); tcgen05 has no
// f64 kind (ptxas rejects .kind::f64), see DESIGN.md.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace chfsi {

enum Op : int { OP_N = 0, OP_C = 1 };  // OP_C = conjugate transpose
// Triangular GEMM operands (zgemm `tri`): the zero blocks of the K range are skipped.
enum Tri : int {
  TRI_NONE = 0,
  TRI_A_LOWER = 1,  // A (op N) lower triangular: row tile m0 needs k < m0 + BM
  TRI_B_UPPER = 2,  // op(B) = L^H, L lower: column tile n0 needs k < n0 + BN
  TRI_B_LOWER = 4,  // B (op N) lower triangular: column tile n0 needs k >= n0
  TRI_A_UPPER = 8,  // op(A) = L^H, L lower: row tile m0 needs k >= m0
  TRI_C_LOWER = 16, // C Hermitian (M == N): only tiles touching the lower triangle are
                    // computed; the caller mirrors (mirror_lower) before using the upper
};

// D(8x8) += A(8x4, row) * B(4x8, col), all f64. One SASS DMMA.8x8x4.
// Fragment ownership (PTX ISA, m8n8k4 .f64):
//   a: row = lane>>2, col = lane&3      b: row = lane&3, col = lane>>2
//   c/d: row = lane>>2, col = 2*(lane&3) + {0,1}
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int sz = pred ? 16 : 0;  // src-size 0 => zero fill, no global read
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 conj2(double2 a) { return make_double2(a.x, -a.y); }

// Deterministic block reduction of one double (fixed tree, no atomics).
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
  #pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = (l < NT / 32) ? red[l] : 0.0;
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (l == 0) red[0] = v;
  }
  __syncthreads();
  const double r = red[0];
  __syncthreads();
  return r;
}

}  // namespace chfsi
