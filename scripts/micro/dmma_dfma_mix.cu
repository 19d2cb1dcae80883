// Do DMMA (FP64 tensor) and DFMA (FP64 vector) share hardware on sm_100a?
// Each CTA has 8 warps; the first `nd` warps issue DMMA.8x8x4 chains, the others DFMA
// chains. Prints achieved TFLOP/s of each pipe for nd = 8 (DMMA only), 0 (DFMA only)
// and mixes.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 dmma_dfma_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void mix(int iters, int nd, double* out) {
  const int warp = threadIdx.x >> 5;
  double acc[16];
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  const double a = 1.0000001, b = 0.9999999;
  if (warp < nd) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(acc[2 * i], acc[2 * i + 1], a, b);
    }
  } else {
    // 16 independent DFMA chains; 4 rounds per iteration -> same instruction pressure
    for (int it = 0; it < iters * 8; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
    }
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000, blocks = sms * 4, threads = 256;
  mix<<<blocks, threads>>>(100, 4, out);
  cudaDeviceSynchronize();
  for (int nd : {8, 0, 4, 6, 2}) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mix<<<blocks, threads>>>(iters, nd, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double dmma_flop = (double)blocks * nd * iters * 8 * 512.0;  // 8x8x4x2 per DMMA
    const double dfma_flop = (double)blocks * (8 - nd) * 32 * iters * 8 * 16 * 2.0;
    printf("dmma warps %d/8: %.3f ms  DMMA %.2f TF/s  DFMA %.2f TF/s  sum %.2f\n", nd, ms,
           dmma_flop / ms / 1e9, dfma_flop / ms / 1e9, (dmma_flop + dfma_flop) / ms / 1e9);
  }
  return 0;
}
