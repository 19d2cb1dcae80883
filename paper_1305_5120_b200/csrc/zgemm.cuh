// Complex128 GEMM on the FP64 tensor pipe (DMMA), sm_100a.
//
//   C = alpha * op(A) * op(B) + beta * C            (EPI_STORE)
//   C = alpha * A * Y1 + beta * Y1 + gamma * Y0     (EPI_FILTER, B == Y1)
//   ws[z] = op(A) * op(B) over K-chunk z            (EPI_PARTIAL, split-K)
//
// This is the contraction behind every n x n x k product of the reference
// (linalg.py:198-251 `gemm`), and with EPI_FILTER one Chebyshev degree step
// of core.py:263-284 `_filter_raw` with the scale/shift/axpy fused into the
// epilogue (reference: gemm(scale, h, y1, beta=-c*scale, c=y1) followed by
// y2 -= sigma*sigma_new*y0).
//
// Complex arithmetic is four real DMMAs per 8x8x4 block:
//   Cr += Ar*Br + (-Ai)*Bi,   Ci += Ar*Bi + Ai*Br.
// Operands are interleaved double2 in global and shared memory, so one
// LDS.128 brings both the real and the imaginary fragment element.
//
// Pipeline: STAGES-deep cp.async (LDGSTS, 16 B = one complex per op)
// global->shared ring; shared strides are padded so every fragment LDS.128
// quarter-warp touches 8 distinct 16-byte bank groups.
#pragma once

#include "common.cuh"

namespace chfsi {

enum Epi : int { EPI_STORE = 0, EPI_FILTER = 1, EPI_PARTIAL = 2 };

struct GemmParams {
  int M, N, K;
  const double2* A; long long lda;
  const double2* B; long long ldb;
  double2* C; long long ldc;
  double2 alpha, beta;
  // EPI_FILTER: Y0 (may alias C) and its real coefficient gamma; Y1e is the beta
  // operand (rows aligned with C): B itself for a full step, B + r0 for a row panel
  const double2* Y0; long long ld0; double gamma;
  const double2* Y1e; long long ld1e;
  // EPI_PARTIAL: K range per blockIdx.z and the [z][N][M] workspace
  int k_chunk;
  double2* ws;
  // grouped raster: blockIdx.x enumerates tiles so that `group` consecutive row tiles
  // share each column tile inside one wave (Y strips are reused from L2)
  int tiles_m, tiles_n, group;
  // EPI_FILTER: when non-null, {alpha, beta, gamma} are read from device memory
  // (CUDA-graph replays of the filter reuse one captured launch sequence while the
  // Chebyshev coefficients change every outer iteration)
  const double* coef;
  // Tri flags (common.cuh): K ranges of triangular operands; the longest tiles go first.
  // tri_off: global index of row/column 0 of C inside the triangular factor (a column
  // shard of L^-1 A L^-H multiplies by rows [tri_off, tri_off + N) of L^-1).
  int tri;
  int tri_off;
  // 3M operand-sum planes: As = Re A + Im A (M x K, M % 8 == 0) in the grouped layout
  // As[(i / 8) * 8 K + j * 8 + ((i % 8) ^ (2 * ((j / 2) % 2)))] (ldas unused); Bs = Re B + Im B (K x N,
  // column-major, ld in doubles); Cs (optional, EPI_FILTER / EPI_STORE of the TMA kernels
  // and the split-K reduce) receives Re C + Im C of the result, column-major: the next
  // step's Bs
  // TMA kernels: A arrives as one 3-D box per stage (M % 8 == 0), set by the launcher
  int a3d;
  // 3M TMA kernels: a last live 8-column block holding <= 4 columns is multiplied in the
  // packed four-product form (zgemm_tma.cuh); set by the launcher (CHFSI_PACK_TAIL=0: off)
  int pack;
  // TMA kernels with one warp column (WN == BN): the first n_wide column tiles are BN wide,
  // the rest BN - 8 (their last 8-column block is skipped), so 32- and 24-column tiles
  // cover a block of 8 m columns exactly in one launch; 0: every tile BN wide
  int n_wide;
  const double* As; long long ldas;
  const double* Bs; long long ldbs;
  double* Cs; long long ldcs;
};

__device__ __forceinline__ void tri_krange(const GemmParams& p, int m0, int n0, int bm, int bn,
                                           int& kbeg, int& kend) {
  if (p.tri & TRI_A_LOWER) kend = min(kend, p.tri_off + m0 + bm);
  if (p.tri & TRI_B_UPPER) kend = min(kend, p.tri_off + n0 + bn);
  if (p.tri & TRI_B_LOWER) kbeg = max(kbeg, p.tri_off + n0);
  if (p.tri & TRI_A_UPPER) kbeg = max(kbeg, p.tri_off + m0);
}

__device__ __forceinline__ void filter_coef(const GemmParams& p, double& a, double& b, double& g) {
  if (p.coef != nullptr) {
    a = p.coef[0];
    b = p.coef[1];
    g = p.coef[2];
  } else {
    a = p.alpha.x;
    b = p.beta.x;
    g = p.gamma;
  }
}

// linear tile id -> (row tile, column tile), grouped raster
__device__ __forceinline__ void tile_coords(const GemmParams& p, int b, int& mi, int& ni) {
  const int per_group = p.group * p.tiles_n;
  const int g = b / per_group;
  const int first = g * p.group;
  const int gsize = min(p.tiles_m - first, p.group);
  const int r = b - g * per_group;
  mi = first + r % gsize;
  ni = r / gsize;
  // triangular operands: the tiles with the longest K range first (fewer idle SMs in
  // the last wave)
  if (p.tri & TRI_A_LOWER) mi = p.tiles_m - 1 - mi;
  if (p.tri & TRI_B_UPPER) ni = p.tiles_n - 1 - ni;
}
// (TRI_A_UPPER / TRI_B_LOWER: the low tiles are the long ones, already first)

template <int BM, int BK, int OPA>
struct ATile {
  static constexpr int LD = (OPA == OP_N) ? (BM + 2) : (BK + 4);
  static constexpr int ELEMS = (OPA == OP_N) ? BK * LD : BM * LD;
};
template <int BN, int BK, int OPB>
struct BTile {
  static constexpr int LD = (OPB == OP_N) ? (BK + 4) : (BN + 2);
  static constexpr int ELEMS = (OPB == OP_N) ? BN * LD : BK * LD;
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int OPA, int OPB>
constexpr int zgemm_smem_bytes() {
  return STAGES * (ATile<BM, BK, OPA>::ELEMS + BTile<BN, BK, OPB>::ELEMS) * 16;
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int OPA, int OPB, int EPI>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32)
zgemm_dmma_kernel(const GemmParams p) {
  constexpr int NWM = BM / WM;
  constexpr int NT = NWM * (BN / WN) * 32;
  constexpr int FM = WM / 8, FN = WN / 8;
  constexpr int LDA = ATile<BM, BK, OPA>::LD, SA = ATile<BM, BK, OPA>::ELEMS;
  constexpr int LDB = BTile<BN, BK, OPB>::LD, SB = BTile<BN, BK, OPB>::ELEMS;
  static_assert(BK % 4 == 0 && WM % 8 == 0 && WN % 8 == 0, "tile shape");

  extern __shared__ __align__(16) double2 smem[];
  double2* sA = smem;
  double2* sB = smem + STAGES * SA;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % NWM, wn = warp / NWM;
  int mi, ni;
  tile_coords(p, blockIdx.x, mi, ni);
  const int m0 = mi * BM, n0 = ni * BN;
  if ((p.tri & TRI_C_LOWER) && m0 + BM <= n0) return;  // strictly upper tile (CTA-uniform)
  int kbeg = 0, kend = p.K;
  if (EPI == EPI_PARTIAL) {
    kbeg = blockIdx.z * p.k_chunk;
    kend = min(p.K, kbeg + p.k_chunk);
  }
  tri_krange(p, m0, n0, BM, BN, kbeg, kend);
  const int KT = (kend > kbeg) ? (kend - kbeg + BK - 1) / BK : 0;

  auto load_tile = [&](int kt, int stage) {
    const int k0 = kbeg + kt * BK;
    double2* a = sA + stage * SA;
    double2* b = sB + stage * SB;
    #pragma unroll
    for (int i = tid; i < BM * BK; i += NT) {
      int m, kk;
      if (OPA == OP_N) { m = i % BM; kk = i / BM; } else { kk = i % BK; m = i / BK; }
      const int gm = m0 + m, gk = k0 + kk;
      const bool ok = (gm < p.M) && (gk < kend);
      const double2* src = p.A;
      if (ok) src = (OPA == OP_N) ? p.A + gm + (long long)gk * p.lda : p.A + gk + (long long)gm * p.lda;
      double2* dst = (OPA == OP_N) ? a + kk * LDA + m : a + m * LDA + kk;
      cp_async16(dst, src, ok);
    }
    #pragma unroll
    for (int i = tid; i < BK * BN; i += NT) {
      int kk, nn;
      if (OPB == OP_N) { kk = i % BK; nn = i / BK; } else { nn = i % BN; kk = i / BN; }
      const int gk = k0 + kk, gn = n0 + nn;
      const bool ok = (gn < p.N) && (gk < kend);
      const double2* src = p.B;
      if (ok) src = (OPB == OP_N) ? p.B + gk + (long long)gn * p.ldb : p.B + gn + (long long)gk * p.ldb;
      double2* dst = (OPB == OP_N) ? b + nn * LDB + kk : b + kk * LDB + nn;
      cp_async16(dst, src, ok);
    }
  };

  double cr[FM][FN][2], ci[FM][FN][2];
  #pragma unroll
  for (int i = 0; i < FM; ++i)
    #pragma unroll
    for (int j = 0; j < FN; ++j) {
      cr[i][j][0] = cr[i][j][1] = 0.0;
      ci[i][j][0] = ci[i][j][1] = 0.0;
    }

  #pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_tile(s, s);
    cp_async_commit();
  }

  const int fr = lane >> 2, fc = lane & 3;
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < KT) load_tile(nk, nk % STAGES);
      cp_async_commit();
    }
    const double2* a = sA + (kt % STAGES) * SA;
    const double2* b = sB + (kt % STAGES) * SB;
    #pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      double2 fa[FM], fb[FN];
      #pragma unroll
      for (int i = 0; i < FM; ++i) {
        const int m = wm * WM + i * 8 + fr, kk = ks * 4 + fc;
        fa[i] = (OPA == OP_N) ? a[kk * LDA + m] : a[m * LDA + kk];
      }
      #pragma unroll
      for (int j = 0; j < FN; ++j) {
        const int kk = ks * 4 + fc, nn = wn * WN + j * 8 + fr;
        fb[j] = (OPB == OP_N) ? b[nn * LDB + kk] : b[kk * LDB + nn];
      }
      #pragma unroll
      for (int i = 0; i < FM; ++i) {
        const double ar = fa[i].x;
        const double ai = (OPA == OP_C) ? -fa[i].y : fa[i].y;
        const double nai = -ai;
        #pragma unroll
        for (int j = 0; j < FN; ++j) {
          const double br = fb[j].x;
          const double bi = (OPB == OP_C) ? -fb[j].y : fb[j].y;
          dmma884(cr[i][j][0], cr[i][j][1], ar, br);
          dmma884(ci[i][j][0], ci[i][j][1], ar, bi);
          dmma884(cr[i][j][0], cr[i][j][1], nai, bi);
          dmma884(ci[i][j][0], ci[i][j][1], ai, br);
        }
      }
    }
  }
  cp_async_wait<0>();

  // epilogue
  #pragma unroll
  for (int i = 0; i < FM; ++i) {
    const int m = m0 + wm * WM + i * 8 + fr;
    if (m >= p.M) continue;
    #pragma unroll
    for (int j = 0; j < FN; ++j) {
      #pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int n = n0 + wn * WN + j * 8 + fc * 2 + t;
        if (n >= p.N) continue;
        const double xr = cr[i][j][t], xi = ci[i][j][t];
        if (EPI == EPI_PARTIAL) {
          p.ws[(long long)blockIdx.z * p.M * p.N + m + (long long)n * p.M] = make_double2(xr, xi);
        } else if (EPI == EPI_FILTER) {
          // out = alpha*acc + beta*Y1 + gamma*Y0 with real coefficients
          double fa, fb, fg;
          filter_coef(p, fa, fb, fg);
          const double2 y1 = p.Y1e[m + (long long)n * p.ld1e];
          double orr = fa * xr + fb * y1.x;
          double oi = fa * xi + fb * y1.y;
          if (p.Y0 != nullptr) {
            const double2 y0 = p.Y0[m + (long long)n * p.ld0];
            orr += fg * y0.x;
            oi += fg * y0.y;
          }
          p.C[m + (long long)n * p.ldc] = make_double2(orr, oi);
        } else {
          double2 o = make_double2(p.alpha.x * xr - p.alpha.y * xi, p.alpha.x * xi + p.alpha.y * xr);
          if (p.beta.x != 0.0 || p.beta.y != 0.0) {
            const double2 c = p.C[m + (long long)n * p.ldc];
            o.x += p.beta.x * c.x - p.beta.y * c.y;
            o.y += p.beta.x * c.y + p.beta.y * c.x;
          }
          p.C[m + (long long)n * p.ldc] = o;
        }
      }
    }
  }
}

// Fixed-order split-K fix-up: C = alpha * sum_z ws[z] + beta * C.
__global__ void zgemm_splitk_reduce(int M, int N, int S, const double2* __restrict__ ws,
                                    double2 alpha, double2 beta, double2* C, long long ldc);

}  // namespace chfsi
