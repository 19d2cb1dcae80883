// Tile-configuration dispatch for the DMMA complex GEMM (zgemm.cuh).
//
// A small cost model picks, per call, the CTA tile (64x64, 64x32, 64x16 or
// 32x16) and a deterministic split-K factor so that the grid fills the 148
// SMs in whole waves: the filter's tail blocks are only nex+few columns wide
// (SURVEY.md section 0.5), where a single 64-row tile column would leave
// most SMs idle. Split-K partials are reduced in fixed z order, so results
// are bit-identical run to run (reference criterion 7, test_acceptance.py:199).
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cmath>
#include <string>
#include <mutex>
#include <unordered_map>

#include "internal.h"
#include "zgemm.cuh"
#include "zgemm_tma.cuh"

#include <cudaTypedefs.h>

namespace chfsi {

__global__ void zgemm_splitk_reduce_kernel(int M, int N, int S, const double2* __restrict__ ws,
                                           int epi, double2 alpha, double2 beta, double2* C,
                                           long long ldc, const double2* Y1, long long ld1,
                                           const double2* Y0, long long ld0, double gamma,
                                           const double* coef, double* Cs, long long ldcs) {
  if (coef != nullptr) {  // graph-replayed filter step: coefficients live on the device
    alpha.x = coef[0];
    beta.x = coef[1];
    gamma = coef[2];
  }
  const long long total = (long long)M * N;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(idx % M);
    const long long n = idx / M;
    double xr = 0.0, xi = 0.0;
    for (int z = 0; z < S; ++z) {
      const double2 v = ws[(long long)z * total + idx];
      xr += v.x;
      xi += v.y;
    }
    if (epi == EPI_FILTER) {
      const double2 y1 = Y1[m + n * ld1];
      double orr = __fma_rn(alpha.x, xr, __dmul_rn(beta.x, y1.x));
      double oi = __fma_rn(alpha.x, xi, __dmul_rn(beta.x, y1.y));
      if (Y0 != nullptr) {
        const double2 y0 = Y0[m + n * ld0];
        orr = __fma_rn(gamma, y0.x, orr);
        oi = __fma_rn(gamma, y0.y, oi);
      }
      C[m + n * ldc] = make_double2(orr, oi);
      if (Cs != nullptr) Cs[m + n * ldcs] = __dadd_rn(orr, oi);
    } else {
      double2 o = make_double2(alpha.x * xr - alpha.y * xi, alpha.x * xi + alpha.y * xr);
      if (beta.x != 0.0 || beta.y != 0.0) {
        const double2 c = C[m + n * ldc];
        o.x += beta.x * c.x - beta.y * c.y;
        o.y += beta.x * c.y + beta.y * c.x;
      }
      C[m + n * ldc] = o;
      if (Cs != nullptr) Cs[m + n * ldcs] = __dadd_rn(o.x, o.y);
    }
  }
}

namespace {

struct Cfg {
  int bm, bn, bk;
  int threads;
  int smem;
  int occ[3];  // per EPI, filled lazily; index by epi
};

// Kernel pointer table: [cfg][opa][opb][epi]
using KFn = void (*)(const GemmParams);

template <int BM, int BN, int BK, int WM, int WN, int ST>
struct CfgT {
  static constexpr int threads = (BM / WM) * (BN / WN) * 32;
  template <int OPA, int OPB>
  static constexpr int smem() { return zgemm_smem_bytes<BM, BN, BK, WM, WN, ST, OPA, OPB>(); }
  template <int OPA, int OPB, int EPI>
  static KFn fn() { return &zgemm_dmma_kernel<BM, BN, BK, WM, WN, ST, OPA, OPB, EPI>; }
};

constexpr int NCFG = 19;
constexpr int FIRST_TMA = 7;  // cfgs >= 7: TMA + mbarrier kernels (zgemm_tma.cuh), op N x N only
constexpr int FIRST_3M = 11;  // cfgs >= 11: the TMA kernels with 3M complex products
constexpr int FIRST_SUMS = 14;  // cfgs >= 14: 3M reading precomputed operand-sum planes
constexpr int FIRST_BSUMS = 17; // cfgs >= 17: 3M reading the B-sum plane only (A sums in the loop)
// cfg 0: 64x64   BK8  warp 32x32 (4 warps)     cfg 4: 64x64  BK16 warp 32x32, 3 stages
// cfg 1: 64x32   BK8  warp 32x16 (4 warps)     cfg 5: 128x64 BK8  warp 32x32 (8 warps)
// cfg 2: 64x16   BK8  warp 16x16 (4 warps)     cfg 6: 128x32 BK8  warp 32x16 (8 warps)
// cfg 3: 32x16   BK8  warp 16x8  (4 warps)
using C0 = CfgT<64, 64, 8, 32, 32, 4>;
using C1 = CfgT<64, 32, 8, 32, 16, 4>;
using C2 = CfgT<64, 16, 8, 16, 16, 4>;
using C3 = CfgT<32, 16, 8, 16, 8, 4>;
using C4 = CfgT<64, 64, 16, 32, 32, 3>;
using C5 = CfgT<128, 64, 8, 32, 32, 4>;
using C6 = CfgT<128, 32, 8, 32, 16, 4>;
// cfg 7: TMA 64x32 warp 32x16, 4 stages; cfg 8: TMA 64x16 warp 16x16; cfg 9: TMA 64x64 warp 32x32
// cfg 10: TMA 64x32 with four 16x32 warps stacked by rows (same fragment loads per DMMA as
// cfg 7; on a ragged column edge every warp keeps the same number of live 8-column blocks)
using TmaFn = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap,
                      const CUtensorMap, const GemmParams);
template <int BM, int BN, int WM, int WN, int ST, int MINB = 1, int MUL = 4, int SUMS = SUMS_NONE>
struct TmaT {
  static constexpr int threads = (BM / WM) * (BN / WN) * 32;
  static constexpr int smem() { return zgemm_tma_smem_bytes<BM, BN, WM, WN, ST, SUMS>(); }
  template <int EPI>
  static TmaFn fn() { return &zgemm_tma_kernel<BM, BN, WM, WN, ST, EPI, MINB, MUL, SUMS>; }
};
// (four-product TMA kernels: 3 CTAs / SM -- the unrolled main loop spills at 128 registers;
// 3 vs 4 CTAs / SM measured equal before the unroll. A register-double-buffered fragment
// variant measured 1.5-2 % slower, profiles/r01)
using T7 = TmaT<64, 32, 32, 16, 4, 3>;
using T8 = TmaT<64, 16, 16, 16, 4, 4>;
using T9 = TmaT<64, 64, 32, 32, 4, 2>;
using T10 = TmaT<64, 32, 16, 32, 4, 3>;
// cfg 11 / 12: cfg 7 / cfg 10 with 3M complex products (three real DMMA products per
// complex MAC; 48 accumulator doubles per thread -> 3 CTAs / SM)
using T11 = TmaT<64, 32, 32, 16, 4, 3, 3>;
using T12 = TmaT<64, 32, 16, 32, 4, 3, 3>;
// cfg 13: 3M, 64x32 with eight 16x16 warps (24 accumulator doubles: 2 CTAs / SM = 16 warps)
using T13 = TmaT<64, 32, 16, 16, 4, 2, 3>;
// cfg 14 / 15: cfg 11 / 12 reading precomputed operand-sum planes (3M without in-loop DADDs)
using T14 = TmaT<64, 32, 32, 16, 4, 3, 3, SUMS_BOTH>;
using T15 = TmaT<64, 32, 16, 32, 4, 3, 3, SUMS_BOTH>;
// cfg 16: sum planes, 64x24 tile of four 16x24 warps stacked by rows: 24-column tiles
// fit block widths that 32-column tiles round up badly (a 550-column shard: 23 x 24 =
// 552 vs 18 x 32 = 576 columns of work)
using T16 = TmaT<64, 24, 16, 24, 4, 3, 3, SUMS_BOTH>;
// cfg 17 / 18: cfg 15 / 16 reading only the B-sum plane: H streams at 16 bytes per element
// (no H sum plane) and Ar + Ai costs FM = 2 DADDs per 24 (18) DMMAs -- the narrow-block
// plan, where streaming 24 bytes per element of H holds the board at its power cap
using T17 = TmaT<64, 32, 16, 32, 4, 3, 3, SUMS_B>;
using T18 = TmaT<64, 24, 16, 24, 4, 3, 3, SUMS_B>;
const int kBM[NCFG] = {64, 64, 64, 32, 64, 128, 128, 64, 64, 64, 64, 64, 64, 64, 64, 64, 64, 64, 64};
const int kBN[NCFG] = {64, 32, 16, 16, 64, 64, 32, 32, 16, 64, 32, 32, 32, 32, 32, 32, 24, 32, 24};
const int kBKc[NCFG] = {8, 8, 8, 8, 16, 8, 8, 8, 8, 8, 8, 8, 8, 8, 8, 8, 8, 8, 8};
const int kWN[NCFG] = {32, 16, 16, 8, 32, 32, 16, 16, 16, 32, 32, 16, 32, 16, 16, 32, 24, 32, 24};  // warp tile width
bool g_tma_enabled = true;
// complex products in the TMA kernels: 3 (3M, default) or 4 real DMMA products
int g_mul = [] {
  const char* e = getenv("CHFSI_COMPLEX_MUL");
  return (e && atoi(e) == 4) ? 4 : 3;
}();
int g_force_cfg = -1, g_force_split = 0;

struct Entry {
  KFn fn = nullptr;
  int threads = 0, smem = 0, occ = 0;
  bool ready = false;
  bool tma = false;
};
Entry g_table[NCFG][2][2][3];
bool g_table_init = false;
// cudaFuncSetAttribute is per device: the devices whose attributes are set (bit i =
// ordinal i; one process may drive several GPUs, one engine per device)
unsigned long long g_table_devices = 0;
std::mutex g_table_mu;

template <class C, int OPA, int OPB, int EPI>
void put(int ci) {
  Entry& e = g_table[ci][OPA][OPB][EPI];
  e.fn = C::template fn<OPA, OPB, EPI>();
  e.threads = C::threads;
  e.smem = C::template smem<OPA, OPB>();
}

template <class C>
void put_all(int ci) {
  put<C, 0, 0, 0>(ci); put<C, 0, 0, 1>(ci); put<C, 0, 0, 2>(ci);
  put<C, 1, 0, 0>(ci); put<C, 1, 0, 2>(ci);
  put<C, 0, 1, 0>(ci); put<C, 0, 1, 2>(ci);
  put<C, 1, 1, 0>(ci); put<C, 1, 1, 2>(ci);
}

template <class T>
void put_tma(int ci) {
  const TmaFn fns[3] = {T::template fn<EPI_STORE>(), T::template fn<EPI_FILTER>(),
                        T::template fn<EPI_PARTIAL>()};
  for (int e = 0; e < 3; ++e) {
    Entry& en = g_table[ci][OP_N][OP_N][e];
    en.fn = reinterpret_cast<KFn>(fns[e]);
    en.threads = T::threads;
    en.smem = T::smem();
    en.tma = true;
  }
}

void fill_table();

int ensure_table() {
  int dev = 0;
  CHFSI_CUDA(cudaGetDevice(&dev));
  const unsigned long long bit = (dev < 64) ? (1ULL << dev) : 0ULL;
  std::lock_guard<std::mutex> lock(g_table_mu);
  if (g_table_init && (g_table_devices & bit)) return OK;
  if (!g_table_init) fill_table();
  for (int c = 0; c < NCFG; ++c)
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b)
        for (int e = 0; e < 3; ++e) {
          Entry& en = g_table[c][a][b][e];
          if (!en.fn) continue;
          CHFSI_CUDA(cudaFuncSetAttribute((const void*)en.fn,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, en.smem));
          if (g_table_init) continue;  // occupancy: the same on every B200
          int occ = 0;
          CHFSI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)en.fn,
                                                                   en.threads, en.smem));
          en.occ = std::max(occ, 1);
          en.ready = true;
        }
  g_table_devices |= bit;
  if (g_table_init) return OK;
  g_table_init = true;
  if (getenv("CHFSI_PLAN_DEBUG")) {
    for (int c = 0; c < NCFG; ++c)
      fprintf(stderr, "chfsi cfg %d: occ NN store %d filter %d partial %d, CN store %d partial %d\n", c,
              g_table[c][0][0][0].occ, g_table[c][0][0][1].occ, g_table[c][0][0][2].occ,
              g_table[c][1][0][0].occ, g_table[c][1][0][2].occ);
  }
  return OK;
}

void fill_table() {
  put_all<C0>(0);
  put_all<C1>(1);
  put_all<C2>(2);
  put_all<C3>(3);
  put_all<C4>(4);
  put_all<C5>(5);
  put_all<C6>(6);
  put_tma<T7>(7);
  put_tma<T8>(8);
  put_tma<T9>(9);
  put_tma<T10>(10);
  put_tma<T11>(11);
  put_tma<T12>(12);
  put_tma<T13>(13);
  put_tma<T14>(14);
  put_tma<T15>(15);
  put_tma<T16>(16);
  put_tma<T17>(17);
  put_tma<T18>(18);
}

struct Plan {
  int cfg = 0;
  int split = 1;
  int k_chunk = 0;
  // mixed tiling (cfg 15 only): n_wide 32-column tiles, then n_narrow 24-column tiles
  int n_wide = 0, n_narrow = 0;
};

// Launch-time model (microseconds), fitted by scripts/fit_cost_model.py to 2900
// measured (shape, config, split) points on B200 (profiles/r01/tune_sweep_*.json; the
// model's pick is within 1.8 % of the best measured plan on geometric mean):
//   * every SM runs q = ceil(CTAs / SMs) CTAs, at most occ at a time; r CTAs sharing
//     the SM's DMMA pipe progress at min(1, r / R0) of it, so a round of r costs
//     W * max(r, R0) / (eff * peak), W = BM * live columns * K-chunk;
//   * a ragged last column tile does DMMA work for its live 8-column blocks only but
//     costs at least kFloor of a full tile (its loads are not skipped); when its live
//     blocks are spread unevenly over the warp columns the CTA waits for the heavy
//     warps (ncu: DMMA pipe 92.5 % vs 95.7 % active at k = 210): x (1 + kRag / tiles_n);
//   * split-K adds the reduce pass: kTred + (s + 3) M N 16 B at HBM speed.
constexpr double kEffNN[NCFG] = {0.906, 0.898, 0.837, 0.823, 0.911, 0.926, 0.885,
                                 0.966, 0.915, 0.962, 0.954, 1.17, 1.16, 1.13, 1.27, 1.26, 1.24,
                                 1.22, 1.20};
constexpr double kEffCN[7] = {0.886, 0.927, 0.877, 0.854, 1.058, 0.971, 0.887};
constexpr double kR0Warps4 = 1.289, kR0Warps8 = 1.108;
constexpr double kRag = 0.122, kFloor = 0.859;
constexpr double kT0 = 5.583, kTred = 3.101, kHbmBytesPerUs = 6.58e6;
constexpr double kPeakCmacPerUsPerSm = 37.16e12 / 8.0 / 1e6 / 148.0;

double plan_cost(int c, int occ, int threads, bool nn, int sms, long long M, long long N,
                 long long K, int s) {
  const long long tm = (M + kBM[c] - 1) / kBM[c];
  const long long tn = (N + kBN[c] - 1) / kBN[c];
  const long long ctas = tm * tn * s;
  const long long q = (ctas + sms - 1) / sms;
  const double r0 = threads >= 256 ? kR0Warps8 : kR0Warps4;
  const double kchunk = (double)((K + s - 1) / s);
  const long long last = ((N - (tn - 1) * kBN[c] + 7) / 8) * 8;
  const double live = ((double)(tn - 1) * kBN[c] +
                       std::max((double)last, kFloor * kBN[c])) / (double)tn;
  const double W = kBM[c] * live * kchunk;
  const long long full = q / occ, rem = q % occ;
  const double rounds = (double)full * std::max((double)occ, r0) +
                        (rem ? std::max((double)rem, r0) : 0.0);
  const double eff = nn ? kEffNN[c] : kEffCN[std::min(c, 6)];
  double t = W * rounds / (eff * kPeakCmacPerUsPerSm);
  // live 8-column blocks of the last column tile per warp column
  const int per = kWN[c] / 8, wcols = kBN[c] / kWN[c];
  const int vb = (int)(last / 8);
  int lo = per, hi = 0;
  for (int w = 0; w < wcols; ++w) {
    const int l = std::max(0, std::min(per, vb - w * per));
    lo = std::min(lo, l);
    hi = std::max(hi, l);
  }
  if (hi != lo) t *= 1.0 + kRag / (double)tn;
  t += kT0;
  if (s > 1) t += kTred + (double)(s + 3) * (double)M * (double)N * 16.0 / kHbmBytesPerUs;
  return t;
}

// Sum-plane filter steps on large operators (M >= 8192): a measured rule instead of the
// cost model. Tile width: the fewest padded columns, ceil(N / BN) * BN, 24-column tiles
// weighted x1.01 and 32-column tiles with unevenly live warp columns (cfg 14 on a
// ragged edge) x(1 + 0.12 / tiles_n); split-K: ~20000 CTAs. On the sweep at n = 20000
// (profiles/r01/sweep_sums16_20000.json, 12 widths 26-2200) the rule's pick is within
// 0.7 % of the best measured plan on geometric mean (worst 2.9 %); the cost model's
// pick was 1.7 % (worst 15.7 %: it under-splits mid widths, e.g. k = 400 at split 1).
long long rule_min_m() {
  static const long long v = [] {
    const char* e = getenv("CHFSI_RULE_MIN_M");  // tuning only
    return e ? atoll(e) : 8192LL;
  }();
  return v;
}
constexpr double kRuleTargetCtas = 20000.0;

// Power: a sum-plane kernel streams H and its 3M sum plane (24 bytes per element of
// H); on a narrow block that is 9.6 GB per step at n = 20000 for little tensor work, and
// the B200 then runs at its 1 kW cap with the SM clock well under 1965 MHz (sustained
// degree-25 filter calls, profiles/r02/narrow_plans.json: k = 26 2.50 ms per step at
// 1700 MHz, k = 51 4.27 ms at 1777 MHz, k = 101 7.98 ms at 1867 MHz). The B-sum-only
// kernels (cfg 17 / 18) read H alone (16 bytes per element) and form Ar + Ai in the loop
// (2 DADDs per 24 DMMAs; the all-in-loop kernel cfg 11 / 12 pays 6). Blocks of
// bsums_min_n() .. bsums_max_n() columns take them; CHFSI_NARROW_INLOOP=0 disables.
long long bsums_min_n() {
  static const long long v = [] {
    const char* e = getenv("CHFSI_BSUMS_MIN_N");  // tuning only
    return e ? atoll(e) : 17LL;
  }();
  return v;
}
long long bsums_max_n() {
  static const long long v = [] {
    const char* e = getenv("CHFSI_BSUMS_MAX_N");  // tuning only
    return e ? atoll(e) : 64LL;
  }();
  return v;
}
bool mixed_tiles() {
  static const bool on = [] {
    const char* e = getenv("CHFSI_MIXED_TILES");  // tuning only
    return !(e && atoi(e) == 0);
  }();
  return on;
}
bool narrow_bsums(long long N) {
  static const bool on = [] {
    const char* e = getenv("CHFSI_NARROW_INLOOP");
    return !(e && atoi(e) == 0);
  }();
  return on && N >= bsums_min_n() && N <= bsums_max_n();
}

Plan choose_sums_rule(long long M, long long N, long long K) {
  Plan best;
  double best_score = 1e300;
  const long long tm = (M + 63) / 64;
  // the kernel family: both sum planes, or (narrow blocks) the B-sum plane only
  const bool bonly = narrow_bsums(N);
  const int c_lo = bonly ? FIRST_BSUMS : FIRST_SUMS, c_hi = bonly ? NCFG : FIRST_BSUMS;
  for (int c = c_lo; c < c_hi; ++c) {
    const long long tn = (N + kBN[c] - 1) / kBN[c];
    const long long last = (N - (tn - 1) * kBN[c] + 7) / 8;
    const int per = kWN[c] / 8, wcols = kBN[c] / kWN[c];
    int lo = per, hi = 0;
    for (int w = 0; w < wcols; ++w) {
      const int l = (int)std::max<long long>(0, std::min<long long>(per, last - w * per));
      lo = std::min(lo, l);
      hi = std::max(hi, l);
    }
    double score = (double)(tn * kBN[c]);
    if (hi != lo) score *= 1.0 + 0.12 / (double)tn;
    if (kBN[c] == 24) score *= 1.01;
    if (c == FIRST_SUMS + 1) score *= 1.004;  // row-stacked 32-wide warps: last resort
    if (score < best_score) {
      best_score = score;
      best.cfg = c;
    }
  }
  // Mixed tiling: 8 m columns of DMMA work are covered exactly by a 32-column and b
  // 24-column tiles of the row-stacked 32-wide kernel (cfg 15: every warp spans the tile's
  // columns, so a 24-column tile keeps 3 live blocks in every warp) in one launch --
  // no ragged last tile, whose loads cost >= 0.86 of a full tile whatever it holds.
  // Measured at n = 20000 (profiles/r02/mixed_tiles.json): k = 80 +6.1 %, 100-104 +5 %,
  // 200 +3.5 %; equal within 0.3 % where the plain plans pad little (201-232, 400); worse
  // on wide blocks (1100: -6.7 %, 2200: -9.3 %) and at 136 (-1.4 %). So it is taken only
  // up to 512 columns and when the best plain plan pads >= 7 % more columns.
  if (!bonly && mixed_tiles() && N <= 512) {
    const long long m8 = (N + 7) / 8;
    const long long pad_plain =
        ((N + kBN[best.cfg] - 1) / kBN[best.cfg]) * (long long)kBN[best.cfg];
    for (long long b = 1; b <= 3; ++b) {
      const long long rest = m8 - 3 * b;
      if (rest < 0 || rest % 4 != 0) continue;
      const long long a = rest / 4;
      if (a < 1) break;  // 24-column tiles only: cfg 16 is that plan
      if ((double)pad_plain >= 1.07 * (double)(8 * m8)) {
        best.cfg = FIRST_SUMS + 1;
        best.n_wide = (int)a;
        best.n_narrow = (int)b;
      }
      break;
    }
  }
  const long long tn = best.n_narrow > 0 ? best.n_wide + best.n_narrow
                                         : (N + kBN[best.cfg] - 1) / kBN[best.cfg];
  const long long ktiles = std::max<long long>(1, (K + 7) / 8);
  const long long ws_cap = std::max<long long>(1, (1LL << 30) / std::max<long long>(1, M * N * 16));
  // (narrow kernels on two column tiles: split 24 measured 1.6 % ahead of 16 at k = 51)
  const long long s_max =
      std::max<long long>(1, std::min<long long>({bonly ? 24 : 17, ktiles / 4, ws_cap}));
  // the nearest (in log) of the swept split factors
  const double s_t = kRuleTargetCtas / (double)(tm * tn);
  static const int kSplits[] = {1, 2, 3, 4, 6, 8, 12, 16, 24};
  int s_best = 1;
  for (int s : kSplits) {
    if (s == 24 && !bonly) continue;
    if (std::fabs(std::log((double)s / s_t)) < std::fabs(std::log((double)s_best / s_t))) s_best = s;
  }
  // one column tile: split 8 measured best of 4 ... 14 (k = 26: 2.19 ms vs 2.20-2.26)
  if (bonly && tn == 1) s_best = std::min(s_best, 8);
  best.split = (int)std::max<long long>(1, std::min<long long>(s_best, s_max));
  best.k_chunk = (int)(((ktiles + best.split - 1) / best.split) * 8);
  return best;
}

Plan choose(Handle* h, int opa, int opb, int epi, long long M, long long N, long long K,
            bool sums, bool tma = true) {
  tma = tma && g_tma_enabled;
  Plan best;
  double best_cost = 1e300;
  const int sms = h->sm_count;
  const bool nn = (opa == OP_N && opb == OP_N);
  if (sums && M >= rule_min_m() && g_force_cfg < 0 && g_force_split <= 0)
    return choose_sums_rule(M, N, K);
  for (int c = 0; c < NCFG; ++c) {
    if (g_force_cfg >= 0 && c != g_force_cfg) continue;
    if (c >= FIRST_TMA && !tma) continue;
    if (g_force_cfg < 0 && c >= FIRST_TMA && (c >= FIRST_3M) != (g_mul == 3)) continue;
    // 3M on: every op N x N product runs a 3M kernel (the cp.async kernels use four
    // products), so the rounding of a product does not depend on the planner's pick
    if (g_force_cfg < 0 && nn && g_mul == 3 && tma && K > 0 && c < FIRST_3M) continue;
    // operand-sum planes: only (and always) the sum-reading kernels; never without planes
    if (c >= FIRST_SUMS && !sums && g_force_cfg < 0) continue;
    if (c >= FIRST_BSUMS && g_force_cfg < 0) continue;  // B-sum-only kernels: the width rule's
    if (g_force_cfg < 0 && sums && c < FIRST_SUMS) continue;
    const Entry& e = g_table[c][opa][opb][epi == EPI_FILTER ? EPI_FILTER : EPI_STORE];
    const Entry& ep = g_table[c][opa][opb][EPI_PARTIAL];
    if (!e.ready && !ep.ready) continue;
    const int bk = kBKc[c];
    const long long ktiles = std::max<long long>(1, (K + bk - 1) / bk);
    int max_split = (int)std::min<long long>(64, ktiles / (32 / bk));
    // cap the split-K workspace at 1 GiB
    const long long ws_cap = (1LL << 30) / std::max<long long>(1, M * N * 16LL);
    max_split = (int)std::min<long long>(max_split, std::max<long long>(1, ws_cap));
    int s_lo = 1, s_hi = std::max(1, max_split);
    if (g_force_split > 0) s_lo = s_hi = g_force_split;
    for (int s = s_lo; s <= s_hi; ++s) {
      const Entry& en = (s == 1) ? e : ep;
      if (!en.ready) continue;
      const long long kt_per = (ktiles + s - 1) / s;
      const double cost = plan_cost(c, en.occ, en.threads, nn, sms, M, N, K, s);
      if (cost < best_cost * 0.999) {
        best_cost = cost;
        best.cfg = c;
        best.split = s;
        best.k_chunk = (int)(kt_per * bk);
      }
    }
  }
  return best;
}

// Plans are pure functions of (ops, epilogue, shape, overrides): memoise them so the
// per-call host cost of a small GEMM is a hash lookup (the solve's tail issues
// thousands of identical small products).
struct PlanKey {
  int opa, opb, epi, fcfg, fsplit, mul, sums, tma, sms;
  long long M, N, K;
  bool operator==(const PlanKey& o) const {
    return opa == o.opa && opb == o.opb && epi == o.epi && fcfg == o.fcfg && fsplit == o.fsplit &&
           mul == o.mul && sums == o.sums && tma == o.tma && sms == o.sms &&
           M == o.M && N == o.N && K == o.K;
  }
};
struct PlanKeyHash {
  size_t operator()(const PlanKey& k) const {
    size_t h = (size_t)k.M * 0x9E3779B97F4A7C15ULL;
    h ^= (size_t)k.N * 0xC2B2AE3D27D4EB4FULL + (h << 6) + (h >> 2);
    h ^= (size_t)k.K * 0x165667B19E3779F9ULL + (h << 6) + (h >> 2);
    h ^= (size_t)(k.opa | (k.opb << 1) | (k.epi << 2) | ((k.fcfg + 1) << 4) | (k.fsplit << 9) |
                  (k.mul << 16) | (k.sums << 20) | (k.tma << 21) | ((size_t)k.sms << 22));
    return h;
  }
};

Plan cached_plan(Handle* h, int opa, int opb, int epi, long long M, long long N, long long K,
                 bool sums, bool tma = true) {
  // shared by every handle (one per device, possibly on several host threads)
  static std::unordered_map<PlanKey, Plan, PlanKeyHash> cache;
  static std::mutex mu;
  const PlanKey key{opa, opb, epi, g_force_cfg, g_force_split, g_mul, sums ? 1 : 0, tma ? 1 : 0,
                    h->sm_count, M, N, K};
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  const Plan pl = choose(h, opa, opb, epi, M, N, K, sums, tma);
  std::lock_guard<std::mutex> lock(mu);
  if (cache.size() > 65536) cache.clear();
  cache.emplace(key, pl);
  return pl;
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// Column-major complex matrix (rows x cols, ld) seen as a 2-D FP64 tensor
// {2*rows doubles, cols}, box {16 doubles = 8 complex rows, box_cols}, 128-B swizzle.
int encode_colmajor(CUtensorMap* map, const double2* base, long long rows, long long cols,
                    long long ld, int box_rows, int box_cols) {
  auto enc = tensor_map_encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled entry point unavailable");
    return ERR_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)(2 * rows), (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 16)};
  cuuint32_t box[2] = {(cuuint32_t)(2 * box_rows), (cuuint32_t)box_cols};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return ERR_CUDA;
  }
  return OK;
}

// Real column-major plane (rows x cols doubles, ld) as a 2-D FP64 tensor, box
// {box_rows, box_cols}; 64-byte swizzle for the Bs tile (conflict-free fragment reads).
int encode_real(CUtensorMap* map, const double* base, long long rows, long long cols, long long ld,
                int box_rows, int box_cols, bool swizzle64) {
  auto enc = tensor_map_encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled entry point unavailable");
    return ERR_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 8)};
  cuuint32_t box[2] = {(cuuint32_t)box_rows, (cuuint32_t)box_cols};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         swizzle64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (sum plane) failed: " + std::to_string((int)r));
    return ERR_CUDA;
  }
  return OK;
}

int encode_3d(CUtensorMap* map, const void* base, const cuuint64_t dims[3],
              const cuuint64_t strides[2], const cuuint32_t box[3], CUtensorMapSwizzle sw) {
  auto enc = tensor_map_encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled entry point unavailable");
    return ERR_CUDA;
  }
  cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims,
                         strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (3-D) failed: " + std::to_string((int)r));
    return ERR_CUDA;
  }
  return OK;
}

// A (column-major, M % 8 == 0) as one 3-D box per stage {16 doubles of an 8-row
// group, BK columns (ld * 16 B), BM/8 groups (128 B apart)}, 128-byte swizzle (four TMA
// issues per stage with sum planes instead of 2 BM/8 + 2: the producer lane's issue
// code had been ~6 % of warp stall samples).
int encode_a3d(CUtensorMap* ma, const GemmParams& p, int bm, int bk) {
  const cuuint64_t G = (cuuint64_t)(p.M / 8);
  // dims ordered {row-in-group, column, group} so the box lands as [group][col][row]
  // (the 2-D kernels' layout; the swizzle phase is the column): strides not monotone
  const cuuint64_t dims[3] = {16, (cuuint64_t)p.K, G};
  const cuuint64_t strides[2] = {(cuuint64_t)p.lda * 16, 128};
  const cuuint32_t box[3] = {16, (cuuint32_t)bk, (cuuint32_t)(bm / 8)};
  return encode_3d(ma, p.A, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

// Sum-plane kernels: A as above; As in the grouped layout {8 rows, K columns (64 B),
// M/8 groups}.
int encode_sums_a(CUtensorMap* ma, CUtensorMap* mas, const GemmParams& p, int bm, int bk) {
  const cuuint64_t G = (cuuint64_t)(p.M / 8);
  CHFSI_TRY(encode_a3d(ma, p, bm, bk));
  const cuuint64_t dims[3] = {8, (cuuint64_t)p.K, G};
  const cuuint64_t strides[2] = {64, (cuuint64_t)p.K * 64};
  const cuuint32_t box[3] = {8, (cuuint32_t)bk, (cuuint32_t)(bm / 8)};
  return encode_3d(mas, p.As, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE);
}

int run_kernel(Handle* h, int c, const Entry& e, dim3 grid, const GemmParams& p) {
  if (!e.tma) {
    e.fn<<<grid, e.threads, e.smem, h->stream>>>(p);
  } else {
    // A: M x K (8-row boxes, BK = 8 columns); B: K x N (BK rows, BN columns)
    CUtensorMap ma, mb, mas, mbs;
    if (p.a3d)
      CHFSI_TRY(encode_a3d(&ma, p, kBM[c], kBKc[c]));
    else
      CHFSI_TRY(encode_colmajor(&ma, p.A, p.M, p.K, p.lda, 8, kBKc[c]));
    CHFSI_TRY(encode_colmajor(&mb, p.B, p.K, p.N, p.ldb, kBKc[c], kBN[c]));
    if (c >= FIRST_SUMS) {
      if (c < FIRST_BSUMS)
        CHFSI_TRY(encode_sums_a(&ma, &mas, p, kBM[c], kBKc[c]));
      else
        mas = ma;  // B-sum plane only (A is the 3-D box encoded above: sums imply M % 8 == 0)
      CHFSI_TRY(encode_real(&mbs, p.Bs, p.K, p.N, p.ldbs, kBKc[c], kBN[c], true));
    } else {
      mas = ma;
      mbs = mb;
    }
    reinterpret_cast<TmaFn>(e.fn)<<<grid, e.threads, e.smem, h->stream>>>(ma, mb, mas, mbs, p);
  }
  h->launches++;
  CHFSI_CHECK_LAUNCH();
  return OK;
}

int launch_plan(Handle* h, int opa, int opb, int epi, long long M, long long N, long long K,
                GemmParams p, const Plan& pl);

int launch(Handle* h, int opa, int opb, int epi, long long M, long long N, long long K,
           GemmParams p) {
  CHFSI_TRY(ensure_table());
  if (M <= 0 || N <= 0) return OK;
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) {
    set_error("zgemm: dimension exceeds int32");
    return ERR_ARG;
  }
  p.M = (int)M;
  p.N = (int)N;
  p.K = (int)K;
  // the TMA kernels load whole 8-column K tiles and cannot mask a triangular K bound
  // that is not a multiple of 8 (the cp.async kernels mask every element)
  const bool tma = g_tma_enabled && !(p.tri != 0 && (p.tri_off & 7) != 0);
  const bool sums = p.As != nullptr && p.Bs != nullptr && g_mul == 3 && opa == OP_N &&
                    opb == OP_N && tma && M % 8 == 0;
  const Plan pl = cached_plan(h, opa, opb, epi, M, N, K, sums, tma);
  const int c = pl.cfg;
  p.a3d = (M % 8 == 0) ? 1 : 0;  // one 3-D A box per stage (TMA kernels)
  static const int pack_tail = [] {
    const char* e = getenv("CHFSI_PACK_TAIL");  // tuning only
    return (e && atoi(e) == 0) ? 0 : 1;
  }();
  p.pack = pack_tail;
  if (c >= FIRST_SUMS && !sums) {
    set_error("zgemm: forced config " + std::to_string(c) + " needs operand sum planes");
    return ERR_ARG;
  }
  // a kernel that does not read the planes (forced config, 4 products, TMA off) leaves
  // the output plane to a separate pass after the product
  double* cs_after = nullptr;
  if (c < FIRST_SUMS) {
    p.As = p.Bs = nullptr;
    cs_after = p.Cs;
    p.Cs = nullptr;
  }
  CHFSI_TRY(launch_plan(h, opa, opb, epi, M, N, K, p, pl));
  if (cs_after != nullptr) CHFSI_TRY(sum_plane(h, M, N, p.C, p.ldc, cs_after, p.ldcs));
  return OK;
}

int launch_plan(Handle* h, int opa, int opb, int epi, long long M, long long N, long long K,
                GemmParams p, const Plan& pl) {
  const int c = pl.cfg;
  p.tiles_m = (int)((M + kBM[c] - 1) / kBM[c]);
  p.tiles_n = (int)((N + kBN[c] - 1) / kBN[c]);
  p.n_wide = 0;
  if (pl.n_narrow > 0) {  // mixed tiling: n_wide full tiles, then n_narrow of BN - 8 columns
    p.n_wide = pl.n_wide;
    p.tiles_n = pl.n_wide + pl.n_narrow;
  }
  // Row-major raster (consecutive CTAs share one H row strip). A grouped raster
  // (several row tiles per wave sharing Y strips) measured 1.5 % slower on B200
  // with the cp.async kernel (profiles/r01), so group = 1 unless CHFSI_RASTER_GROUP
  // (tuning only) says otherwise.
  // TMA kernels: when the B panel (16 K N bytes) overflows L2, group row tiles so one
  // resident wave covers `group` row tiles x all column tiles and the Y strips are
  // re-read from L2: DRAM 115 -> 78 GB per c4 filter launch at identical speed
  // (profiles/r01/raster.json); narrow blocks (Y resident in L2) keep group 1.
  static const int env_group = [] {
    const char* s = getenv("CHFSI_RASTER_GROUP");
    return s ? std::max(1, atoi(s)) : 0;
  }();
  int group = 1;
  // (split-K: the panel of one K chunk; at k = 210, split 8 the full-K test had grouped
  // anyway and read 56 GB of DRAM per launch instead of 12.7 GB, at equal speed)
  const double panel_k = pl.split > 1 ? (double)pl.k_chunk : (double)K;
  if (g_table[c][opa][opb][epi].tma && 16.0 * panel_k * (double)N > 64e6) {
    const long long resident = (long long)g_table[c][opa][opb][epi].occ * h->sm_count;
    group = (int)std::max<long long>(1, resident / std::max(1, p.tiles_n));
  }
  if (env_group > 0) group = env_group;
  p.group = std::max(1, std::min(group, p.tiles_m));
  const unsigned ntiles = (unsigned)((long long)p.tiles_m * p.tiles_n);
  if (pl.split == 1) {
    return run_kernel(h, c, g_table[c][opa][opb][epi], dim3(ntiles, 1, 1), p);
  }
  const size_t ws_bytes = (size_t)pl.split * M * N * sizeof(double2);
  // while a filter graph is being captured, partials go to the graph's own workspace
  double2* ws = (h->ws_override && h->ws_override_bytes >= ws_bytes)
                    ? h->ws_override
                    : (double2*)scratch(h, SLOT_SPLITK, ws_bytes);
  if (!ws) return ERR_NOMEM;
  GemmParams q = p;
  q.k_chunk = pl.k_chunk;
  q.ws = ws;
  CHFSI_TRY(run_kernel(h, c, g_table[c][opa][opb][EPI_PARTIAL], dim3(ntiles, 1, (unsigned)pl.split),
                       q));
  const long long total = M * N;
  const int threads = 256;
  const int blocks = (int)std::min<long long>((total + threads - 1) / threads, 148LL * 16);
  zgemm_splitk_reduce_kernel<<<blocks, threads, 0, h->stream>>>(
      (int)M, (int)N, pl.split, ws, epi, p.alpha, p.beta, p.C, p.ldc, p.Y1e, p.ld1e, p.Y0, p.ld0,
      p.gamma, epi == EPI_FILTER ? p.coef : nullptr, p.Cs, p.ldcs);
  h->launches++;
  CHFSI_CHECK_LAUNCH();
  return OK;
}

}  // namespace

int gemm_override(int cfg, int split) {
  if (cfg >= NCFG || split < 0 || split > 64) {
    set_error("gemm_override: cfg must be < " + std::to_string(NCFG) + " and split in [0, 64]");
    return ERR_ARG;
  }
  g_force_cfg = cfg;
  g_force_split = split;
  return OK;
}

int set_complex_mul(int mul) {
  if (mul != 3 && mul != 4) {
    set_error("set_complex_mul: mul must be 3 (3M) or 4");
    return ERR_ARG;
  }
  g_mul = mul;
  return OK;
}

int complex_mul() { return g_mul; }

void gemm_overrides(int* cfg, int* split) {
  *cfg = g_force_cfg;
  *split = g_force_split;
}

int gemm_plan(Handle* h, int opa, int opb, int epi, long long M, long long N, long long K,
              int* cfg, int* split) {
  CHFSI_TRY(ensure_table());
  const bool sums = epi == 2 && g_mul == 3 && opa == OP_N && opb == OP_N && g_tma_enabled;
  const Plan pl = choose(h, opa, opb, epi ? EPI_FILTER : EPI_STORE, M, N, K, sums);
  *cfg = pl.cfg;
  *split = pl.split;
  return OK;
}

int zgemm(Handle* h, int opa, int opb, long long M, long long N, long long K, double2 alpha,
          const double2* A, long long lda, const double2* B, long long ldb, double2 beta,
          double2* C, long long ldc, int tri, long long tri_off) {
  if ((opa != OP_N && opa != OP_C) || (opb != OP_N && opb != OP_C)) {
    set_error("zgemm: op must be 0 (N) or 1 (C)");
    return ERR_ARG;
  }
  GemmParams p{};
  p.A = A; p.lda = lda;
  p.B = B; p.ldb = ldb;
  p.C = C; p.ldc = ldc;
  p.alpha = alpha; p.beta = beta;
  p.Y0 = nullptr; p.ld0 = 0; p.gamma = 0.0;
  // a triangular operand is square in the full factor; C covers rows (A flags) or
  // columns (B flags) [tri_off, tri_off + M or N) of it
  const bool a_tri = tri & (TRI_A_LOWER | TRI_A_UPPER), b_tri = tri & (TRI_B_LOWER | TRI_B_UPPER);
  if ((tri & TRI_C_LOWER) && M != N) {
    set_error("zgemm: a lower-triangle-only C must be square");
    return ERR_ARG;
  }
  if (tri & ~(TRI_A_LOWER | TRI_B_UPPER | TRI_B_LOWER | TRI_A_UPPER | TRI_C_LOWER)) {
    set_error("zgemm: unknown tri flags");
    return ERR_ARG;
  }
  if ((a_tri && b_tri) || tri_off < 0 || (a_tri && tri_off + M > K) ||
      (b_tri && tri_off + N > K)) {
    set_error("zgemm: tri flags need one triangular operand of order K covering C");
    return ERR_ARG;
  }
  if (((tri & TRI_A_LOWER) && opa != OP_N) || ((tri & TRI_A_UPPER) && opa != OP_C) ||
      ((tri & TRI_B_LOWER) && opb != OP_N) || ((tri & TRI_B_UPPER) && opb != OP_C)) {
    set_error("zgemm: tri flag does not match the operand's op (lower: N, L^H: C)");
    return ERR_ARG;
  }
  p.tri = tri;
  p.tri_off = (int)tri_off;
  // a matrix-vector product is HBM-bound: a dedicated GEMV instead of padding the one
  // column to an 8-wide tensor-core tile (the Lanczos H v)
  if (N == 1 && opa == OP_N && opb == OP_N && tri == 0 && M >= 256 && K >= 1 &&
      g_force_cfg < 0)
    return zgemv_n(h, M, K, alpha, A, lda, B, beta, C);
  return launch(h, opa, opb, EPI_STORE, M, N, K, p);
}

int zgemm_nn_sums(Handle* h, long long M, long long N, long long K, const double2* A, long long lda,
                  const double2* B, long long ldb, double2* C, long long ldc,
                  const SumPlanes* sp) {
  GemmParams p{};
  p.A = A; p.lda = lda;
  p.B = B; p.ldb = ldb;
  p.C = C; p.ldc = ldc;
  p.alpha = make_double2(1.0, 0.0);
  p.beta = make_double2(0.0, 0.0);
  if (sp != nullptr) {
    p.As = sp->As; p.ldas = sp->ldas;
    p.Bs = sp->Bs; p.ldbs = sp->ldbs;
    p.Cs = sp->Cs; p.ldcs = sp->ldcs;
  }
  return launch(h, OP_N, OP_N, EPI_STORE, M, N, K, p);
}

int zgemm_filter_panel(Handle* h, long long M, long long N, long long K, const double2* A,
                       long long lda, const double2* B, long long ldb, const double2* Y1e,
                       long long ld1e, double alpha, double beta, const double2* Y0, long long ld0,
                       double gamma, double2* C, long long ldc, const double* coef_dev,
                       const SumPlanes* sp) {
  GemmParams p{};
  if (sp != nullptr) {
    p.As = sp->As; p.ldas = sp->ldas;
    p.Bs = sp->Bs; p.ldbs = sp->ldbs;
    p.Cs = sp->Cs; p.ldcs = sp->ldcs;
  }
  p.A = A; p.lda = lda;
  p.B = B; p.ldb = ldb;
  p.C = C; p.ldc = ldc;
  p.alpha = make_double2(alpha, 0.0);
  p.beta = make_double2(beta, 0.0);
  p.Y0 = Y0; p.ld0 = ld0; p.gamma = gamma;
  p.Y1e = Y1e; p.ld1e = ld1e;
  p.coef = coef_dev;
  return launch(h, OP_N, OP_N, EPI_FILTER, M, N, K, p);
}

int zgemm_filter_step(Handle* h, long long M, long long N, const double2* A, long long lda,
                      const double2* Y1, long long ld1, double alpha, double beta,
                      const double2* Y0, long long ld0, double gamma, double2* C, long long ldc,
                      const double* coef_dev, const SumPlanes* sp) {
  return zgemm_filter_panel(h, M, N, M, A, lda, Y1, ld1, Y1, ld1, alpha, beta, Y0, ld0, gamma, C,
                            ldc, coef_dev, sp);
}

size_t filter_step_workspace(Handle* h, long long M, long long N) {
  if (ensure_table() != OK) return 0;
  const Plan pl = cached_plan(h, OP_N, OP_N, EPI_FILTER, M, N, M, false);
  return pl.split > 1 ? (size_t)pl.split * M * N * sizeof(double2) : 0;
}

}  // namespace chfsi
