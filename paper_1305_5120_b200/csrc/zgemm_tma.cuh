// TMA + mbarrier pipelined complex128 DMMA GEMM for op(A) = op(B) = N (sm_100a).
//
// Same arithmetic and epilogues as zgemm.cuh (EPI_STORE / EPI_FILTER /
// EPI_PARTIAL), different data movement:
//   * operand tiles arrive by cp.async.bulk.tensor (TMA, SASS UTMALDG) into a
//     STAGES-deep ring, 128-byte swizzled, completion tracked by an mbarrier
//     transaction count (no LDGSTS address math in the consumer warps);
//   * stage reuse is released by per-warp mbarrier arrivals, so there is no
//     CTA-wide __syncthreads in the main loop; the refill of a stage is issued
//     by lane 0 of warp (kt mod 4), spreading the producer duty;
//   * 128B swizzle XORs the 16-byte chunk index with the 128-byte row index.
//     Reading fragment row r from tile row p(r) = (r>>1) | ((r&1)<<2) makes
//     every LDS.128 quarter-warp hit 8 distinct bank groups; the epilogue
//     applies the same permutation to output rows and columns.
//
// Layouts (complex = 16 B; "row" = 128 B):
//   A tile (column-major A, BM/8 boxes of {8 rows, BK cols}, box g at g*BK rows):
//     chunk(mg, k, m8) = (mg*BK + k)*8 + (m8 ^ (k & 7))
//   B tile (column-major B, box {BK rows, BN cols}):
//     chunk(n, k)      = n*8 + (k ^ (n & 7))               (BK == 8)
#pragma once

#include <cuda.h>

#include <type_traits>

#include "zgemm.cuh"

namespace chfsi {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ double2 lds128(unsigned addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

__device__ __forceinline__ double lds64(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ int perm8(int r) { return (r >> 1) | ((r & 1) << 2); }

// Stage refill lag: at k-tile kt the producer lane refills the stage of tile
// kt - kDefer (released by every warp kDefer iterations earlier).
#ifndef CHFSI_TMA_DEFER
#define CHFSI_TMA_DEFER 1
#endif
constexpr int kDefer = CHFSI_TMA_DEFER;

// operand-sum planes read by a 3M kernel: none (sums formed in the loop), both, B only
constexpr int SUMS_NONE = 0, SUMS_BOTH = 1, SUMS_B = 2;

// One k-tile sweep per stage: wait for the stage, run the BK/4 DMMA k-steps of the
// warp tile, release the stage, and (rotating producer lane) refill the stage that
// was released one iteration earlier.
// TAIL: 0 interior warp tile (every 8-column block live), 1 ragged (blocks >= jvalid are
// skipped), 2 ragged with a PACKED last live block (3M only): a block holding at most 4
// real columns is multiplied as the real 8-column operand [Re y_0..3 | Im y_0..3], two
// DMMAs per row group (Ar x, Ai x) instead of 3M's three -- the block of a 26-column
// shard that holds 2 columns costs 2/3 of a padded one (8 % of that shard's step).
template <int BM, int BN, int WM, int WN, int STAGES, int MUL, int SUMS, int TAIL, int JV, class Issue>
__device__ __forceinline__ void tma_mainloop(const double2* sA,
                                             const double2* sB, const double* sAs,
                                             const double* sBs, uint64_t* full, uint64_t* empty,
                                             Issue& issue, int KT, int wm, int wn, int lane,
                                             int warp, int fc, int pr, int jvalid,
                                             double (&c0)[WM / 8][WN / 8][2],
                                             double (&c1)[WM / 8][WN / 8][2],
                                             double (&c2)[WM / 8][WN / 8][2]) {
  constexpr int BK = 8;
  constexpr int NWARP = (BM / WM) * (BN / WN);
  constexpr int FM = WM / 8, FN = WN / 8;
  constexpr int A_ELEMS = BM * BK, B_ELEMS = BN * BK;
  constexpr bool RAGGED = TAIL != 0;
  // TAIL == 2: the live-block count is the compile-time JV (one instantiation per count),
  // so the packed block's operands are fixed registers, not run-time selects
  constexpr int jpack = (TAIL == 2) ? JV - 1 : -1;
  if (TAIL == 2) jvalid = JV;
  const int q = lane >> 2;
  // unrolled by the ring depth: the stage index, its smem addresses and barrier slots
  // become compile-time constants in each copy (ncu: DMMA pipe 95.5 -> 97.4 % for the
  // sum-plane filter kernel, 47.1 -> 48.2 TF/s at k = 2200)
  #pragma unroll 4
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % STAGES;
    const unsigned phase = (kt / STAGES) & 1;
    mbar_wait(&full[s], phase);
    // 32-bit shared-window addresses: LDS instead of generic loads (fewer address
    // registers, shorter load-to-use latency)
    const unsigned a = smem_u32(sA + s * A_ELEMS);
    const unsigned b = smem_u32(sB + s * B_ELEMS);
    const unsigned as_base = SUMS == SUMS_BOTH ? smem_u32(sAs + s * A_ELEMS) : 0u;
    const unsigned bs_base = SUMS != SUMS_NONE ? smem_u32(sBs + s * B_ELEMS) : 0u;
    #pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const int kk = ks * 4 + fc;
      double2 fa[FM], fb[FN];
      #pragma unroll
      for (int i = 0; i < FM; ++i) {
        const int mg = (wm * WM) / 8 + i;
        // smem [group][col][8 rows] (one 3-D box or BM/8 2-D boxes): 128-byte row index
        // mg * BK + kk, swizzle phase kk -- every quarter-warp reads 8 distinct 16-byte
        // bank groups
        fa[i] = lds128(a + 16u * ((mg * BK + kk) * 8 + (pr ^ kk)));
      }
      #pragma unroll
      for (int j = 0; j < FN; ++j) {
        if (TAIL == 2 && j == jpack) {
          // packed block: fragment column q <- Re (q < 4) or Im (q >= 4) of tile column q & 3
          const int nn = wn * WN + j * 8 + (q & 3);
          const double2 v = lds128(b + 16u * (nn * 8 + (kk ^ (q & 3))));
          fb[j].x = (q < 4) ? v.x : v.y;
          fb[j].y = 0.0;
        } else {
          const int nn = wn * WN + j * 8 + pr;
          fb[j] = lds128(b + 16u * (nn * 8 + (kk ^ pr)));
        }
      }
      if (MUL == 3) {
        // 3M: three real products per complex MAC. The operand sums cost FM + FN DADDs
        // per 3 FM FN DMMAs.
        double as[FM], bs[FN];
        if (SUMS == SUMS_BOTH) {
          // precomputed operand sums: As [group][col][8 rows] (64 B per group column,
          // rows permuted by column: sum_plane_grouped), conflict-free per half-warp
          #pragma unroll
          for (int i = 0; i < FM; ++i) {
            const int mg = (wm * WM) / 8 + i;
            as[i] = lds64(as_base + 8u * (mg * 64 + kk * 8 + (pr ^ (((kk >> 1) & 1) << 1))));
          }
        } else {
          #pragma unroll
          for (int i = 0; i < FM; ++i) as[i] = fa[i].x + fa[i].y;
        }
        if (SUMS != SUMS_NONE) {
          // Bs = {BK rows, BN cols} with 64-byte swizzle (conflict-free per half-warp)
          #pragma unroll
          for (int j = 0; j < FN; ++j) {
            const int nn = wn * WN + j * 8 + pr;
            const unsigned off = 64u * nn + 8u * kk;
            bs[j] = lds64(bs_base + (off ^ (((off >> 7) & 3u) << 4)));
          }
        } else {
          #pragma unroll
          for (int j = 0; j < FN; ++j) bs[j] = fb[j].x + fb[j].y;
        }
        #pragma unroll
        for (int i = 0; i < FM; ++i)
          #pragma unroll
          for (int j = 0; j < FN; ++j)
            if (!RAGGED || j < jvalid) {
              // (packed block: c0 = Ar [yr | yi], c1 = Ai [yr | yi])
              dmma884(c0[i][j][0], c0[i][j][1], fa[i].x, fb[j].x);
              dmma884(c1[i][j][0], c1[i][j][1], fa[i].y,
                      (TAIL == 2 && j == jpack) ? fb[j].x : fb[j].y);
            }
        #pragma unroll
        for (int i = 0; i < FM; ++i)
          #pragma unroll
          for (int j = 0; j < FN; ++j)
            if ((!RAGGED || j < jvalid) && !(TAIL == 2 && j == jpack))
              dmma884(c2[i][j][0], c2[i][j][1], as[i], bs[j]);
      } else {
        // two sweeps over the warp tile: the second update of each accumulator is
        // 2*FM*FN DMMAs after the first, so no DMMA waits on its predecessor
        #pragma unroll
        for (int i = 0; i < FM; ++i)
          #pragma unroll
          for (int j = 0; j < FN; ++j)
            if (!RAGGED || j < jvalid) {
              dmma884(c0[i][j][0], c0[i][j][1], fa[i].x, fb[j].x);
              dmma884(c1[i][j][0], c1[i][j][1], fa[i].x, fb[j].y);
            }
        #pragma unroll
        for (int i = 0; i < FM; ++i) {
          const double nai = -fa[i].y;
          #pragma unroll
          for (int j = 0; j < FN; ++j)
            if (!RAGGED || j < jvalid) {
              dmma884(c0[i][j][0], c0[i][j][1], nai, fb[j].y);
              dmma884(c1[i][j][0], c1[i][j][1], fa[i].y, fb[j].x);
            }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    // refill the stage released one iteration ago with tile kt - 1 + STAGES: by now
    // every warp has normally finished tile kt - 1, so this empty-barrier wait is
    // almost always already complete and the producer lane does not stall its warp
    // (waiting on the just-released stage cost ~8 % of warp samples, profiles/r01)
    if (lane == 0 && kt >= kDefer && warp == (kt % NWARP) && kt - kDefer + STAGES < KT) {
      mbar_wait(&empty[(kt - kDefer) % STAGES], ((kt - kDefer) / STAGES) & 1);
      issue(kt - kDefer + STAGES);
    }
  }
}

template <int BM, int BN, int WM, int WN, int STAGES, int SUMS = SUMS_NONE>
constexpr int zgemm_tma_smem_bytes() {
  return STAGES * (BM * 8 * (SUMS == SUMS_BOTH ? 24 : 16) + BN * 8 * (SUMS != SUMS_NONE ? 24 : 16)) +
         1024 /* alignment slack */ + 2 * STAGES * 8;
}

// MUL = 4: four real products per complex MAC; MUL = 3: 3M. SUMS (3M only): the operand
// sums Ar + Ai and Br + Bi arrive precomputed as real planes (p.As, p.Bs; maps mapAs,
// mapBs), so the main loop issues no DADDs (an in-loop DADD stalls the DMMA stream:
// ncu, DMMA pipe 88.6 % active with in-loop sums vs 95.8 % without). SUMS_B: only the
// B plane is read (8 bytes per element of the narrow block); Ar + Ai is formed in the
// loop, FM DADDs per 3 FM FN DMMAs, so H streams at 16 instead of 24 bytes per element:
// the plan for narrow blocks, where the sum-plane kernel runs at the board's power cap.
template <int BM, int BN, int WM, int WN, int STAGES, int EPI, int MINB = 1, int MUL = 4,
          int SUMS = SUMS_NONE>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32, MINB)
zgemm_tma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                 const __grid_constant__ CUtensorMap mapAs,
                 const __grid_constant__ CUtensorMap mapBs, const GemmParams p) {
  static_assert(SUMS == SUMS_NONE || MUL == 3, "operand sums are a 3M feature");
  // packed tail blocks: the narrow-block kernels (B-sum plane only). Measured A/B on one
  // B200, sustained degree-25 calls at n = 20000: k = 26 2.303 -> 2.184 ms, k = 51 4.10 ->
  // 4.03 ms; in the both-plane kernels (k = 201, 210) it was -1 % / +0.4 % at the power
  // cap, so they keep the plain ragged path.
  constexpr bool PACK_TAIL = (MUL == 3 && SUMS == SUMS_B);
  constexpr int BK = 8;
  constexpr int NWM = BM / WM;
  constexpr int NWARP = NWM * (BN / WN);
  constexpr int FM = WM / 8, FN = WN / 8;
  constexpr int A_ELEMS = BM * BK, B_ELEMS = BN * BK;
  constexpr unsigned STAGE_BYTES = A_ELEMS * (SUMS == SUMS_BOTH ? 24 : 16) +
                                   B_ELEMS * (SUMS != SUMS_NONE ? 24 : 16);
  static_assert((A_ELEMS * 16) % 1024 == 0 && (B_ELEMS * 16) % 1024 == 0, "1 KB aligned tiles");

  extern __shared__ unsigned char smem_raw[];
  double2* base = reinterpret_cast<double2*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  double2* sA = base;
  double2* sB = base + STAGES * A_ELEMS;
  double* sAs = reinterpret_cast<double*>(sB + STAGES * B_ELEMS);  // SUMS_BOTH only
  double* sBs = sAs + (SUMS == SUMS_BOTH ? STAGES * A_ELEMS : 0);   // SUMS_BOTH / SUMS_B
  uint64_t* full = reinterpret_cast<uint64_t*>(
      SUMS != SUMS_NONE ? reinterpret_cast<void*>(sBs + STAGES * B_ELEMS)
                        : reinterpret_cast<void*>(sAs));
  uint64_t* empty = full + STAGES;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % NWM, wn = warp / NWM;
  int mi, ni;
  tile_coords(p, blockIdx.x, mi, ni);
  const int m0 = mi * BM;
  // column tile [n0, nend): BN wide, or (mixed tiling, GemmParams::n_wide) BN - 8 wide
  // after the first n_wide tiles
  // (only the kernels whose warps span the tile's columns compile it: a narrower tile
  // keeps the same live blocks in every warp)
  int n0 = ni * BN, nend = p.N;
  if constexpr (WN == BN && BN == 32) {
    if (p.n_wide > 0) {
      n0 = (ni < p.n_wide) ? ni * BN : p.n_wide * BN + (ni - p.n_wide) * (BN - 8);
      nend = min(p.N, n0 + ((ni < p.n_wide) ? BN : BN - 8));
    }
  }
  if ((p.tri & TRI_C_LOWER) && m0 + BM <= n0) return;  // strictly upper tile (CTA-uniform)
  int kbeg = 0, kend = p.K;
  if (EPI == EPI_PARTIAL) {
    kbeg = blockIdx.z * p.k_chunk;
    kend = min(p.K, kbeg + p.k_chunk);
  }
  tri_krange(p, m0, n0, BM, BN, kbeg, kend);
  const int KT = (kend > kbeg) ? (kend - kbeg + BK - 1) / BK : 0;

  if (tid == 0) {
    #pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWARP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
    if (SUMS == SUMS_BOTH)
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mapAs)) : "memory");
    if (SUMS != SUMS_NONE)
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mapBs)) : "memory");
  }
  __syncthreads();

  auto issue = [&](int kt) {
    const int s = kt % STAGES;
    const int k0 = kbeg + kt * BK;
    mbar_expect_tx(&full[s], STAGE_BYTES);
    // A: one {8 rows x BK cols} box per 8-row group (coords in doubles, columns);
    // B: one {BK rows x BN cols} box. Out-of-range rows/cols arrive zero-filled.
    if (SUMS != SUMS_NONE) {
      // four boxes per stage: A {16 doubles, BK cols, BM/8 groups} (M % 8 == 0), B, the
      // grouped A-sum plane {8 rows, BK cols, BM/8 groups} and the B-sum plane (SUMS_B:
      // three, no A-sum plane)
      tma_load_3d(sA + s * A_ELEMS, &mapA, 0, k0, m0 / 8, &full[s]);
      tma_load_2d(sB + s * B_ELEMS, &mapB, 2 * k0, n0, &full[s]);
      if (SUMS == SUMS_BOTH) tma_load_3d(sAs + s * A_ELEMS, &mapAs, 0, k0, m0 / 8, &full[s]);
      tma_load_2d(sBs + s * B_ELEMS, &mapBs, k0, n0, &full[s]);
    } else {
      // A: one 3-D box when M % 8 == 0 (p.a3d, same smem layout), else BM/8 2-D boxes
      if (p.a3d) {
        tma_load_3d(sA + s * A_ELEMS, &mapA, 0, k0, m0 / 8, &full[s]);
      } else {
        #pragma unroll
        for (int g = 0; g < BM / 8; ++g)
          tma_load_2d(sA + s * A_ELEMS + g * BK * 8, &mapA, 2 * (m0 + 8 * g), k0, &full[s]);
      }
      tma_load_2d(sB + s * B_ELEMS, &mapB, 2 * k0, n0, &full[s]);
    }
  };

  if (tid == 0) {
    #pragma unroll
    for (int s = 0; s < STAGES; ++s)
      if (s < KT) issue(s);
  }

  const int fc = lane & 3;
  const int pr = perm8(lane >> 2);
  // 8-column MMA blocks of this warp that hold at least one real column: blocks
  // entirely past N (the padded tail of a narrow filter block) issue no DMMAs.
  // Warp-uniform, so DMMA's warp-collective semantics are kept.
  const int jvalid = min(FN, max(0, (nend - (n0 + wn * WN) + 7) / 8));
  // MUL == 4: c0 = Re, c1 = Im, four real products per complex MAC.
  // MUL == 3: c0 = Ar Br, c1 = Ai Bi, c2 = (Ar + Ai)(Br + Bi) (3M); the epilogue forms
  // Re = c0 - c1, Im = c2 - c0 - c1.
  double c0[FM][FN][2], c1[FM][FN][2], c2[FM][FN][2];
  #pragma unroll
  for (int i = 0; i < FM; ++i)
    #pragma unroll
    for (int j = 0; j < FN; ++j)
      #pragma unroll
      for (int t = 0; t < 2; ++t) c0[i][j][t] = c1[i][j][t] = c2[i][j][t] = 0.0;

  // 3M narrow-block kernels: a last live block with at most 4 real columns is packed
  // (TAIL = 2 above); warp-uniform
  int jpack = -1;
  if constexpr (PACK_TAIL) {
    const int last_cols = nend - (n0 + wn * WN + (jvalid - 1) * 8);  // of block jvalid - 1
    if (p.pack && jvalid >= 1 && last_cols <= 4) jpack = jvalid - 1;
  }
  if (jpack >= 0) {
    if constexpr (PACK_TAIL) {
      // one main-loop instantiation per live-block count: the packed block's operands are
      // fixed registers
      auto run = [&](auto jv) {
        tma_mainloop<BM, BN, WM, WN, STAGES, MUL, SUMS, 2, decltype(jv)::value>(
            sA, sB, sAs, sBs, full, empty, issue, KT, wm, wn, lane, warp, fc, pr, jvalid, c0, c1,
            c2);
      };
      if (FN >= 4 && jvalid == 4) run(std::integral_constant<int, (FN >= 4 ? 4 : 1)>{});
      else if (FN >= 3 && jvalid == 3) run(std::integral_constant<int, (FN >= 3 ? 3 : 1)>{});
      else if (FN >= 2 && jvalid == 2) run(std::integral_constant<int, (FN >= 2 ? 2 : 1)>{});
      else run(std::integral_constant<int, 1>{});
      // fragment columns 0-3 hold the products with Re y, 4-7 with Im y: lanes fc < 2 take
      // the other half from lane ^ 2 and form Re = Ar yr - Ai yi, Im = Ar yi + Ai yr
      #pragma unroll
      for (int i = 0; i < FM; ++i)
        #pragma unroll
        for (int j = 0; j < FN; ++j)
          if (j == jpack) {
            #pragma unroll
            for (int t = 0; t < 2; ++t) {
              const double o1 = __shfl_xor_sync(0xffffffffu, c0[i][j][t], 2);
              const double o2 = __shfl_xor_sync(0xffffffffu, c1[i][j][t], 2);
              const double re = __dsub_rn(c0[i][j][t], o2);
              const double im = __dadd_rn(o1, c1[i][j][t]);
              c0[i][j][t] = re;
              c1[i][j][t] = im;
            }
          }
    }
  } else if (jvalid == FN) {  // interior warp tile: unconditional DMMA stream
    tma_mainloop<BM, BN, WM, WN, STAGES, MUL, SUMS, 0, 0>(sA, sB, sAs, sBs, full, empty, issue, KT, wm, wn,
                                                    lane, warp, fc, pr, jvalid, c0, c1, c2);
  } else {  // ragged column edge: skip 8-column blocks past N
    tma_mainloop<BM, BN, WM, WN, STAGES, MUL, SUMS, 1, 0>(sA, sB, sAs, sBs, full, empty, issue, KT, wm, wn,
                                                   lane, warp, fc, pr, jvalid, c0, c1, c2);
  }

  // epilogue: fragment row r <-> tile row perm8(r); fragment column c <-> perm8(c)
  #pragma unroll
  for (int i = 0; i < FM; ++i) {
    const int m = m0 + wm * WM + i * 8 + pr;
    if (m >= p.M) continue;
    #pragma unroll
    for (int j = 0; j < FN; ++j) {
      #pragma unroll
      for (int t = 0; t < 2; ++t) {
        const bool pk = (j == jpack);  // packed block: columns in fragment order, fc < 2
        const int n = n0 + wn * WN + j * 8 + (pk ? fc * 2 + t : perm8(fc * 2 + t));
        if (n >= nend || (pk && fc >= 2)) continue;
        // explicit roundings (no contraction choices left to the compiler): every
        // instantiation -- tile shape, sum planes or not -- rounds the same way, so a
        // product is bit-identical whichever config the planner picks without split-K
        // (a packed tail block is a four-product result: same inputs, its own rounding)
        double xr, xi;
        if (pk) {
          xr = c0[i][j][t];
          xi = c1[i][j][t];
        } else if (MUL == 3) {
          xr = __dsub_rn(c0[i][j][t], c1[i][j][t]);
          xi = __dsub_rn(__dsub_rn(c2[i][j][t], c0[i][j][t]), c1[i][j][t]);
        } else {
          xr = c0[i][j][t];
          xi = c1[i][j][t];
        }
        if (EPI == EPI_PARTIAL) {
          p.ws[(long long)blockIdx.z * p.M * p.N + m + (long long)n * p.M] = make_double2(xr, xi);
        } else if (EPI == EPI_FILTER) {
          double fa, fb, fg;
          filter_coef(p, fa, fb, fg);
          const double2 y1 = p.Y1e[m + (long long)n * p.ld1e];
          double orr = __fma_rn(fa, xr, __dmul_rn(fb, y1.x));
          double oi = __fma_rn(fa, xi, __dmul_rn(fb, y1.y));
          if (p.Y0 != nullptr) {
            const double2 y0 = p.Y0[m + (long long)n * p.ld0];
            orr = __fma_rn(fg, y0.x, orr);
            oi = __fma_rn(fg, y0.y, oi);
          }
          p.C[m + (long long)n * p.ldc] = make_double2(orr, oi);
          if (p.Cs != nullptr) p.Cs[m + (long long)n * p.ldcs] = __dadd_rn(orr, oi);
        } else {
          double2 o = make_double2(p.alpha.x * xr - p.alpha.y * xi, p.alpha.x * xi + p.alpha.y * xr);
          if (p.beta.x != 0.0 || p.beta.y != 0.0) {
            const double2 c = p.C[m + (long long)n * p.ldc];
            o.x += p.beta.x * c.x - p.beta.y * c.y;
            o.y += p.beta.x * c.y + p.beta.y * c.x;
          }
          p.C[m + (long long)n * p.ldc] = o;
          if (p.Cs != nullptr) p.Cs[m + (long long)n * p.ldcs] = __dadd_rn(o.x, o.y);
        }
      }
    }
  }
}

}  // namespace chfsi
