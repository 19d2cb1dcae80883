// Bandwidth-bound helper kernels of the ChFSI path (HBM roofline):
// residual norms (core.py:347-358, :477), column dots (Lanczos, core.py:230-238),
// Hermitian check + symmetrisation (linalg.py:104-121), Cholesky-factor
// cleanup (linalg.py:262-270) and the blocked triangular inverse used for
// CholQR and the generalized reduction (linalg.py:326-366).
//
// All reductions use a fixed tree (block_sum) and fixed partial order: no
// atomics, so repeated runs are bit-identical.
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace chfsi {

namespace {

constexpr int RT = 256;

__global__ void residual_norms_kernel(long long n, const double2* __restrict__ HY, long long ldhy,
                                      const double2* __restrict__ Y, long long ldy,
                                      const double* __restrict__ lam, double* __restrict__ res) {
  __shared__ double red[RT / 32];
  const long long j = blockIdx.x;
  const double l = lam[j];
  const double2* hy = HY + j * ldhy;
  const double2* y = Y + j * ldy;
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += RT) {
    const double2 a = hy[i], b = y[i];
    const double rr = a.x - l * b.x, ri = a.y - l * b.y;
    s += rr * rr + ri * ri;
  }
  s = block_sum<RT>(s, red);
  if (threadIdx.x == 0) res[j] = sqrt(s);
}

__global__ void zdotc_cols_kernel(long long n, const double2* __restrict__ X, long long ldx,
                                  const double2* __restrict__ Y, long long ldy,
                                  double2* __restrict__ out) {
  __shared__ double red[RT / 32];
  const long long j = blockIdx.x;
  const double2* x = X + j * ldx;
  const double2* y = Y + j * ldy;
  double sr = 0.0, si = 0.0;
  for (long long i = threadIdx.x; i < n; i += RT) {
    const double2 a = x[i], b = y[i];
    sr += a.x * b.x + a.y * b.y;
    si += a.x * b.y - a.y * b.x;
  }
  sr = block_sum<RT>(sr, red);
  si = block_sum<RT>(si, red);
  if (threadIdx.x == 0) out[j] = make_double2(sr, si);
}

// Narrow blocks (the tail of a solve: k ~ 200 columns) give one CTA per column too few
// CTAs to saturate HBM, so columns are split into S row chunks; partial sums land in
// partial[j*S + s] and a second kernel adds them in fixed s order (deterministic).
__global__ void residual_partial_kernel(long long n, int S, const double2* __restrict__ HY,
                                        long long ldhy, const double2* __restrict__ Y,
                                        long long ldy, const double* __restrict__ lam,
                                        double* __restrict__ partial) {
  __shared__ double red[RT / 32];
  const long long j = blockIdx.x;
  const int s = blockIdx.y;
  const long long chunk = (n + S - 1) / S;
  const long long i0 = s * chunk, i1 = min(n, i0 + chunk);
  const double l = lam[j];
  const double2* hy = HY + j * ldhy;
  const double2* y = Y + j * ldy;
  double acc = 0.0;
  for (long long i = i0 + threadIdx.x; i < i1; i += RT) {
    const double2 a = hy[i], b = y[i];
    const double rr = a.x - l * b.x, ri = a.y - l * b.y;
    acc += rr * rr + ri * ri;
  }
  acc = block_sum<RT>(acc, red);
  if (threadIdx.x == 0) partial[j * S + s] = acc;
}

__global__ void zdotc_partial_kernel(long long n, int S, const double2* __restrict__ X,
                                     long long ldx, const double2* __restrict__ Y, long long ldy,
                                     double2* __restrict__ partial) {
  __shared__ double red[RT / 32];
  const long long j = blockIdx.x;
  const int s = blockIdx.y;
  const long long chunk = (n + S - 1) / S;
  const long long i0 = s * chunk, i1 = min(n, i0 + chunk);
  const double2* x = X + j * ldx;
  const double2* y = Y + j * ldy;
  double sr = 0.0, si = 0.0;
  for (long long i = i0 + threadIdx.x; i < i1; i += RT) {
    const double2 a = x[i], b = y[i];
    sr += a.x * b.x + a.y * b.y;
    si += a.x * b.y - a.y * b.x;
  }
  sr = block_sum<RT>(sr, red);
  si = block_sum<RT>(si, red);
  if (threadIdx.x == 0) partial[j * S + s] = make_double2(sr, si);
}

// GEMV y = alpha A x + beta y, A column-major M x K (the Lanczos H v, core.py:202-256):
// HBM-bound (16 bytes of A per complex MAC). Thread r of the grid owns row r, so each
// column of A is read by consecutive threads (coalesced 512-byte warp segments) with
// streaming loads (A is read once); every thread keeps GV_U independent loads in
// flight. The K columns are split over blockIdx.y (S chunks) so the grid holds
// enough loads in flight to saturate HBM even for one column; the S partial rows are
// summed in fixed order by zgemv_finish_kernel (deterministic, no atomics).
constexpr int GV_T = 256;
constexpr int GV_U = 8;

__global__ void __launch_bounds__(GV_T) zgemv_partial_kernel(long long M, long long K, int S,
                                                             const double2* __restrict__ A,
                                                             long long lda,
                                                             const double2* __restrict__ x,
                                                             double2* __restrict__ partial) {
  const long long r = (long long)blockIdx.x * GV_T + threadIdx.x;
  const int s = blockIdx.y;
  const long long chunk = (K + S - 1) / S;
  const long long c0 = s * chunk, c1 = min(K, c0 + chunk);
  if (r >= M) return;
  const double2* a = A + r;
  double ar = 0.0, ai = 0.0;
  long long c = c0;
  for (; c + GV_U <= c1; c += GV_U) {
    double2 hv[GV_U];
    #pragma unroll
    for (int u = 0; u < GV_U; ++u) hv[u] = __ldcs(a + (c + u) * lda);
    #pragma unroll
    for (int u = 0; u < GV_U; ++u) {
      const double2 xv = __ldg(x + c + u);
      ar = fma(hv[u].x, xv.x, ar);
      ar = fma(-hv[u].y, xv.y, ar);
      ai = fma(hv[u].x, xv.y, ai);
      ai = fma(hv[u].y, xv.x, ai);
    }
  }
  for (; c < c1; ++c) {
    const double2 hv = __ldcs(a + c * lda);
    const double2 xv = __ldg(x + c);
    ar = fma(hv.x, xv.x, ar);
    ar = fma(-hv.y, xv.y, ar);
    ai = fma(hv.x, xv.y, ai);
    ai = fma(hv.y, xv.x, ai);
  }
  partial[(long long)s * M + r] = make_double2(ar, ai);
}

__global__ void zgemv_finish_kernel(long long M, int S, const double2* __restrict__ partial,
                                    double2 alpha, double2 beta, double2* __restrict__ y) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= M) return;
  double sr = 0.0, si = 0.0;
  for (int t = 0; t < S; ++t) {
    const double2 p = partial[(long long)t * M + r];
    sr += p.x;
    si += p.y;
  }
  double2 out = make_double2(alpha.x * sr - alpha.y * si, alpha.x * si + alpha.y * sr);
  if (beta.x != 0.0 || beta.y != 0.0) {
    const double2 o = y[r];
    out.x += beta.x * o.x - beta.y * o.y;
    out.y += beta.x * o.y + beta.y * o.x;
  }
  y[r] = out;
}

__global__ void finish_sqrt_kernel(long long k, int S, const double* __restrict__ partial,
                                   double* __restrict__ out) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= k) return;
  double s = 0.0;
  for (int t = 0; t < S; ++t) s += partial[j * S + t];
  out[j] = sqrt(s);
}

__global__ void finish_sum2_kernel(long long k, int S, const double2* __restrict__ partial,
                                   double2* __restrict__ out) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= k) return;
  double sr = 0.0, si = 0.0;
  for (int t = 0; t < S; ++t) {
    sr += partial[j * S + t].x;
    si += partial[j * S + t].y;
  }
  out[j] = make_double2(sr, si);
}

// row chunks per column so that k * S CTAs cover >= ~8 CTAs per SM (1 when k is wide)
inline int column_splits(long long n, long long k) {
  const long long want = 148LL * 8;
  if (k >= want) return 1;
  long long s = (want + k - 1) / k;
  s = std::min<long long>(s, std::max<long long>(1, n / 2048));  // >= 2048 rows per chunk
  return (int)std::max<long long>(1, std::min<long long>(s, 64));
}

constexpr int TS = 32;  // tile for transpose-type kernels

// partials[2*(by*gx+bx)+{0,1}] = (sum |A_ij|^2, sum |A_ij - conj(A_ji)|^2) over tile (bx,by)
__global__ void hermitian_norms_kernel(long long n, const double2* __restrict__ A, long long lda,
                                       double* __restrict__ partials) {
  __shared__ double2 t[TS][TS + 1];
  __shared__ double red[8];
  const long long c0 = (long long)blockIdx.x * TS, r0 = (long long)blockIdx.y * TS;
  const int tx = threadIdx.x % TS, ty = threadIdx.x / TS;  // 32 x 8 threads
  // load transposed source tile A[c0.., r0..] -> t[col][row]
  for (int yy = ty; yy < TS; yy += 8) {
    const long long r = c0 + tx, c = r0 + yy;  // element A[r, c] with r in tile cols
    t[yy][tx] = (r < n && c < n) ? A[r + c * lda] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  double s_all = 0.0, s_dev = 0.0;
  for (int yy = ty; yy < TS; yy += 8) {
    const long long r = r0 + tx, c = c0 + yy;  // element A[r, c]
    if (r < n && c < n) {
      const double2 a = A[r + c * lda];
      const double2 b = t[tx][yy];  // A[c, r]
      s_all += a.x * a.x + a.y * a.y;
      const double dr = a.x - b.x, di = a.y + b.y;
      s_dev += dr * dr + di * di;
    }
  }
  s_all = block_sum<256>(s_all, red);
  s_dev = block_sum<256>(s_dev, red);
  if (threadIdx.x == 0) {
    const long long b = (long long)blockIdx.y * gridDim.x + blockIdx.x;
    partials[2 * b] = s_all;
    partials[2 * b + 1] = s_dev;
  }
}

__global__ void sum_pairs_kernel(long long count, const double* __restrict__ partials,
                                 double* __restrict__ out) {
  __shared__ double red[8];
  double a = 0.0, d = 0.0;
  for (long long i = threadIdx.x; i < count; i += 256) {
    a += partials[2 * i];
    d += partials[2 * i + 1];
  }
  a = block_sum<256>(a, red);
  d = block_sum<256>(d, red);
  if (threadIdx.x == 0) {
    out[0] = a;
    out[1] = d;
  }
}

// A <- (A + A^H)/2 with a real diagonal, in place; CTA (bx, by) with bx >= by owns
// the tile pair {(by,bx), (bx,by)}.
__global__ void hermitize_kernel(long long n, double2* A, long long lda) {
  if (blockIdx.x < blockIdx.y) return;
  __shared__ double2 up[TS][TS + 1], lo[TS][TS + 1];
  const long long r0 = (long long)blockIdx.y * TS, c0 = (long long)blockIdx.x * TS;
  const int tx = threadIdx.x % TS, ty = threadIdx.x / TS;
  for (int yy = ty; yy < TS; yy += 8) {
    long long r = r0 + tx, c = c0 + yy;  // tile (r0, c0): up[yy][tx] = A[r, c]
    up[yy][tx] = (r < n && c < n) ? A[r + c * lda] : make_double2(0.0, 0.0);
    r = c0 + tx; c = r0 + yy;            // tile (c0, r0): lo[yy][tx] = A[r, c]
    lo[yy][tx] = (r < n && c < n) ? A[r + c * lda] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int yy = ty; yy < TS; yy += 8) {
    // element A[r0+tx, c0+yy] pairs with A[c0+yy, r0+tx] = lo[tx][yy]
    long long r = r0 + tx, c = c0 + yy;
    if (r < n && c < n) {
      const double2 a = up[yy][tx], b = lo[tx][yy];
      double2 o = make_double2((a.x + b.x) / 2.0, (a.y - b.y) / 2.0);
      if (r == c) o.y = 0.0;
      A[r + c * lda] = o;
    }
    r = c0 + tx; c = r0 + yy;
    if (blockIdx.x != blockIdx.y && r < n && c < n) {
      const double2 a = lo[yy][tx], b = up[tx][yy];
      const double2 o = make_double2((a.x + b.x) / 2.0, (a.y - b.y) / 2.0);
      A[r + c * lda] = o;
    }
  }
}

// zero the strict upper triangle, force a real diagonal (zpotrf clean=1 semantics)
__global__ void clean_lower_kernel(long long n, double2* L, long long ldl) {
  const long long total = n * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long i = idx % n, j = idx / n;
    if (i < j) L[i + j * ldl] = make_double2(0.0, 0.0);
    else if (i == j) L[i + j * ldl].y = 0.0;
  }
}

__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  // a / b, scaled to avoid overflow
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, d = b.x + r * b.y;
    return make_double2((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  }
  const double r = b.x / b.y, d = b.y + r * b.x;
  return make_double2((a.x * r + a.y) / d, (a.y * r - a.x) / d);
}

// Inverse of a lower-triangular nb x nb block (nb <= TRI_BASE): CTA j computes
// column j of X = L^-1 by column-oriented forward substitution.
constexpr int TRI_BASE = 256;
__global__ void __launch_bounds__(TRI_BASE) trtri_base_kernel(int nb, const double2* __restrict__ L,
                                                              long long ldl, double2* X,
                                                              long long ldx) {
  __shared__ double2 xs[2];
  const int j = blockIdx.x, r = threadIdx.x;
  double2 x = make_double2(r == j ? 1.0 : 0.0, 0.0);
  for (int i = j; i < nb; ++i) {
    if (r == i) {
      x = cdiv(x, L[i + (long long)i * ldl]);
      xs[i & 1] = x;
    }
    __syncthreads();
    const double2 xi = xs[i & 1];
    if (r > i && r < nb) {
      const double2 l = L[r + (long long)i * ldl];
      x.x -= xi.x * l.x - xi.y * l.y;
      x.y -= xi.x * l.y + xi.y * l.x;
    }
  }
  if (r < nb) X[r + (long long)j * ldx] = (r >= j) ? x : make_double2(0.0, 0.0);
}

__global__ void zaxpby_kernel(long long n, long long k, double2 alpha, const double2* X,
                              long long ldx, double2 beta, double2* Y, long long ldy) {
  const long long total = n * k;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long i = idx % n, j = idx / n;
    double2 y = Y[i + j * ldy];
    double2 o = make_double2(beta.x * y.x - beta.y * y.y, beta.x * y.y + beta.y * y.x);
    if (X != nullptr) {
      const double2 x = X[i + j * ldx];
      o.x += alpha.x * x.x - alpha.y * x.y;
      o.y += alpha.x * x.y + alpha.y * x.x;
    }
    Y[i + j * ldy] = o;
  }
}

// 3M operand-sum plane Xs = Re X + Im X (HBM-bound: 16 B read + 8 B written per entry).
__global__ void sum_plane_kernel(long long rows, long long cols, const double2* __restrict__ X,
                                 long long ldx, double* __restrict__ Xs, long long ldxs) {
  for (long long j = blockIdx.y; j < cols; j += gridDim.y) {
    const double2* x = X + j * ldx;
    double* xs = Xs + j * ldxs;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows;
         i += (long long)gridDim.x * blockDim.x) {
      const double2 v = x[i];
      xs[i] = __dadd_rn(v.x, v.y);
    }
  }
}

// The same plane in the grouped layout of an A operand (rows % 8 == 0): one 8-row group
// of every column is a contiguous 64-byte run, Xs[(i / 8) * 8 cols + j * 8 + p], with the
// row position p = (i % 8) ^ (2 * ((j / 2) % 2)) so that the fragment reads of a half-warp
// (4 rows x 4 columns) fall in 16 distinct 8-byte bank pairs (unpermuted, columns j and
// j + 2 collide: 2-way conflicts).
__global__ void sum_plane_grouped_kernel(long long rows, long long cols,
                                         const double2* __restrict__ X, long long ldx,
                                         double* __restrict__ Xs) {
  for (long long j = blockIdx.y; j < cols; j += gridDim.y) {
    const double2* x = X + j * ldx;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows;
         i += (long long)gridDim.x * blockDim.x) {
      const double2 v = x[i];
      Xs[(i >> 3) * 8 * cols + j * 8 + ((i & 7) ^ (((j >> 1) & 1) << 1))] = __dadd_rn(v.x, v.y);
    }
  }
}

__global__ void real_diag_kernel(long long n, const double2* A, long long lda, double* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = A[i + i * lda].x;
}

__global__ void shift_diag_kernel(long long n, double2* A, long long lda, double s) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    A[i + i * lda].x += s;
}

inline int grid_for(long long total, int threads = 256) {
  return (int)std::max<long long>(1, std::min<long long>((total + threads - 1) / threads, 148LL * 32));
}

}  // namespace

int residual_norms(Handle* h, long long n, long long k, const double2* HY, long long ldhy,
                   const double2* Y, long long ldy, const double* lam_dev, double* res_dev) {
  if (k <= 0) return OK;
  const int S = column_splits(n, k);
  if (S == 1) {
    residual_norms_kernel<<<(unsigned)k, RT, 0, h->stream>>>(n, HY, ldhy, Y, ldy, lam_dev,
                                                             res_dev);
    h->launches++;
    CHFSI_CHECK_LAUNCH();
    return OK;
  }
  double* part = (double*)scratch(h, SLOT_COLRED, (size_t)k * S * sizeof(double));
  if (!part) return ERR_NOMEM;
  residual_partial_kernel<<<dim3((unsigned)k, (unsigned)S), RT, 0, h->stream>>>(
      n, S, HY, ldhy, Y, ldy, lam_dev, part);
  finish_sqrt_kernel<<<(unsigned)((k + 255) / 256), 256, 0, h->stream>>>(k, S, part, res_dev);
  h->launches += 2;
  CHFSI_CHECK_LAUNCH();
  return OK;
}

int zdotc_cols(Handle* h, long long n, long long k, const double2* X, long long ldx,
               const double2* Y, long long ldy, double2* out_dev) {
  if (k <= 0) return OK;
  const int S = column_splits(n, k);
  if (S == 1) {
    zdotc_cols_kernel<<<(unsigned)k, RT, 0, h->stream>>>(n, X, ldx, Y, ldy, out_dev);
    h->launches++;
    CHFSI_CHECK_LAUNCH();
    return OK;
  }
  double2* part = (double2*)scratch(h, SLOT_COLRED, (size_t)k * S * sizeof(double2));
  if (!part) return ERR_NOMEM;
  zdotc_partial_kernel<<<dim3((unsigned)k, (unsigned)S), RT, 0, h->stream>>>(n, S, X, ldx, Y,
                                                                           ldy, part);
  finish_sum2_kernel<<<(unsigned)((k + 255) / 256), 256, 0, h->stream>>>(k, S, part, out_dev);
  h->launches += 2;
  CHFSI_CHECK_LAUNCH();
  return OK;
}

int hermitian_norms(Handle* h, long long n, const double2* A, long long lda, double* out2_dev) {
  const long long t = (n + TS - 1) / TS;
  double* partials = (double*)scratch(h, SLOT_TRI, (size_t)(2 * t * t) * sizeof(double));
  if (!partials) return ERR_NOMEM;
  dim3 grid((unsigned)t, (unsigned)t);
  hermitian_norms_kernel<<<grid, 256, 0, h->stream>>>(n, A, lda, partials);
  h->launches++;
  CHFSI_CHECK_LAUNCH();
  sum_pairs_kernel<<<1, 256, 0, h->stream>>>(t * t, partials, out2_dev);
  h->launches++;
  CHFSI_CHECK_LAUNCH();
  return OK;
}

int hermitize(Handle* h, long long n, double2* A, long long lda) {
  const long long t = (n + TS - 1) / TS;
  dim3 grid((unsigned)t, (unsigned)t);
  hermitize_kernel<<<grid, 256, 0, h->stream>>>(n, A, lda);
  h->launches++;
  CHFSI_CHECK_LAUNCH();
  return OK;
}

// Upper triangle <- conj(lower), real diagonal: completes a Hermitian matrix of which
// only the lower triangle was computed (zgemm TRI_C_LOWER). Tile (r0, c0) above the
// diagonal is filled from the transposed lower tile through shared memory.
__global__ void mirror_lower_kernel(long long n, double2* A, long long lda) {
  if (blockIdx.x < blockIdx.y) return;
  __shared__ double2 lo[TS][TS + 1];
  const long long r0 = (long long)blockIdx.y * TS, c0 = (long long)blockIdx.x * TS;
  const int tx = threadIdx.x % TS, ty = threadIdx.x / TS;
  for (int yy = ty; yy < TS; yy += 8) {
    const long long r = c0 + tx, c = r0 + yy;  // lo[yy][tx] = A[c0 + tx, r0 + yy]
    lo[yy][tx] = (r < n && c < n) ? A[r + c * lda] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int yy = ty; yy < TS; yy += 8) {
    const long long r = r0 + tx, c = c0 + yy;  // A[r, c] = conj(A[c, r]) = conj(lo[tx][yy])
    if (r >= n || c >= n) continue;
    if (r < c) {
      const double2 v = lo[tx][yy];
      A[r + c * lda] = make_double2(v.x, -v.y);
    } else if (r == c) {
      A[r + c * lda].y = 0.0;
    }
  }
}

int mirror_lower(Handle* h, long long n, double2* A, long long lda) {
  if (n <= 0) return OK;
  const long long t = (n + TS - 1) / TS;
  mirror_lower_kernel<<<dim3((unsigned)t, (unsigned)t), 256, 0, h->stream>>>(n, A, lda);
  h->launches++;
  CHFSI_CHECK_LAUNCH();
  return OK;
}

int clean_lower_factor(Handle* h, long long n, double2* L, long long ldl) {
  clean_lower_kernel<<<grid_for(n * n), 256, 0, h->stream>>>(n, L, ldl);
  h->launches++;
  CHFSI_CHECK_LAUNCH();
  return OK;
}

// Recursive blocked inverse: [[L11,0],[L21,L22]]^-1 = [[X11,0],[-X22 L21 X11, X22]].
static int trtri_rec(Handle* h, long long n, const double2* L, long long ldl, double2* X,
                     long long ldx, double2* tmp) {
  if (n <= TRI_BASE) {
    trtri_base_kernel<<<(unsigned)n, TRI_BASE, 0, h->stream>>>((int)n, L, ldl, X, ldx);
    h->launches++;
    CHFSI_CHECK_LAUNCH();
    return OK;
  }
  long long n1 = ((n / 2) + 31) / 32 * 32;
  const long long n2 = n - n1;
  CHFSI_TRY(trtri_rec(h, n1, L, ldl, X, ldx, tmp));
  CHFSI_TRY(trtri_rec(h, n2, L + n1 + n1 * ldl, ldl, X + n1 + n1 * ldx, ldx, tmp));
  // tmp(n2 x n1) = L21 * X11 ; X21 = -X22 * tmp ; X12 = 0
  // (X11 and X22 are lower triangular: their zero blocks are skipped)
  CHFSI_TRY(zgemm(h, OP_N, OP_N, n2, n1, n1, make_double2(1.0, 0.0), L + n1, ldl, X, ldx,
                  make_double2(0.0, 0.0), tmp, n2, TRI_B_LOWER));
  CHFSI_TRY(zgemm(h, OP_N, OP_N, n2, n1, n2, make_double2(-1.0, 0.0), X + n1 + n1 * ldx, ldx,
                  tmp, n2, make_double2(0.0, 0.0), X + n1, ldx, TRI_A_LOWER));
  CHFSI_CUDA(cudaMemset2DAsync(X + n1 * ldx, ldx * sizeof(double2), 0, n1 * sizeof(double2), n2,
                               h->stream));
  return OK;
}

int trtri_lower(Handle* h, long long n, const double2* L, long long ldl, double2* X,
                long long ldx) {
  if (n <= 0) return OK;
  double2* tmp = nullptr;
  if (n > TRI_BASE) {
    const long long n1 = ((n / 2) + 31) / 32 * 32;
    tmp = (double2*)scratch(h, SLOT_TRI, (size_t)n1 * (n - n1) * sizeof(double2));
    if (!tmp) return ERR_NOMEM;
  }
  return trtri_rec(h, n, L, ldl, X, ldx, tmp);
}

int zaxpby_cols(Handle* h, long long n, long long k, double2 alpha, const double2* X,
                long long ldx, double2 beta, double2* Y, long long ldy) {
  if (n * k <= 0) return OK;
  zaxpby_kernel<<<grid_for(n * k), 256, 0, h->stream>>>(n, k, alpha, X, ldx, beta, Y, ldy);
  h->launches++;
  CHFSI_CHECK_LAUNCH();
  return OK;
}

int sum_plane(Handle* h, long long rows, long long cols, const double2* X, long long ldx,
              double* Xs, long long ldxs) {
  if (rows * cols <= 0) return OK;
  const long long bx = std::min<long long>((rows + 255) / 256, 64);
  const long long by = std::min<long long>(cols, 65535);
  sum_plane_kernel<<<dim3((unsigned)bx, (unsigned)by), 256, 0, h->stream>>>(rows, cols, X, ldx, Xs,
                                                                           ldxs);
  h->launches++;
  CHFSI_CHECK_LAUNCH();
  return OK;
}

int sum_plane_grouped(Handle* h, long long rows, long long cols, const double2* X, long long ldx,
                      double* Xs) {
  if (rows * cols <= 0) return OK;
  if (rows % 8 != 0) {
    set_error("sum_plane_grouped: rows must be a multiple of 8");
    return ERR_ARG;
  }
  const long long bx = std::min<long long>((rows + 255) / 256, 64);
  const long long by = std::min<long long>(cols, 65535);
  sum_plane_grouped_kernel<<<dim3((unsigned)bx, (unsigned)by), 256, 0, h->stream>>>(rows, cols, X,
                                                                                   ldx, Xs);
  h->launches++;
  CHFSI_CHECK_LAUNCH();
  return OK;
}

int get_real_diag(Handle* h, long long n, const double2* A, long long lda, double* out_dev) {
  real_diag_kernel<<<grid_for(n), 256, 0, h->stream>>>(n, A, lda, out_dev);
  h->launches++;
  CHFSI_CHECK_LAUNCH();
  return OK;
}

int shift_diag(Handle* h, long long n, double2* A, long long lda, double shift) {
  shift_diag_kernel<<<grid_for(n), 256, 0, h->stream>>>(n, A, lda, shift);
  h->launches++;
  CHFSI_CHECK_LAUNCH();
  return OK;
}

int zgemv_n(Handle* h, long long M, long long K, double2 alpha, const double2* A, long long lda,
            const double2* x, double2 beta, double2* y) {
  if (M <= 0) return OK;
  const long long bx = (M + GV_T - 1) / GV_T;
  // ~8 resident 256-thread CTAs per SM (full occupancy) over the whole grid
  const long long want = 8LL * h->sm_count;
  long long S = std::max<long long>(1, (want + bx - 1) / bx);
  S = std::min<long long>(S, std::max<long long>(1, K / (4 * GV_U)));
  S = std::min<long long>(S, 64);
  double2* part = (double2*)scratch(h, SLOT_GEMV, (size_t)S * M * sizeof(double2));
  if (!part) return ERR_NOMEM;
  zgemv_partial_kernel<<<dim3((unsigned)bx, (unsigned)S), GV_T, 0, h->stream>>>(M, K, (int)S, A,
                                                                              lda, x, part);
  h->launches++;
  CHFSI_CHECK_LAUNCH();
  zgemv_finish_kernel<<<(unsigned)((M + 255) / 256), 256, 0, h->stream>>>(M, (int)S, part, alpha,
                                                                          beta, y);
  h->launches++;
  CHFSI_CHECK_LAUNCH();
  return OK;
}

int zcopy2d(Handle* h, long long rows, long long cols, const double2* src, long long lds,
            double2* dst, long long ldd) {
  if (rows * cols <= 0) return OK;
  CHFSI_CUDA(cudaMemcpy2DAsync(dst, ldd * sizeof(double2), src, lds * sizeof(double2),
                               rows * sizeof(double2), cols, cudaMemcpyDeviceToDevice, h->stream));
  return OK;
}

}  // namespace chfsi
