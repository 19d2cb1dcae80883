// Composite ChFSI phases built on the DMMA GEMM and helper kernels.
//
//   filter          core.py:263-284 (_filter_raw)
//   lanczos_bound   core.py:202-256 (lanczos_upper_bound)
//   orthonormalize  core.py:365-382 (_qr_against_locked): CGS2 against the
//                   locked block, then CholQR2 (shifted CholQR3 when the first
//                   Cholesky breaks down); rank test on |prod diag R| like
//                   linalg.py:284-288 / core.py:374-377.
//   rayleigh_ritz   core.py:318-330 (_rr_raw); cuSOLVER zheevd for the k x k
//                   eigenproblem (replaces the numba Jacobi _jacobi.py:14-80).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace chfsi {

namespace {
const double2 ONE = {1.0, 0.0};
const double2 ZERO = {0.0, 0.0};
const double2 MONE = {-1.0, 0.0};

#define CHFSI_SOLVER(call)                                                          \
  do {                                                                              \
    cusolverStatus_t s_ = (call);                                                   \
    if (s_ != CUSOLVER_STATUS_SUCCESS) {                                            \
      ::chfsi::set_error(std::string(#call) + ": cusolver status " + std::to_string((int)s_)); \
      return ::chfsi::ERR_CUSOLVER;                                                 \
    }                                                                               \
  } while (0)

}  // namespace

static int filter_issue(Handle* h, long long n, long long k, int degree, const double* coef,
                        const double* coef_dev, const double2* H, long long ldh, double2* Y,
                        long long ldy, double2* W, long long ldw, int* result_in_w);
static int filter_graphed(Handle* h, long long n, long long k, int degree, const double* coef,
                          const double2* H, long long ldh, double2* Y, long long ldy, double2* W,
                          long long ldw, int* result_in_w);
bool filter_graphs_enabled();

int potrf_lower(Handle* h, long long n, double2* A, long long lda, int* info_host) {
  int lwork = 0;
  CHFSI_SOLVER(cusolverDnZpotrf_bufferSize(h->solver, CUBLAS_FILL_MODE_LOWER, (int)n,
                                           (cuDoubleComplex*)A, (int)lda, &lwork));
  void* work = scratch(h, SLOT_SOLVER, (size_t)std::max(lwork, 1) * sizeof(cuDoubleComplex));
  if (!work) return ERR_NOMEM;
  CHFSI_SOLVER(cusolverDnZpotrf(h->solver, CUBLAS_FILL_MODE_LOWER, (int)n, (cuDoubleComplex*)A,
                                (int)lda, (cuDoubleComplex*)work, lwork, h->d_info));
  h->launches++;
  CHFSI_CUDA(cudaMemcpyAsync(info_host, h->d_info, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CHFSI_CUDA(cudaStreamSynchronize(h->stream));
  return OK;
}

// k x k Hermitian eigensolve (cuSOLVER zheevd): ascending eigenvalues to w_dev,
// eigenvectors over A, status to info_dev; enqueued on the handle's stream, no host
// sync. Measured on B200 (scripts/heevd_probe.py): 0.3 ms at k = 24, 2.3 ms at 120,
// 44 ms at 2200; cuSOLVER's Jacobi solvers (zheevj, zheevjBatched) were no faster at
// any of these widths (0.76 / 4.1 / 618 ms).
static int eig_small(Handle* h, long long n, double2* A, long long lda, double* w_dev,
                     int* info_dev) {
  const auto jobz = CUSOLVER_EIG_MODE_VECTOR;
  const auto uplo = CUBLAS_FILL_MODE_LOWER;
  int lwork = 0;
  CHFSI_SOLVER(cusolverDnZheevd_bufferSize(h->solver, jobz, uplo, (int)n, (cuDoubleComplex*)A,
                                           (int)lda, w_dev, &lwork));
  void* work = scratch(h, SLOT_SOLVER, (size_t)std::max(lwork, 1) * sizeof(cuDoubleComplex));
  if (!work) return ERR_NOMEM;
  CHFSI_SOLVER(cusolverDnZheevd(h->solver, jobz, uplo, (int)n, (cuDoubleComplex*)A, (int)lda,
                                w_dev, (cuDoubleComplex*)work, lwork, info_dev));
  h->launches++;
  return OK;
}

int heevd(Handle* h, long long n, double2* A, long long lda, double* w_dev) {
  CHFSI_TRY(eig_small(h, n, A, lda, w_dev, h->d_info));
  int info = 0;
  CHFSI_CUDA(cudaMemcpyAsync(&info, h->d_info, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CHFSI_CUDA(cudaStreamSynchronize(h->stream));
  if (info != 0) {
    set_error("zheevd failed to converge, info=" + std::to_string(info));
    return ERR_CUSOLVER;
  }
  return OK;
}

// Scaled three-term recurrence coefficients {alpha, beta, gamma} per degree step
// (core.py:263-284 `_filter_raw`).
static std::vector<double> filter_coefs(int degree, double a, double b, double lam_ref) {
  std::vector<double> coef(3 * (size_t)degree);
  const double c = (a + b) / 2.0;
  const double e = (b - a) / 2.0;
  const double sigma1 = e / (lam_ref - c);
  double sigma = sigma1;
  // y1 = sigma1/e * H y - c*sigma1/e * y
  coef[0] = sigma1 / e;
  coef[1] = -c * sigma1 / e;
  coef[2] = 0.0;
  for (int j = 1; j < degree; ++j) {
    // y2 = scale*(H y1) - c*scale*y1 - sigma*sigma_new*y0, written over y0
    const double sigma_new = 1.0 / (2.0 / sigma1 - sigma);
    const double scale = 2.0 * sigma_new / e;
    coef[3 * j] = scale;
    coef[3 * j + 1] = -c * scale;
    coef[3 * j + 2] = -(sigma * sigma_new);
    sigma = sigma_new;
  }
  return coef;
}

// 3M operand-sum planes of one filter call (complex_mul() == 3, n % 8 == 0): Hs = Re H +
// Im H in the grouped A layout and one column-major plane per rotating block (Y, W), ld
// rounded up to an even count (TMA strides are multiples of 16 B). Each fused step reads the planes of H and of its input block and
// writes the plane of its output from the epilogue, so no step adds DADDs to the DMMA
// stream. nullptr when 3M is off or the block is empty.
struct FilterSums {
  double* Hs = nullptr;
  double* Ys = nullptr;  // plane of Y (slot 0) and of W (slot 1)
  double* Ws = nullptr;
  long long ldh = 0, ldy = 0;
};

static int filter_sums(Handle* h, long long n, long long k, const double2* H, long long ldh,
                       const double2* Y, long long ldy, FilterSums* fs, bool h_plane = true) {
  *fs = FilterSums{};
  if (complex_mul() != 3 || n <= 0 || k <= 0 || n % 8 != 0) return OK;
  const long long ld = (n + 1) & ~1LL;
  fs->ldh = fs->ldy = ld;
  // a declared operator (chfsi_declare_operator) keeps its plane across calls
  const bool declared = h->op_ptr == (const void*)H && h->op_n == n && h->op_ld == ldh;
  if (!declared) h->op_ptr = nullptr;  // the plane is about to be overwritten
  fs->Hs = (double*)scratch(h, SLOT_HSUM, (size_t)ld * n * sizeof(double));
  fs->Ys = (double*)scratch(h, SLOT_YSUM, (size_t)2 * ld * k * sizeof(double));
  if (!fs->Hs || !fs->Ys) return ERR_NOMEM;
  fs->Ws = fs->Ys + ld * k;
  // (h_plane = false: the caller fills Hs itself -- the streamed filter, panel by panel)
  if (!declared && h_plane) CHFSI_TRY(sum_plane_grouped(h, n, n, H, ldh, fs->Hs));
  return sum_plane(h, n, k, Y, ldy, fs->Ys, ld);
}

int apply_operator(Handle* h, long long n, long long k, const double2* H, long long ldh,
                   const double2* X, long long ldx, double2* Y, long long ldy) {
  const bool declared = h->op_ptr == (const void*)H && h->op_n == n && h->op_ld == ldh &&
                        complex_mul() == 3 && n % 8 == 0;
  if (!declared || k <= 0)
    return zgemm(h, OP_N, OP_N, n, k, n, ONE, H, ldh, X, ldx, ZERO, Y, ldy);
  const long long ld = (n + 1) & ~1LL;
  double* hs = (double*)scratch(h, SLOT_HSUM, (size_t)ld * n * sizeof(double));
  double* xs = (double*)scratch(h, SLOT_YSUM, (size_t)ld * k * sizeof(double));
  if (!hs || !xs) return ERR_NOMEM;
  CHFSI_TRY(sum_plane(h, n, k, X, ldx, xs, ld));
  SumPlanes sp{hs, ld, xs, ld, nullptr, 0};
  return zgemm_nn_sums(h, n, k, n, H, ldh, X, ldx, Y, ldy, &sp);
}

// chfsi_declare_operator: H stays unchanged until the next declaration (or a clear with
// H = nullptr); its sum plane is computed now and reused by the filter calls on it.
int declare_operator(Handle* h, long long n, const double2* H, long long ldh) {
  h->op_ptr = nullptr;
  h->op_n = h->op_ld = 0;
  if (H == nullptr || n <= 0 || complex_mul() != 3 || n % 8 != 0) return OK;
  if (ldh < n) {
    set_error("declare_operator: ldh must be >= n");
    return ERR_ARG;
  }
  const long long ld = (n + 1) & ~1LL;
  double* hs = (double*)scratch(h, SLOT_HSUM, (size_t)ld * n * sizeof(double));
  if (!hs) return ERR_NOMEM;
  CHFSI_TRY(sum_plane_grouped(h, n, n, H, ldh, hs));
  h->op_ptr = H;
  h->op_n = n;
  h->op_ld = ldh;
  return OK;
}

// Degree steps j0 .. degree-1 (step j0 - 1 left its result in `cur`, its input in `prev`).
static int filter_steps(Handle* h, long long n, long long k, int degree, int j0, const double* coef,
                        const double* coef_dev, const double2* H, long long ldh, double2* prev,
                        long long ldp, double2* cur, long long ldc, double2* W,
                        int* result_in_w, const FilterSums* fs = nullptr) {
  // sum planes follow their blocks: after step j0 - 1 the output (cur) is W iff j0 is odd
  const bool sums = fs != nullptr && fs->Hs != nullptr;
  double* s_prev = nullptr;
  double* s_cur = nullptr;
  if (sums) {
    s_cur = (cur == W) ? fs->Ws : fs->Ys;
    s_prev = (cur == W) ? fs->Ys : fs->Ws;
  }
  for (int j = j0; j < degree; ++j) {
    SumPlanes sp{fs ? fs->Hs : nullptr, fs ? fs->ldh : 0, s_cur, fs ? fs->ldy : 0, s_prev,
                 fs ? fs->ldy : 0};
    CHFSI_TRY(zgemm_filter_step(h, n, k, H, ldh, cur, ldc, coef[3 * j], coef[3 * j + 1], prev, ldp,
                                coef[3 * j + 2], prev, ldp, coef_dev ? coef_dev + 3 * j : nullptr,
                                sums ? &sp : nullptr));
    std::swap(prev, cur);
    std::swap(ldp, ldc);
    std::swap(s_prev, s_cur);
  }
  *result_in_w = (cur == W) ? 1 : 0;
  return OK;
}

int filter(Handle* h, long long n, long long k, int degree, double a, double b, double lam_ref,
           const double2* H, long long ldh, double2* Y, long long ldy, double2* W, long long ldw,
           int* result_in_w) {
  if (degree < 1) {
    set_error("filter degree must be >= 1");
    return ERR_ARG;
  }
  const std::vector<double> coef = filter_coefs(degree, a, b, lam_ref);
  if (filter_graphs_enabled())
    return filter_graphed(h, n, k, degree, coef.data(), H, ldh, Y, ldy, W, ldw, result_in_w);
  return filter_issue(h, n, k, degree, coef.data(), nullptr, H, ldh, Y, ldy, W, ldw, result_in_w);
}

// The degree fused steps; with coef_dev the epilogues read the coefficients from
// device memory (graph capture), else from the launch arguments.
static int filter_issue(Handle* h, long long n, long long k, int degree, const double* coef,
                        const double* coef_dev, const double2* H, long long ldh, double2* Y,
                        long long ldy, double2* W, long long ldw, int* result_in_w) {
  // graph capture (coef_dev) keeps the plain kernels: no scratch growth inside a capture
  FilterSums fs;
  if (coef_dev == nullptr) CHFSI_TRY(filter_sums(h, n, k, H, ldh, Y, ldy, &fs));
  SumPlanes sp{fs.Hs, fs.ldh, fs.Ys, fs.ldy, fs.Ws, fs.ldy};
  CHFSI_TRY(zgemm_filter_step(h, n, k, H, ldh, Y, ldy, coef[0], coef[1], nullptr, 0, 0.0, W, ldw,
                              coef_dev, fs.Hs ? &sp : nullptr));
  return filter_steps(h, n, k, degree, 1, coef, coef_dev, H, ldh, Y, ldy, W, ldw, W, result_in_w,
                      &fs);
}

// Filter whose operator arrives from host memory (core.py:287-311 `chebyshev_filter`
// called with an ndarray H): H is uploaded in `panels` row panels on a copy stream
// (strided 2-D copies of the column-major rows [r0, r1)), and the first degree step
// runs panel by panel as the rows land -- output rows [r0, r1) need only H[r0:r1, :]
// and the (already resident) Y. Degree steps 2.. need all of H and start once the last
// panel is in. With pinned host memory the upload (PCIe) hides behind the first step
// except for one panel. Every panel step accumulates each output over K in the same
// order as the full-height step, so the result is identical when no panel uses split-K.
// Rows [r0, r0 + m) of a device block (column-major, ld) to the same rows of a host
// block, on the copy stream once the compute stream has produced them (event `ev`).
static int panel_to_host(Handle* h, cudaEvent_t ev, const double2* src, long long lds,
                         long long m, long long k, double2* dst, long long ldd) {
  CHFSI_CUDA(cudaEventRecord(ev, h->stream));
  CHFSI_CUDA(cudaStreamWaitEvent(h->copy_stream, ev, 0));
  CHFSI_CUDA(cudaMemcpy2DAsync(dst, (size_t)ldd * sizeof(double2), src,
                               (size_t)lds * sizeof(double2), (size_t)m * sizeof(double2),
                               (size_t)k, cudaMemcpyDeviceToHost, h->copy_stream));
  return OK;
}

int filter_streamed(Handle* h, long long n, long long k, int degree, double a, double b,
                    double lam_ref, const double2* H_host, long long ldh_host, double2* H,
                    long long ldh, double2* Y, long long ldy, double2* W, long long ldw,
                    int panels, int* result_in_w, double2* out_host, long long ld_out) {
  if (degree < 1) {
    set_error("filter degree must be >= 1");
    return ERR_ARG;
  }
  if (n <= 0 || k <= 0) {
    *result_in_w = 0;
    return OK;
  }
  if (ldh_host < n || ldh < n || (out_host != nullptr && ld_out < n)) {
    set_error("filter_streamed: leading dimensions must be >= n");
    return ERR_ARG;
  }
  if (h->op_ptr == (const void*)H) h->op_ptr = nullptr;  // H is rewritten below
  if (panels <= 0) panels = n >= 8192 ? 8 : (n >= 2048 ? 4 : 1);
  // panel height: a multiple of 64 rows (the CTA tile height)
  long long rows = (n + panels - 1) / panels;
  rows = ((rows + 63) / 64) * 64;
  panels = (int)((n + rows - 1) / rows);
  if (!h->copy_stream)
    CHFSI_CUDA(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
  if (!h->copy_events) h->copy_events = new std::vector<cudaEvent_t>();
  auto& ev = *h->copy_events;
  // events: [0, panels) H panels landed, [panels] stream fence, [panels + 1 + p] output
  // panel p computed (D2H of the last step)
  while ((int)ev.size() < 2 * panels + 1) {
    cudaEvent_t e;
    CHFSI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ev.push_back(e);
  }
  const std::vector<double> coef = filter_coefs(degree, a, b, lam_ref);
  // 3M sum planes: Y's now, H's panel by panel as its rows land, the first step's
  // output plane from the panel epilogues -- so the first step runs the sum-plane
  // kernels too and no full-H plane pass follows the upload
  FilterSums fs;
  CHFSI_TRY(filter_sums(h, n, k, H, ldh, Y, ldy, &fs, /*h_plane=*/false));
  // the destination may still be read by earlier work queued on the compute stream
  CHFSI_CUDA(cudaEventRecord(ev[panels], h->stream));
  CHFSI_CUDA(cudaStreamWaitEvent(h->copy_stream, ev[panels], 0));
  for (int p = 0; p < panels; ++p) {
    const long long r0 = p * rows;
    const long long m = std::min(rows, n - r0);
    // pinned: one strided 2-D copy; pageable: through the pinned staging ring, the host
    // threads filling panel p + 1 while panel p's step runs (staging.cu)
    CHFSI_TRY(upload_2d(h, H_host + r0, ldh_host, m, n, H + r0, ldh, h->copy_stream));
    CHFSI_CUDA(cudaEventRecord(ev[p], h->copy_stream));
    // enqueue the panel's step right behind its copy: with pageable host memory the
    // copy call returns only once staged, and the step of panel p then overlaps the
    // staging of panel p + 1
    CHFSI_CUDA(cudaStreamWaitEvent(h->stream, ev[p], 0));
    if (fs.Hs != nullptr) {
      // grouped plane rows [r0, r0 + m) start at group r0 / 8 (r0, m multiples of 8)
      double* hs_panel = fs.Hs + r0 * n;
      CHFSI_TRY(sum_plane_grouped(h, m, n, H + r0, ldh, hs_panel));
      SumPlanes sp{hs_panel, 0, fs.Ys, fs.ldy, fs.Ws + r0, fs.ldy};
      CHFSI_TRY(zgemm_filter_panel(h, m, k, n, H + r0, ldh, Y, ldy, Y + r0, ldy, coef[0],
                                   coef[1], nullptr, 0, 0.0, W + r0, ldw, nullptr, &sp));
    } else {
      CHFSI_TRY(zgemm_filter_panel(h, m, k, n, H + r0, ldh, Y, ldy, Y + r0, ldy, coef[0],
                                   coef[1], nullptr, 0, 0.0, W + r0, ldw, nullptr));
    }
    if (out_host != nullptr && degree == 1)
      CHFSI_TRY(panel_to_host(h, ev[panels + 1 + p], W + r0, ldw, m, k, out_host + r0, ld_out));
  }
  if (out_host == nullptr || degree == 1) {
    CHFSI_TRY(filter_steps(h, n, k, degree, 1, coef.data(), nullptr, H, ldh, Y, ldy, W, ldw, W,
                           result_in_w, &fs));
  } else {
    // steps 2 .. degree - 1, then the last step by row panels, each panel read back to
    // the host on the copy stream while the next panel computes
    int in_w = 1;
    CHFSI_TRY(filter_steps(h, n, k, degree - 1, 1, coef.data(), nullptr, H, ldh, Y, ldy, W, ldw,
                           W, &in_w, &fs));
    double2* cur = in_w ? W : Y;
    double2* prev = in_w ? Y : W;
    const long long ldc = in_w ? ldw : ldy, ldp = in_w ? ldy : ldw;
    double* s_cur = fs.Hs ? (in_w ? fs.Ws : fs.Ys) : nullptr;
    const int j = degree - 1;
    for (int p = 0; p < panels; ++p) {
      const long long r0 = p * rows;
      const long long m = std::min(rows, n - r0);
      SumPlanes sp{fs.Hs ? fs.Hs + r0 * n : nullptr, 0, s_cur, fs.ldy, nullptr, 0};
      CHFSI_TRY(zgemm_filter_panel(h, m, k, n, H + r0, ldh, cur, ldc, cur + r0, ldc,
                                   coef[3 * j], coef[3 * j + 1], prev + r0, ldp,
                                   coef[3 * j + 2], prev + r0, ldp, nullptr,
                                   fs.Hs ? &sp : nullptr));
      CHFSI_TRY(panel_to_host(h, ev[panels + 1 + p], prev + r0, ldp, m, k, out_host + r0, ld_out));
    }
    *result_in_w = (prev == W) ? 1 : 0;
  }
  // everything is queued; return once the host buffer has been read so the caller
  // may free or reuse it (the GPU keeps filtering meanwhile) -- or, with out_host, once
  // the result has landed there
  CHFSI_CUDA(cudaEventSynchronize(ev[panels - 1]));
  if (out_host != nullptr) CHFSI_CUDA(cudaStreamSynchronize(h->copy_stream));
  return OK;
}

void destroy_copy_stream(Handle* h) {
  if (h->copy_events) {
    for (cudaEvent_t e : *h->copy_events) cudaEventDestroy(e);
    delete h->copy_events;
    h->copy_events = nullptr;
  }
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  h->copy_stream = nullptr;
}

// Opt-in (CHFSI_FILTER_GRAPHS=1). Measured on B200 (scripts/graph_micro.py): a replay
// saves 12 % of a filter call at n = 1000 (each fused step is ~23 us of GPU work, so
// the calls are not launch-bound), while a c0 solve hits 115 distinct
// (width, buffer) configurations whose capture + instantiate cost more than the
// replays save (c0 filter time 1.07 s -> 2.82 s). Off by default.
bool filter_graphs_enabled() {
  static const bool on = [] {
    const char* s = getenv("CHFSI_FILTER_GRAPHS");
    return s && s[0] == '1';
  }();
  return on;
}

void destroy_filter_graphs(Handle* h) {
  if (!h->graphs) return;
  for (auto& g : *h->graphs) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
    if (g.ws) cudaFree(g.ws);
    if (g.coef) cudaFree(g.coef);
  }
  delete h->graphs;
  h->graphs = nullptr;
}

// CUDA-graph path: one captured launch sequence per (buffers, shape, degree); each
// call only uploads the 3*degree coefficients and replays it. Small solves are
// launch-bound (a fused step at n = 1000 is a few microseconds of GPU work).
static int filter_graphed(Handle* h, long long n, long long k, int degree, const double* coef,
                          const double2* H, long long ldh, double2* Y, long long ldy, double2* W,
                          long long ldw, int* result_in_w) {
  constexpr size_t kMaxGraphs = 32;
  if (!h->graphs) h->graphs = new std::vector<FilterGraph>();
  int fcfg = -1, fsplit = 0;
  gemm_overrides(&fcfg, &fsplit);
  FilterGraph* hit = nullptr;
  for (auto& g : *h->graphs)
    if (g.H == H && g.Y == Y && g.W == W && g.n == n && g.k == k && g.ldh == ldh &&
        g.ldy == ldy && g.ldw == ldw && g.degree == degree && g.force_cfg == fcfg &&
        g.force_split == fsplit) {
      hit = &g;
      break;
    }
  if (!hit) {
    if (h->graphs->size() >= kMaxGraphs) {  // evict the least recently used entry
      auto lru = h->graphs->begin();
      for (auto it = h->graphs->begin(); it != h->graphs->end(); ++it)
        if (it->last_use < lru->last_use) lru = it;
      CHFSI_CUDA(cudaStreamSynchronize(h->stream));
      cudaGraphExecDestroy(lru->exec);
      cudaGraphDestroy(lru->graph);
      if (lru->ws) cudaFree(lru->ws);
      cudaFree(lru->coef);
      h->graphs->erase(lru);
    }
    FilterGraph g;
    g.H = H; g.Y = Y; g.W = W;
    g.n = n; g.k = k; g.ldh = ldh; g.ldy = ldy; g.ldw = ldw;
    g.degree = degree; g.force_cfg = fcfg; g.force_split = fsplit;
    const size_t ws_bytes = filter_step_workspace(h, n, k);  // also builds the kernel table
    if (ws_bytes) CHFSI_CUDA(cudaMalloc(&g.ws, ws_bytes));
    CHFSI_CUDA(cudaMalloc(&g.coef, 3 * (size_t)degree * sizeof(double)));
    h->ws_override = g.ws;
    h->ws_override_bytes = ws_bytes;
    const long long before = h->launches;
    // capture on a private stream (capture executes nothing; the caller's stream may be
    // the legacy default stream, which cannot capture), replay on the caller's stream
    if (!h->capture_stream)
      CHFSI_CUDA(cudaStreamCreateWithFlags(&h->capture_stream, cudaStreamNonBlocking));
    cudaStream_t user_stream = h->stream;
    h->stream = h->capture_stream;
    cudaError_t ce = cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal);
    int st = OK;
    cudaGraph_t graph = nullptr;
    if (ce == cudaSuccess) {
      st = filter_issue(h, n, k, degree, coef, g.coef, H, ldh, Y, ldy, W, ldw, &g.result_in_w);
      ce = cudaStreamEndCapture(h->stream, &graph);
    }
    h->stream = user_stream;
    h->ws_override = nullptr;
    h->ws_override_bytes = 0;
    if (st != OK || ce != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      if (g.ws) cudaFree(g.ws);
      cudaFree(g.coef);
      if (st != OK) return st;
      set_error(std::string("filter graph capture: ") + cudaGetErrorString(ce));
      return ERR_CUDA;
    }
    g.launches = h->launches - before;
    h->launches = before;  // captured, not executed
    static const bool dbg = getenv("CHFSI_GRAPH_DEBUG") != nullptr;
    if (dbg)
      fprintf(stderr, "[chfsi] filter graph capture #%zu: n=%lld k=%lld degree=%d Y=%p W=%p\n",
              h->graphs->size() + 1, n, k, degree, (const void*)Y, (const void*)W);
    g.graph = graph;
    CHFSI_CUDA(cudaGraphInstantiate(&g.exec, graph, 0));
    h->graphs->push_back(g);
    hit = &h->graphs->back();
  }
  hit->last_use = ++h->graph_tick;
  CHFSI_CUDA(cudaMemcpyAsync(hit->coef, coef, 3 * (size_t)degree * sizeof(double),
                             cudaMemcpyHostToDevice, h->stream));
  CHFSI_CUDA(cudaGraphLaunch(hit->exec, h->stream));
  h->launches += hit->launches;
  *result_in_w = hit->result_in_w;
  return OK;
}

// eigenvalues of a real symmetric tridiagonal (diag d, offdiag e) by cyclic Jacobi
static void sym_eig_small(int m, const double* d, const double* e, double* lam) {
  std::vector<double> A((size_t)m * m, 0.0);
  for (int i = 0; i < m; ++i) {
    A[i * m + i] = d[i];
    if (i + 1 < m) A[i * m + i + 1] = A[(i + 1) * m + i] = e[i];
  }
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, fro = 0.0;
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) {
        fro += A[i * m + j] * A[i * m + j];
        if (i != j) off += A[i * m + j] * A[i * m + j];
      }
    if (off <= 1e-32 * fro || off == 0.0) break;
    for (int p = 0; p < m - 1; ++p)
      for (int q = p + 1; q < m; ++q) {
        const double apq = A[p * m + q];
        if (apq == 0.0) continue;
        const double tau = (A[q * m + q] - A[p * m + p]) / (2.0 * apq);
        const double t = (tau >= 0 ? 1.0 : -1.0) / (std::fabs(tau) + std::sqrt(1.0 + tau * tau));
        const double cs = 1.0 / std::sqrt(1.0 + t * t), sn = t * cs;
        for (int r = 0; r < m; ++r) {
          const double arp = A[r * m + p], arq = A[r * m + q];
          A[r * m + p] = cs * arp - sn * arq;
          A[r * m + q] = sn * arp + cs * arq;
        }
        for (int r = 0; r < m; ++r) {
          const double apr = A[p * m + r], aqr = A[q * m + r];
          A[p * m + r] = cs * apr - sn * aqr;
          A[q * m + r] = sn * apr + cs * aqr;
        }
      }
  }
  for (int i = 0; i < m; ++i) lam[i] = A[i * m + i];
  std::sort(lam, lam + m);
}

int lanczos_bound(Handle* h, long long n, int k, const double2* H, long long ldh,
                  const double2* v0, double* alphas, double* betas, int* steps, double* bound) {
  if (k < 2) {
    set_error("lanczos steps must be >= 2");
    return ERR_ARG;
  }
  if (k > n) k = (int)n;
  double2* basis = (double2*)scratch(h, SLOT_LANCZOS, (size_t)n * (k + 1) * sizeof(double2));
  double2* vec = (double2*)scratch(h, SLOT_VEC, (size_t)(2 * k + 8) * sizeof(double2));
  if (!basis || !vec) return ERR_NOMEM;
  double2* w = basis + (long long)n * k;
  double2* coeff = vec + 2;
  double* hst = pinned(h, 4 * sizeof(double));
  if (!hst) return ERR_NOMEM;
  CHFSI_TRY(zcopy2d(h, n, 1, v0, n, basis, n));
  int j = 0;
  for (; j < k; ++j) {
    double2* bj = basis + (long long)j * n;
    CHFSI_TRY(zgemm(h, OP_N, OP_N, n, 1, n, ONE, H, ldh, bj, n, ZERO, w, n));
    CHFSI_TRY(zdotc_cols(h, n, 1, bj, n, w, n, vec));
    CHFSI_CUDA(cudaMemcpyAsync(hst, vec, sizeof(double2), cudaMemcpyDeviceToHost, h->stream));
    CHFSI_CUDA(cudaStreamSynchronize(h->stream));
    const double aj = hst[0];
    alphas[j] = aj;
    CHFSI_TRY(zaxpby_cols(h, n, 1, make_double2(-aj, 0.0), bj, n, ONE, w, n));
    if (j > 0)
      CHFSI_TRY(zaxpby_cols(h, n, 1, make_double2(-betas[j - 1], 0.0), bj - n, n, ONE, w, n));
    // full reorthogonalisation: w -= B (B^H w)
    CHFSI_TRY(zgemm(h, OP_C, OP_N, j + 1, 1, n, ONE, basis, n, w, n, ZERO, coeff, j + 1));
    CHFSI_TRY(zgemm(h, OP_N, OP_N, n, 1, j + 1, MONE, basis, n, coeff, j + 1, ONE, w, n));
    CHFSI_TRY(zdotc_cols(h, n, 1, w, n, w, n, vec));
    CHFSI_CUDA(cudaMemcpyAsync(hst, vec, sizeof(double2), cudaMemcpyDeviceToHost, h->stream));
    CHFSI_CUDA(cudaStreamSynchronize(h->stream));
    const double bj_norm = std::sqrt(hst[0]);
    betas[j] = bj_norm;
    if (bj_norm < 1e-14 || j == k - 1) {
      ++j;
      break;
    }
    CHFSI_TRY(zaxpby_cols(h, n, 1, make_double2(1.0 / bj_norm, 0.0), w, n, ZERO, bj + n, n));
  }
  *steps = j;
  std::vector<double> lam(j);
  sym_eig_small(j, alphas, betas, lam.data());
  const double guard = 4.0 * j * 2.220446049250313e-16 * std::max(std::fabs(lam[0]), std::fabs(lam[j - 1]));
  *bound = lam[j - 1] + betas[j - 1] + guard;
  return OK;
}

// One Cholesky-QR pass, fully stream-ordered (no host sync):
//   G = X^H X (+ shift I); G = L L^H (zpotrf, info -> info_dev); diag(L) -> diag_dev;
//   out = X L^-H  (R = L^H, so R^-1 = (L^-1)^H).
// A failed factorisation leaves garbage in `out`; callers check info after one sync.
static int cholqr_pass_async(Handle* h, long long n, long long k, const double2* X, long long ldx,
                             double2* out, long long ldo, double shift, double* diag_dev,
                             int* info_dev) {
  double2* G = (double2*)scratch(h, SLOT_SMALL, (size_t)k * k * sizeof(double2));
  double2* Li = (double2*)scratch(h, SLOT_SMALL2, (size_t)k * k * sizeof(double2));
  if (!G || !Li) return ERR_NOMEM;
  // Gram X^H X: lower-triangle tiles only (zpotrf reads the lower triangle; the mirror
  // keeps G Hermitian for the shifted pass and for callers reading it whole)
  CHFSI_TRY(zgemm(h, OP_C, OP_N, k, k, n, ONE, X, ldx, X, ldx, ZERO, G, k, TRI_C_LOWER));
  CHFSI_TRY(mirror_lower(h, k, G, k));
  if (shift != 0.0) CHFSI_TRY(shift_diag(h, k, G, k, shift));
  int lwork = 0;
  CHFSI_SOLVER(cusolverDnZpotrf_bufferSize(h->solver, CUBLAS_FILL_MODE_LOWER, (int)k,
                                           (cuDoubleComplex*)G, (int)k, &lwork));
  void* work = scratch(h, SLOT_SOLVER, (size_t)std::max(lwork, 1) * sizeof(cuDoubleComplex));
  if (!work) return ERR_NOMEM;
  CHFSI_SOLVER(cusolverDnZpotrf(h->solver, CUBLAS_FILL_MODE_LOWER, (int)k, (cuDoubleComplex*)G,
                                (int)k, (cuDoubleComplex*)work, lwork, info_dev));
  h->launches++;
  CHFSI_TRY(get_real_diag(h, k, G, k, diag_dev));
  CHFSI_TRY(trtri_lower(h, k, G, k, Li, k));
  // X R^-1 = X Li^H with Li = L^-1 lower triangular: skip its zero triangle
  CHFSI_TRY(zgemm(h, OP_N, OP_C, n, k, k, ONE, X, ldx, Li, k, ZERO, out, ldo, TRI_B_UPPER));
  return OK;
}

// Device-side small-vector block of one orthonormalisation, copied to the host in one go.
struct OrthVec {
  double* dots;  // 2k doubles (complex column self-dots)
  double* d[3];  // k each: diag(R) of up to three passes
  int* info;     // 3 ints
  size_t bytes;
};

static OrthVec orth_vec_layout(double* base, long long k) {
  OrthVec v;
  v.dots = base;
  v.d[0] = base + 2 * k;
  v.d[1] = base + 3 * k;
  v.d[2] = base + 4 * k;
  v.info = reinterpret_cast<int*>(base + 5 * k);
  v.bytes = (size_t)(5 * k) * sizeof(double) + 4 * sizeof(int);
  return v;
}

int orthonormalize(Handle* h, long long n, long long k, double2* F, long long ldf,
                   const double2* Lk, long long ldl, long long nl, double2* T, long long ldt,
                   double2* Q, long long ldq, double rank_rel_tol, long long* bad_col,
                   double* fro_out) {
  *bad_col = -1;
  if (k <= 0) return OK;
  CHFSI_TRY(project_out(h, n, k, F, ldf, Lk, ldl, nl));  // CGS2 against the locked block
  double* vbase = (double*)scratch(h, SLOT_VEC, (size_t)(5 * k + 4) * sizeof(double));
  if (!vbase) return ERR_NOMEM;
  const OrthVec dv = orth_vec_layout(vbase, k);
  double* hbase = pinned(h, dv.bytes);
  if (!hbase) return ERR_NOMEM;
  const OrthVec hv = orth_vec_layout(hbase, k);
  CHFSI_CUDA(cudaMemsetAsync(dv.info, 0, 3 * sizeof(int), h->stream));
  // ||W||_F via deterministic column dots; CholQR2 passes F -> T -> Q, all async
  CHFSI_TRY(zdotc_cols(h, n, k, F, ldf, F, ldf, (double2*)dv.dots));
  CHFSI_TRY(cholqr_pass_async(h, n, k, F, ldf, T, ldt, 0.0, dv.d[0], dv.info + 0));
  CHFSI_TRY(cholqr_pass_async(h, n, k, T, ldt, Q, ldq, 0.0, dv.d[1], dv.info + 1));
  CHFSI_CUDA(cudaMemcpyAsync(hbase, vbase, dv.bytes, cudaMemcpyDeviceToHost, h->stream));
  CHFSI_CUDA(cudaStreamSynchronize(h->stream));  // the one host sync of the fast path
  double s = 0.0;
  for (long long j = 0; j < k; ++j) s += hv.dots[2 * j];
  const double fro = std::sqrt(s);
  *fro_out = fro;
  bool shifted = false;
  if (hv.info[0] != 0) {
    // first Cholesky broke down (ill-conditioned block): shifted CholQR3
    // (Fukaya et al.), s = 11 (n k + k (k+1)) u ||F||^2, then two plain passes
    const double u = 1.1102230246251565e-16;
    const double sh = 11.0 * ((double)n * k + (double)k * (k + 1)) * u * fro * fro;
    CHFSI_CUDA(cudaMemsetAsync(dv.info, 0, 3 * sizeof(int), h->stream));
    CHFSI_TRY(cholqr_pass_async(h, n, k, F, ldf, T, ldt, sh, dv.d[0], dv.info + 0));
    CHFSI_TRY(cholqr_pass_async(h, n, k, T, ldt, Q, ldq, 0.0, dv.d[1], dv.info + 1));
    CHFSI_TRY(cholqr_pass_async(h, n, k, Q, ldq, T, ldt, 0.0, dv.d[2], dv.info + 2));
    CHFSI_TRY(zcopy2d(h, n, k, T, ldt, Q, ldq));
    CHFSI_CUDA(cudaMemcpyAsync(hbase, vbase, dv.bytes, cudaMemcpyDeviceToHost, h->stream));
    CHFSI_CUDA(cudaStreamSynchronize(h->stream));
    shifted = true;
  }
  for (int pass = 0; pass < (shifted ? 3 : 2); ++pass) {
    if (hv.info[pass] != 0) {
      *bad_col = hv.info[pass] - 1;
      set_error("rank collapse in column " + std::to_string(*bad_col));
      return ERR_RANK;
    }
  }
  for (long long j = 0; j < k; ++j) {
    double r = std::fabs(hv.d[0][j] * hv.d[1][j]);
    if (shifted) r *= std::fabs(hv.d[2][j]);
    if (r < rank_rel_tol * fro) {
      *bad_col = j;
      set_error("rank collapse in column " + std::to_string(j));
      return ERR_RANK;
    }
  }
  return OK;
}

// The replicated k x k step of a column-sharded CholQR pass (distributed.py
// ShardedPhases.orthonormalize; the n-sized Gram and X R^-1 products are split over
// the ranks by columns): G <- (G + G^H)/2 (+ shift I), trace(G) to the host, G = L L^H
// (zpotrf, lower, in place), Li = L^-1, diag(L) and the zpotrf info to the host --
// one host sync.
int cholesky_inverse(Handle* h, long long k, double2* G, long long ldg, double shift,
                     double2* Li, long long ldli, double* diag_host, double* trace_host,
                     int* info_host) {
  if (k <= 0) {
    *info_host = 0;
    *trace_host = 0.0;
    return OK;
  }
  double* v = (double*)scratch(h, SLOT_VEC, (size_t)(2 * k + 2) * sizeof(double));
  if (!v) return ERR_NOMEM;
  double* dg = v;          // diag(G) before the factorisation
  double* dl = v + k;      // diag(L)
  int* info_dev = reinterpret_cast<int*>(v + 2 * k);
  CHFSI_TRY(hermitize(h, k, G, ldg));
  CHFSI_TRY(get_real_diag(h, k, G, ldg, dg));
  if (shift != 0.0) CHFSI_TRY(shift_diag(h, k, G, ldg, shift));
  int lwork = 0;
  CHFSI_SOLVER(cusolverDnZpotrf_bufferSize(h->solver, CUBLAS_FILL_MODE_LOWER, (int)k,
                                           (cuDoubleComplex*)G, (int)ldg, &lwork));
  void* work = scratch(h, SLOT_SOLVER, (size_t)std::max(lwork, 1) * sizeof(cuDoubleComplex));
  if (!work) return ERR_NOMEM;
  CHFSI_CUDA(cudaMemsetAsync(info_dev, 0, sizeof(int), h->stream));
  CHFSI_SOLVER(cusolverDnZpotrf(h->solver, CUBLAS_FILL_MODE_LOWER, (int)k, (cuDoubleComplex*)G,
                                (int)ldg, (cuDoubleComplex*)work, lwork, info_dev));
  h->launches++;
  CHFSI_TRY(get_real_diag(h, k, G, ldg, dl));
  CHFSI_TRY(trtri_lower(h, k, G, ldg, Li, ldli));
  const size_t bytes = (size_t)(2 * k) * sizeof(double) + sizeof(int);
  double* hb = pinned(h, bytes + 16);
  if (!hb) return ERR_NOMEM;
  CHFSI_CUDA(cudaMemcpyAsync(hb, v, bytes, cudaMemcpyDeviceToHost, h->stream));
  CHFSI_CUDA(cudaStreamSynchronize(h->stream));
  double tr = 0.0;
  for (long long j = 0; j < k; ++j) tr += hb[j];
  *trace_host = tr;
  std::copy(hb + k, hb + 2 * k, diag_host);
  *info_host = *reinterpret_cast<int*>(hb + 2 * k);
  return OK;
}

// CGS2 projection of F against the locked block L (first half of core.py:371-372);
// column-local, so a column-sharded caller can run it on its own shard only.
int project_out(Handle* h, long long n, long long k, double2* F, long long ldf,
                const double2* Lk, long long ldl, long long nl) {
  if (nl <= 0 || k <= 0) return OK;
  double2* P = (double2*)scratch(h, SLOT_PROJ, (size_t)nl * k * sizeof(double2));
  if (!P) return ERR_NOMEM;
  for (int pass = 0; pass < 2; ++pass) {
    CHFSI_TRY(zgemm(h, OP_C, OP_N, nl, k, n, ONE, Lk, ldl, F, ldf, ZERO, P, nl));
    CHFSI_TRY(zgemm(h, OP_N, OP_N, n, k, nl, MONE, Lk, ldl, P, nl, ONE, F, ldf));
  }
  return OK;
}

// core.py:172-188 `reduce_to_standard`: H = L^-1 A L^-H from the triangular inverse
// Linv = L^-1 as two DMMA GEMMs that skip Linv's zero triangle (half the flops each):
// W = Linv A (row tile m needs k <= m), H = W Linv^H (column tile j needs k <= j).
int reduce_to_standard(Handle* h, long long n, const double2* A, long long lda,
                       const double2* Linv, long long ldli, double2* W, long long ldw,
                       double2* H, long long ldh) {
  CHFSI_TRY(zgemm(h, OP_N, OP_N, n, n, n, ONE, Linv, ldli, A, lda, ZERO, W, ldw, TRI_A_LOWER));
  return zgemm(h, OP_N, OP_C, n, n, n, ONE, W, ldw, Linv, ldli, ZERO, H, ldh, TRI_B_UPPER);
}

// core.py:318-330 `_rr_raw` plus the residual norms of core.py:477, with a single
// host sync: Ritz values, residuals and the zheevd info come back together.
// hq_ready: the caller already holds HQ = H Q (column-sharded multi-GPU path).
int rayleigh_ritz(Handle* h, long long n, long long k, const double2* H, long long ldh,
                  const double2* Q, long long ldq, double2* HQ, long long ldhq, double2* Z,
                  long long ldz, double2* HZ, long long ldhz, double* w_host, double* res_host,
                  bool hq_ready) {
  double2* G = (double2*)scratch(h, SLOT_SMALL, (size_t)k * k * sizeof(double2));
  double* v = (double*)scratch(h, SLOT_VEC, (size_t)(2 * k + 2) * sizeof(double));
  if (!G || !v) return ERR_NOMEM;
  double* w_dev = v;
  double* r_dev = v + k;
  int* info_dev = reinterpret_cast<int*>(v + 2 * k);
  if (!hq_ready) CHFSI_TRY(apply_operator(h, n, k, H, ldh, Q, ldq, HQ, ldhq));
  CHFSI_TRY(zgemm(h, OP_C, OP_N, k, k, n, ONE, Q, ldq, HQ, ldhq, ZERO, G, k));
  CHFSI_TRY(hermitize(h, k, G, k));
  CHFSI_TRY(eig_small(h, k, G, k, w_dev, info_dev));
  CHFSI_TRY(zgemm(h, OP_N, OP_N, n, k, k, ONE, Q, ldq, G, k, ZERO, Z, ldz));
  CHFSI_TRY(zgemm(h, OP_N, OP_N, n, k, k, ONE, HQ, ldhq, G, k, ZERO, HZ, ldhz));
  if (res_host) CHFSI_TRY(residual_norms(h, n, k, HZ, ldhz, Z, ldz, w_dev, r_dev));
  const size_t bytes = (size_t)(2 * k) * sizeof(double) + sizeof(int);
  double* hb = pinned(h, bytes + 16);
  if (!hb) return ERR_NOMEM;
  CHFSI_CUDA(cudaMemcpyAsync(hb, v, bytes, cudaMemcpyDeviceToHost, h->stream));
  CHFSI_CUDA(cudaStreamSynchronize(h->stream));
  const int info = *reinterpret_cast<int*>(hb + 2 * k);
  if (info != 0) {
    set_error("zheevd failed to converge, info=" + std::to_string(info));
    return ERR_CUSOLVER;
  }
  std::copy(hb, hb + k, w_host);
  if (res_host) std::copy(hb + k, hb + 2 * k, res_host);
  return OK;
}

}  // namespace chfsi
