// Internal (C++) interface shared by the translation units of libchfsi_b200.
#pragma once

#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace chfsi {

// Status codes returned through the C ABI (include/chfsi_b200.h).
enum Status : int {
  OK = 0,
  ERR_ARG = -1,        // contract violation on arguments
  ERR_CUDA = -2,       // CUDA runtime failure
  ERR_CUSOLVER = -3,   // cuSOLVER failure
  ERR_NOT_PD = -4,     // Cholesky pivot failure (detail = 1-based pivot)
  ERR_RANK = -5,       // rank collapse (detail = 0-based column)
  ERR_NOMEM = -6,
};

// One captured filter call (degree fused GEMM steps) for fixed buffers and shape.
// The graph bakes in pointers, so the entry owns its split-K workspace and its
// coefficient buffer; only the coefficients are rewritten before each replay.
struct FilterGraph {
  const void *H = nullptr, *Y = nullptr, *W = nullptr;
  long long n = 0, k = 0, ldh = 0, ldy = 0, ldw = 0;
  int degree = 0, force_cfg = -1, force_split = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  double2* ws = nullptr;
  double* coef = nullptr;
  int result_in_w = 0;
  long long launches = 0;
  unsigned long long last_use = 0;
};

struct Handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  cusolverDnHandle_t solver = nullptr;
  // grow-only scratch arenas (stream-ordered reuse is safe: one stream)
  static constexpr int kSlots = 12;
  void* scratch[kSlots] = {nullptr};
  size_t scratch_bytes[kSlots] = {0};
  int* d_info = nullptr;
  double* h_pinned = nullptr;   // small pinned host staging
  size_t h_pinned_bytes = 0;
  int sm_count = 148;
  // operator declared immutable by chfsi_declare_operator: its 3M sum plane (SLOT_HSUM)
  // is reused by every filter call on the same (pointer, order, ld)
  const void* op_ptr = nullptr;
  long long op_n = 0, op_ld = 0;
  // launch counter: kernels this library launched since the last reset
  long long launches = 0;
  // CUDA-graph cache of filter calls (solver_ops.cu) and the split-K workspace
  // override used while capturing one
  std::vector<FilterGraph>* graphs = nullptr;
  unsigned long long graph_tick = 0;
  cudaStream_t capture_stream = nullptr;  // private: the legacy default stream cannot capture
  double2* ws_override = nullptr;
  size_t ws_override_bytes = 0;
  // host->device upload stream and its per-panel events (streamed filter)
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t>* copy_events = nullptr;
  // pinned staging ring + host worker pool for pageable uploads (staging.cu)
  struct Stager* stager = nullptr;
};

void destroy_filter_graphs(Handle* h);
void destroy_copy_stream(Handle* h);
void destroy_stager(Handle* h);

// rows x cols column-major host block (ld_host, complex) -> device (ld_dev) on `stream`.
// Pinned sources: one async 2-D copy. Pageable sources: through the handle's pinned
// staging ring (host worker threads fill a slot while the DMA drains the previous one);
// returns once the host source has been read.
int upload_2d(Handle* h, const double2* host, long long ld_host, long long rows,
              long long cols, double2* dev, long long ld_dev, cudaStream_t stream);
bool host_is_pinned(const void* p);

// scratch slots
enum Slot : int {
  SLOT_SPLITK = 0,  // split-K partials
  SLOT_SMALL = 1,   // k x k Gram / eigvecs
  SLOT_SMALL2 = 2,  // k x k inverse factors
  SLOT_PROJ = 3,    // locked-projection coefficients nl x k
  SLOT_SOLVER = 4,  // cuSOLVER workspace
  SLOT_VEC = 5,     // small vectors (eigvalues, diagonals, norms)
  SLOT_TRI = 6,     // triangular-inverse temporaries
  SLOT_LANCZOS = 7, // Lanczos basis
  SLOT_COLRED = 8,  // per-column partial sums (split column reductions)
  SLOT_HSUM = 9,    // 3M sum plane of the filter operator H (n x n doubles)
  SLOT_YSUM = 10,   // 3M sum planes of the two rotating filter blocks (2 x n x k doubles)
  SLOT_GEMV = 11,   // column-split partial products of the HBM-bound GEMV
};

void set_error(const std::string& msg);
void* scratch(Handle* h, int slot, size_t bytes);  // nullptr on failure (error set)
double* pinned(Handle* h, size_t bytes);

#define CHFSI_CUDA(call)                                                            \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      ::chfsi::set_error(std::string(#call) + ": " + cudaGetErrorString(e_));      \
      return ::chfsi::ERR_CUDA;                                                     \
    }                                                                               \
  } while (0)

#define CHFSI_CHECK_LAUNCH()                                                        \
  do {                                                                              \
    cudaError_t e_ = cudaGetLastError();                                            \
    if (e_ != cudaSuccess) {                                                        \
      ::chfsi::set_error(std::string("kernel launch: ") + cudaGetErrorString(e_)); \
      return ::chfsi::ERR_CUDA;                                                     \
    }                                                                               \
  } while (0)

#define CHFSI_TRY(expr)            \
  do {                             \
    int s_ = (expr);               \
    if (s_ != ::chfsi::OK) return s_; \
  } while (0)

// ---- GEMM (zgemm.cu) ----
// C = alpha op(A) op(B) + beta C, complex128 column-major.
// tri: one triangular operand (common.cuh Tri flags); the zero blocks of the K range
// are skipped. tri_off: first row (A flags) / column (B flags) of C in the factor.
int zgemm(Handle* h, int opa, int opb, long long M, long long N, long long K, double2 alpha,
          const double2* A, long long lda, const double2* B, long long ldb, double2 beta,
          double2* C, long long ldc, int tri = 0, long long tri_off = 0);
// One fused Chebyshev degree step: C = alpha*A*Y1 + beta*Y1 + gamma*Y0 (Y0 may be null,
// C may alias Y0). A is M x M, Y1/Y0/C are M x N.
// 3M operand-sum planes (real, column-major, ld in doubles): As = Re A + Im A, Bs =
// Re B + Im B; Cs (optional) receives Re C + Im C of the step's output.
struct SumPlanes {
  const double* As; long long ldas;  // As grouped (zgemm.cuh), ldas unused
  const double* Bs; long long ldbs;
  double* Cs; long long ldcs;
};
int sum_plane(Handle* h, long long rows, long long cols, const double2* X, long long ldx,
              double* Xs, long long ldxs);
int sum_plane_grouped(Handle* h, long long rows, long long cols, const double2* X, long long ldx,
                      double* Xs);
int declare_operator(Handle* h, long long n, const double2* H, long long ldh);
// C = A B (op N x N) reading 3M sum planes (sp may be null)
int zgemm_nn_sums(Handle* h, long long M, long long N, long long K, const double2* A, long long lda,
                  const double2* B, long long ldb, double2* C, long long ldc,
                  const SumPlanes* sp);
// Y = H X; with the declared operator H (chfsi_declare_operator) the product reads H's
// sum plane and a plane of X formed here (3M without in-loop sums)
int apply_operator(Handle* h, long long n, long long k, const double2* H, long long ldh,
                   const double2* X, long long ldx, double2* Y, long long ldy);
int zgemm_filter_step(Handle* h, long long M, long long N, const double2* A, long long lda,
                      const double2* Y1, long long ld1, double alpha, double beta,
                      const double2* Y0, long long ld0, double gamma, double2* C, long long ldc,
                      const double* coef_dev = nullptr, const SumPlanes* sp = nullptr);
// Row panel of a fused step: rows [r0, r0 + M) of C = alpha*A*B + beta*Y1e + gamma*Y0
// with A = H + r0 (M x K), B the full K x N block and Y1e = B + r0.
int zgemm_filter_panel(Handle* h, long long M, long long N, long long K, const double2* A,
                       long long lda, const double2* B, long long ldb, const double2* Y1e,
                       long long ld1e, double alpha, double beta, const double2* Y0, long long ld0,
                       double gamma, double2* C, long long ldc, const double* coef_dev,
                       const SumPlanes* sp = nullptr);
// split-K workspace bytes the filter step's plan needs (pre-sized before graph capture)
size_t filter_step_workspace(Handle* h, long long M, long long N);

// Tuning hooks: force a tile config (-1 = cost model) / split-K factor (0 = auto).
int gemm_override(int cfg, int split);
void gemm_overrides(int* cfg, int* split);
int set_complex_mul(int mul);
int complex_mul();
int gemm_plan(Handle* h, int opa, int opb, int epi, long long M, long long N, long long K,
              int* cfg, int* split);

// ---- solver phases (solver_ops.cu) ----
int project_out(Handle* h, long long n, long long k, double2* F, long long ldf,
                const double2* Lk, long long ldl, long long nl);

// ---- misc kernels (kernels.cu) ----
int residual_norms(Handle* h, long long n, long long k, const double2* HY, long long ldhy,
                   const double2* Y, long long ldy, const double* lam_dev, double* res_dev);
int zdotc_cols(Handle* h, long long n, long long k, const double2* X, long long ldx,
               const double2* Y, long long ldy, double2* out_dev);
int hermitian_norms(Handle* h, long long n, const double2* A, long long lda, double* out2_dev);
int hermitize(Handle* h, long long n, double2* A, long long lda);
int mirror_lower(Handle* h, long long n, double2* A, long long lda);
int clean_lower_factor(Handle* h, long long n, double2* L, long long ldl);
int trtri_lower(Handle* h, long long n, const double2* L, long long ldl, double2* X, long long ldx);
int zaxpby_cols(Handle* h, long long n, long long k, double2 alpha, const double2* X,
                long long ldx, double2 beta, double2* Y, long long ldy);
int get_real_diag(Handle* h, long long n, const double2* A, long long lda, double* out_dev);
// y = alpha A x + beta y for a column-major M x K matrix A (HBM-bound GEMV; the
// Lanczos H v of core.py:202-256): one row per thread, the K columns split over
// blockIdx.y, partial products summed in fixed order (deterministic).
int zgemv_n(Handle* h, long long M, long long K, double2 alpha, const double2* A, long long lda,
            const double2* x, double2 beta, double2* y);
int zcopy2d(Handle* h, long long rows, long long cols, const double2* src, long long lds,
            double2* dst, long long ldd);
int shift_diag(Handle* h, long long n, double2* A, long long lda, double shift);

}  // namespace chfsi
