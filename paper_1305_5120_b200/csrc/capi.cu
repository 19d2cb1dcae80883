// extern "C" boundary of libchfsi_b200.so (declared in include/chfsi_b200.h).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "../../include/chfsi_b200.h"
#include "common.cuh"
#include "internal.h"

namespace chfsi {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

void* scratch(Handle* h, int slot, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (h->scratch_bytes[slot] >= bytes) return h->scratch[slot];
  if (h->scratch[slot]) {
    cudaStreamSynchronize(h->stream);
    cudaFree(h->scratch[slot]);
    h->scratch[slot] = nullptr;
    h->scratch_bytes[slot] = 0;
  }
  const size_t want = bytes + bytes / 4;  // grow with headroom
  if (cudaMalloc(&h->scratch[slot], want) != cudaSuccess) {
    cudaGetLastError();
    if (cudaMalloc(&h->scratch[slot], bytes) != cudaSuccess) {
      cudaGetLastError();
      set_error("scratch allocation of " + std::to_string(bytes) + " bytes failed");
      h->scratch[slot] = nullptr;
      return nullptr;
    }
    h->scratch_bytes[slot] = bytes;
    return h->scratch[slot];
  }
  h->scratch_bytes[slot] = want;
  return h->scratch[slot];
}

double* pinned(Handle* h, size_t bytes) {
  if (h->h_pinned_bytes >= bytes) return h->h_pinned;
  if (h->h_pinned) cudaFreeHost(h->h_pinned);
  h->h_pinned = nullptr;
  h->h_pinned_bytes = 0;
  if (cudaMallocHost(&h->h_pinned, bytes) != cudaSuccess) {
    cudaGetLastError();
    set_error("pinned allocation failed");
    return nullptr;
  }
  h->h_pinned_bytes = bytes;
  return h->h_pinned;
}

// forward declarations from solver_ops.cu
int potrf_lower(Handle* h, long long n, double2* A, long long lda, int* info_host);
int heevd(Handle* h, long long n, double2* A, long long lda, double* w_dev);
int filter(Handle* h, long long n, long long k, int degree, double a, double b, double lam_ref,
           const double2* H, long long ldh, double2* Y, long long ldy, double2* W, long long ldw,
           int* result_in_w);
int filter_streamed(Handle* h, long long n, long long k, int degree, double a, double b,
                    double lam_ref, const double2* H_host, long long ldh_host, double2* H,
                    long long ldh, double2* Y, long long ldy, double2* W, long long ldw,
                    int panels, int* result_in_w, double2* out_host, long long ld_out);
int cholesky_inverse(Handle* h, long long k, double2* G, long long ldg, double shift,
                     double2* Li, long long ldli, double* diag_host, double* trace_host,
                     int* info_host);
int reduce_to_standard(Handle* h, long long n, const double2* A, long long lda,
                       const double2* Linv, long long ldli, double2* W, long long ldw,
                       double2* H, long long ldh);
int lanczos_bound(Handle* h, long long n, int k, const double2* H, long long ldh,
                  const double2* v0, double* alphas, double* betas, int* steps, double* bound);
int orthonormalize(Handle* h, long long n, long long k, double2* F, long long ldf,
                   const double2* Lk, long long ldl, long long nl, double2* T, long long ldt,
                   double2* Q, long long ldq, double rank_rel_tol, long long* bad_col,
                   double* fro_out);
int rayleigh_ritz(Handle* h, long long n, long long k, const double2* H, long long ldh,
                  const double2* Q, long long ldq, double2* HQ, long long ldhq, double2* Z,
                  long long ldz, double2* HZ, long long ldhz, double* w_host, double* res_host,
                  bool hq_ready);
int project_out(Handle* h, long long n, long long k, double2* F, long long ldf,
                const double2* Lk, long long ldl, long long nl);

// ---------------------------------------------------------------- peaks
// Register-resident 4 x 4 block of independent 8x8 accumulators fed by 4 A and
// 4 B fragments, the same operand reuse as a GEMM warp tile (16 DMMA/iteration).
__global__ void peak_dmma_kernel(int iters, double* out) {
  double acc[4][4][2];
  double a[4], b[4];
  #pragma unroll
  for (int i = 0; i < 4; ++i) {
    a[i] = 1.0 + 1e-9 * (threadIdx.x + i);
    b[i] = 1.0 - 1e-9 * (threadIdx.x + 3 * i);
    #pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 1e-3 * (i + 4 * j);
  }
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < 4; ++i)
      #pragma unroll
      for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
  double s = 0.0;
  #pragma unroll
  for (int i = 0; i < 4; ++i)
    #pragma unroll
    for (int j = 0; j < 4; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 123.456) out[0] = s;  // defeat dead-code elimination
}

__global__ void peak_dfma_kernel(int iters, double* out) {
  constexpr int U = 16;
  double acc[U];
  #pragma unroll
  for (int u = 0; u < U; ++u) acc[u] = 1e-3 * (threadIdx.x + u);
  const double a = 1.0 + 1e-9 * threadIdx.x, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = fma(acc[u], a, b);
  }
  double s = 0.0;
  #pragma unroll
  for (int u = 0; u < U; ++u) s += acc[u];
  if (s == 123.456) out[0] = s;
}

template <class K>
static int time_peak(int device, K kernel, int iters, double flops_per_thread_iter,
                     double* tflops) {
  CHFSI_CUDA(cudaSetDevice(device));
  int sms = 0;
  CHFSI_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  double* out = nullptr;
  CHFSI_CUDA(cudaMalloc(&out, sizeof(double)));
  const int threads = 256, blocks = sms * 4;
  cudaEvent_t e0, e1;
  CHFSI_CUDA(cudaEventCreate(&e0));
  CHFSI_CUDA(cudaEventCreate(&e1));
  kernel<<<blocks, threads>>>(iters / 4 + 1, out);  // warm-up
  CHFSI_CHECK_LAUNCH();
  CHFSI_CUDA(cudaEventRecord(e0));
  kernel<<<blocks, threads>>>(iters, out);
  CHFSI_CUDA(cudaEventRecord(e1));
  CHFSI_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  CHFSI_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  const double flops = (double)blocks * threads * iters * flops_per_thread_iter;
  *tflops = flops / (ms * 1e-3) / 1e12;
  return OK;
}

}  // namespace chfsi

using namespace chfsi;

struct chfsi_handle_s : public Handle {};

#define H_CHECK(h)                          \
  do {                                      \
    if (!(h)) {                             \
      set_error("null chfsi handle");       \
      return ERR_ARG;                       \
    }                                       \
    cudaSetDevice((h)->device);             \
  } while (0)

static inline double2 c2(double re, double im) { return make_double2(re, im); }

extern "C" {

int chfsi_abi_version(void) { return CHFSI_ABI_VERSION; }

const char* chfsi_last_error(void) { return g_last_error.c_str(); }

int chfsi_create(int device, void* stream, chfsi_handle_t* out) {
  if (!out) {
    set_error("chfsi_create: null out");
    return ERR_ARG;
  }
  *out = nullptr;
  CHFSI_CUDA(cudaSetDevice(device));
  auto* h = new chfsi_handle_s();
  h->device = device;
  h->stream = (cudaStream_t)stream;
  cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (cusolverDnCreate(&h->solver) != CUSOLVER_STATUS_SUCCESS) {
    delete h;
    set_error("cusolverDnCreate failed");
    return ERR_CUSOLVER;
  }
  cusolverDnSetStream(h->solver, h->stream);
  if (cudaMalloc(&h->d_info, sizeof(int)) != cudaSuccess) {
    cusolverDnDestroy(h->solver);
    delete h;
    set_error("cudaMalloc(info) failed");
    return ERR_NOMEM;
  }
  *out = h;
  return OK;
}

int chfsi_destroy(chfsi_handle_t h) {
  if (!h) return OK;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  destroy_filter_graphs(h);
  destroy_copy_stream(h);
  destroy_stager(h);
  if (h->capture_stream) cudaStreamDestroy(h->capture_stream);
  for (int i = 0; i < Handle::kSlots; ++i)
    if (h->scratch[i]) cudaFree(h->scratch[i]);
  if (h->d_info) cudaFree(h->d_info);
  if (h->h_pinned) cudaFreeHost(h->h_pinned);
  if (h->solver) cusolverDnDestroy(h->solver);
  delete h;
  return OK;
}

int chfsi_set_stream(chfsi_handle_t h, void* stream) {
  H_CHECK(h);
  h->stream = (cudaStream_t)stream;
  cusolverDnSetStream(h->solver, h->stream);
  return OK;
}

int chfsi_synchronize(chfsi_handle_t h) {
  H_CHECK(h);
  CHFSI_CUDA(cudaStreamSynchronize(h->stream));
  return OK;
}

long long chfsi_launch_count(chfsi_handle_t h, int reset) {
  if (!h) return -1;
  const long long c = h->launches;
  if (reset) h->launches = 0;
  return c;
}

int chfsi_zgemm(chfsi_handle_t h, int opa, int opb, int64_t m, int64_t n, int64_t k,
                double alpha_re, double alpha_im, const void* d_A, int64_t lda, const void* d_B,
                int64_t ldb, double beta_re, double beta_im, void* d_C, int64_t ldc) {
  H_CHECK(h);
  if (m < 0 || n < 0 || k < 0) {
    set_error("chfsi_zgemm: negative dimension");
    return ERR_ARG;
  }
  return zgemm(h, opa, opb, m, n, k, c2(alpha_re, alpha_im), (const double2*)d_A, lda,
               (const double2*)d_B, ldb, c2(beta_re, beta_im), (double2*)d_C, ldc);
}

int chfsi_zgemm_tri(chfsi_handle_t h, int opa, int opb, int64_t m, int64_t n, int64_t k,
                    double alpha_re, double alpha_im, const void* d_A, int64_t lda,
                    const void* d_B, int64_t ldb, double beta_re, double beta_im, void* d_C,
                    int64_t ldc, int tri, int64_t tri_offset) {
  H_CHECK(h);
  if (m < 0 || n < 0 || k < 0) {
    set_error("chfsi_zgemm_tri: negative dimension");
    return ERR_ARG;
  }
  return zgemm(h, opa, opb, m, n, k, c2(alpha_re, alpha_im), (const double2*)d_A, lda,
               (const double2*)d_B, ldb, c2(beta_re, beta_im), (double2*)d_C, ldc, tri,
               tri_offset);
}

int chfsi_filter(chfsi_handle_t h, int64_t n, int64_t k, int degree, double a, double b,
                 double lam_ref, const void* d_H, int64_t ldh, void* d_Y, int64_t ldy, void* d_W,
                 int64_t ldw, int* h_result_in_w) {
  H_CHECK(h);
  if (!(a < b)) {
    set_error("filter interval requires a < b");
    return ERR_ARG;
  }
  return filter(h, n, k, degree, a, b, lam_ref, (const double2*)d_H, ldh, (double2*)d_Y, ldy,
                (double2*)d_W, ldw, h_result_in_w);
}

int chfsi_upload(chfsi_handle_t h, const void* h_src, int64_t ld_src, int64_t rows,
                 int64_t cols, void* d_dst, int64_t ld_dst) {
  H_CHECK(h);
  if ((!h_src || !d_dst) && rows > 0 && cols > 0) {
    set_error("chfsi_upload: null pointer");
    return ERR_ARG;
  }
  CHFSI_TRY(upload_2d(h, (const double2*)h_src, ld_src, rows, cols, (double2*)d_dst, ld_dst,
                      h->stream));
  // a page-locked source is read by the DMA engine asynchronously: return only once it
  // has been, so the caller may free or overwrite it (the staged path already has)
  if (host_is_pinned(h_src)) CHFSI_CUDA(cudaStreamSynchronize(h->stream));
  return OK;
}

int chfsi_filter_streamed(chfsi_handle_t h, int64_t n, int64_t k, int degree, double a,
                          double b, double lam_ref, const void* h_H, int64_t ldh_host, void* d_H,
                          int64_t ldh, void* d_Y, int64_t ldy, void* d_W, int64_t ldw, int panels,
                          int* h_result_in_w) {
  H_CHECK(h);
  if (!(a < b)) {
    set_error("filter interval requires a < b");
    return ERR_ARG;
  }
  if (!h_H || !d_H) {
    set_error("filter_streamed: null H");
    return ERR_ARG;
  }
  return filter_streamed(h, n, k, degree, a, b, lam_ref, (const double2*)h_H, ldh_host,
                         (double2*)d_H, ldh, (double2*)d_Y, ldy, (double2*)d_W, ldw, panels,
                         h_result_in_w, nullptr, 0);
}

int chfsi_filter_streamed_to_host(chfsi_handle_t h, int64_t n, int64_t k, int degree, double a,
                                  double b, double lam_ref, const void* h_H, int64_t ldh_host,
                                  void* d_H, int64_t ldh, void* d_Y, int64_t ldy, void* d_W,
                                  int64_t ldw, int panels, void* h_out, int64_t ld_out,
                                  int* h_result_in_w) {
  H_CHECK(h);
  if (!(a < b)) {
    set_error("filter interval requires a < b");
    return ERR_ARG;
  }
  if (!h_H || !d_H || !h_out) {
    set_error("filter_streamed_to_host: null H or output");
    return ERR_ARG;
  }
  return filter_streamed(h, n, k, degree, a, b, lam_ref, (const double2*)h_H, ldh_host,
                         (double2*)d_H, ldh, (double2*)d_Y, ldy, (double2*)d_W, ldw, panels,
                         h_result_in_w, (double2*)h_out, ld_out);
}

int chfsi_filter_step(chfsi_handle_t h, int64_t n, int64_t k, const void* d_H, int64_t ldh,
                      const void* d_Y1, int64_t ld1, double alpha, double beta, const void* d_Y0,
                      int64_t ld0, double gamma, void* d_C, int64_t ldc) {
  H_CHECK(h);
  return zgemm_filter_step(h, n, k, (const double2*)d_H, ldh, (const double2*)d_Y1, ld1, alpha,
                           beta, (const double2*)d_Y0, ld0, gamma, (double2*)d_C, ldc);
}

int chfsi_lanczos_bound(chfsi_handle_t h, int64_t n, int k, const void* d_H, int64_t ldh,
                        const void* d_v0, double* h_alphas, double* h_betas, int* h_steps,
                        double* h_bound) {
  H_CHECK(h);
  return lanczos_bound(h, n, k, (const double2*)d_H, ldh, (const double2*)d_v0, h_alphas,
                       h_betas, h_steps, h_bound);
}

int chfsi_orthonormalize(chfsi_handle_t h, int64_t n, int64_t k, void* d_F, int64_t ldf,
                         const void* d_L, int64_t ldl, int64_t nl, void* d_T, int64_t ldt,
                         void* d_Q, int64_t ldq, double rank_tol, int64_t* h_bad_col,
                         double* h_fro) {
  H_CHECK(h);
  long long bad = -1;
  double fro = 0.0;
  const int st = orthonormalize(h, n, k, (double2*)d_F, ldf, (const double2*)d_L, ldl, nl,
                                (double2*)d_T, ldt, (double2*)d_Q, ldq, rank_tol, &bad, &fro);
  if (h_bad_col) *h_bad_col = bad;
  if (h_fro) *h_fro = fro;
  return st;
}

int chfsi_rayleigh_ritz(chfsi_handle_t h, int64_t n, int64_t k, const void* d_H, int64_t ldh,
                        const void* d_Q, int64_t ldq, void* d_HQ, int64_t ldhq, void* d_Z,
                        int64_t ldz, void* d_HZ, int64_t ldhz, double* h_w, double* h_res) {
  H_CHECK(h);
  if (k <= 0) return OK;
  return rayleigh_ritz(h, n, k, (const double2*)d_H, ldh, (const double2*)d_Q, ldq,
                       (double2*)d_HQ, ldhq, (double2*)d_Z, ldz, (double2*)d_HZ, ldhz, h_w, h_res,
                       false);
}

int chfsi_rayleigh_ritz_from_hq(chfsi_handle_t h, int64_t n, int64_t k, const void* d_Q,
                                int64_t ldq, const void* d_HQ, int64_t ldhq, void* d_Z,
                                int64_t ldz, void* d_HZ, int64_t ldhz, double* h_w,
                                double* h_res) {
  H_CHECK(h);
  if (k <= 0) return OK;
  return rayleigh_ritz(h, n, k, nullptr, 0, (const double2*)d_Q, ldq, (double2*)d_HQ, ldhq,
                       (double2*)d_Z, ldz, (double2*)d_HZ, ldhz, h_w, h_res, true);
}

int chfsi_project_out(chfsi_handle_t h, int64_t n, int64_t k, void* d_F, int64_t ldf,
                      const void* d_L, int64_t ldl, int64_t nl) {
  H_CHECK(h);
  return project_out(h, n, k, (double2*)d_F, ldf, (const double2*)d_L, ldl, nl);
}

int chfsi_residual_norms(chfsi_handle_t h, int64_t n, int64_t k, const void* d_HY, int64_t ldhy,
                         const void* d_Y, int64_t ldy, const double* h_lam, double* h_res) {
  H_CHECK(h);
  if (k <= 0) return OK;
  double* v = (double*)scratch(h, SLOT_VEC, (size_t)(2 * k + 8) * sizeof(double));
  if (!v) return ERR_NOMEM;
  CHFSI_CUDA(cudaMemcpyAsync(v, h_lam, k * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  CHFSI_TRY(residual_norms(h, n, k, (const double2*)d_HY, ldhy, (const double2*)d_Y, ldy, v,
                           v + k));
  CHFSI_CUDA(cudaMemcpyAsync(h_res, v + k, k * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CHFSI_CUDA(cudaStreamSynchronize(h->stream));
  return OK;
}

int chfsi_hermitian_norms(chfsi_handle_t h, int64_t n, const void* d_A, int64_t lda,
                          double* h_out) {
  H_CHECK(h);
  double* v = (double*)scratch(h, SLOT_VEC, 8 * sizeof(double));
  if (!v) return ERR_NOMEM;
  CHFSI_TRY(hermitian_norms(h, n, (const double2*)d_A, lda, v));
  double tmp[2];
  CHFSI_CUDA(cudaMemcpyAsync(tmp, v, 2 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CHFSI_CUDA(cudaStreamSynchronize(h->stream));
  h_out[0] = std::sqrt(tmp[0]);
  h_out[1] = std::sqrt(tmp[1]);
  return OK;
}

int chfsi_hermitize(chfsi_handle_t h, int64_t n, void* d_A, int64_t lda) {
  H_CHECK(h);
  return hermitize(h, n, (double2*)d_A, lda);
}

int chfsi_cholesky(chfsi_handle_t h, int64_t n, void* d_A, int64_t lda, int* h_info) {
  H_CHECK(h);
  int info = 0;
  CHFSI_TRY(potrf_lower(h, n, (double2*)d_A, lda, &info));
  *h_info = info;
  if (info != 0) return OK;  // caller maps info > 0 to NotPositiveDefinite(pivot)
  CHFSI_TRY(clean_lower_factor(h, n, (double2*)d_A, lda));
  return OK;
}

int chfsi_cholesky_inverse(chfsi_handle_t h, int64_t k, void* d_G, int64_t ldg, double shift,
                           void* d_Li, int64_t ldli, double* h_diag, double* h_trace,
                           int* h_info) {
  H_CHECK(h);
  if (k < 0 || ldg < k || ldli < k) {
    set_error("cholesky_inverse: bad order or leading dimension");
    return ERR_ARG;
  }
  return cholesky_inverse(h, k, (double2*)d_G, ldg, shift, (double2*)d_Li, ldli, h_diag,
                          h_trace, h_info);
}

int chfsi_reduce_to_standard(chfsi_handle_t h, int64_t n, const void* d_A, int64_t lda,
                             const void* d_Linv, int64_t ldli, void* d_W, int64_t ldw, void* d_H,
                             int64_t ldh) {
  H_CHECK(h);
  if (n < 0 || lda < n || ldli < n || ldw < n || ldh < n) {
    set_error("reduce_to_standard: bad order or leading dimension");
    return ERR_ARG;
  }
  return reduce_to_standard(h, n, (const double2*)d_A, lda, (const double2*)d_Linv, ldli,
                            (double2*)d_W, ldw, (double2*)d_H, ldh);
}

int chfsi_trtri_lower(chfsi_handle_t h, int64_t n, const void* d_L, int64_t ldl, void* d_X,
                      int64_t ldx) {
  H_CHECK(h);
  return trtri_lower(h, n, (const double2*)d_L, ldl, (double2*)d_X, ldx);
}

int chfsi_heevd(chfsi_handle_t h, int64_t n, void* d_A, int64_t lda, double* h_w) {
  H_CHECK(h);
  double* w = (double*)scratch(h, SLOT_VEC, (size_t)(n + 8) * sizeof(double));
  if (!w) return ERR_NOMEM;
  CHFSI_TRY(heevd(h, n, (double2*)d_A, lda, w));
  CHFSI_CUDA(cudaMemcpyAsync(h_w, w, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CHFSI_CUDA(cudaStreamSynchronize(h->stream));
  return OK;
}

int chfsi_axpby(chfsi_handle_t h, int64_t n, int64_t k, double alpha_re, double alpha_im,
                const void* d_X, int64_t ldx, double beta_re, double beta_im, void* d_Y,
                int64_t ldy) {
  H_CHECK(h);
  return zaxpby_cols(h, n, k, c2(alpha_re, alpha_im), (const double2*)d_X, ldx,
                     c2(beta_re, beta_im), (double2*)d_Y, ldy);
}

int chfsi_gemm_override(int cfg, int split) { return gemm_override(cfg, split); }

int chfsi_set_complex_mul(int mul) { return set_complex_mul(mul); }

int chfsi_declare_operator(chfsi_handle_t h, int64_t n, const void* d_H, int64_t ldh) {
  H_CHECK(h);
  return declare_operator(h, n, (const double2*)d_H, ldh);
}

int chfsi_apply_operator(chfsi_handle_t h, int64_t n, int64_t k, const void* d_H, int64_t ldh,
                         const void* d_X, int64_t ldx, void* d_Y, int64_t ldy) {
  H_CHECK(h);
  if (n < 0 || k < 0 || ldh < std::max<int64_t>(1, n) || ldx < std::max<int64_t>(1, n) ||
      ldy < std::max<int64_t>(1, n)) {
    set_error("apply_operator: bad dimensions");
    return ERR_ARG;
  }
  return apply_operator(h, n, k, (const double2*)d_H, ldh, (const double2*)d_X, ldx,
                        (double2*)d_Y, ldy);
}

int chfsi_get_complex_mul(void) { return complex_mul(); }

int chfsi_gemm_plan(chfsi_handle_t h, int opa, int opb, int filter_epilogue, int64_t m, int64_t n,
                    int64_t k, int* h_cfg, int* h_split) {
  H_CHECK(h);
  return gemm_plan(h, opa, opb, filter_epilogue < 0 ? 0 : std::min(filter_epilogue, 2), m, n, k,
                   h_cfg, h_split);
}

int chfsi_peak_dmma(int device, int iters, double* h_tflops) {
  // 16 DMMA.8x8x4 per thread-iteration, each 512 flop per warp => 16*512/32 per thread
  return time_peak(device, peak_dmma_kernel, iters, 16.0 * 512.0 / 32.0, h_tflops);
}

int chfsi_peak_dfma(int device, int iters, double* h_tflops) {
  return time_peak(device, peak_dfma_kernel, iters, 16.0 * 2.0, h_tflops);
}

}  // extern "C"
