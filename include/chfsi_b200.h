/*
 * chfsi_b200.h -- C ABI of libchfsi_b200.so, the B200 (sm_100a) ChFSI hot path.
 *
 * The reference (arxiv 1305.5120 Python package `chfsi`, /root/reference/pkg)
 * has no native FFI: its hot path calls numpy/scipy/numba. Each entry point
 * below replaces one of those calls; the comment names the reference
 * interface it stands in for (file:line under pkg/src/chfsi/). A ctypes
 * binding (paper_1305_5120_b200/_native.py) is the only
 * caller.
 *
 * Conventions
 *   - complex128 matrices are interleaved (re, im) doubles, COLUMN-MAJOR with
 *     a leading dimension `ld*` counted in complex elements: numpy F-order.
 *   - pointers named d_* are DEVICE pointers on the handle's device; h_* are
 *     host pointers. Calls that return host data synchronise the stream.
 *   - every function returns 0 on success or a negative status; the message
 *     is in chfsi_last_error() (thread-local). Status codes:
 *        -1 CHFSI_ERR_ARG       contract violation
 *        -2 CHFSI_ERR_CUDA      CUDA runtime error
 *        -3 CHFSI_ERR_CUSOLVER  cuSOLVER error
 *        -4 CHFSI_ERR_NOT_PD    Cholesky pivot failed (info = 1-based pivot)
 *        -5 CHFSI_ERR_RANK      rank collapse (bad column, 0-based)
 *        -6 CHFSI_ERR_NOMEM     device allocation failed
 *   - op codes: 0 = N (as is), 1 = C (conjugate transpose).
 */
#ifndef CHFSI_B200_H
#define CHFSI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CHFSI_ABI_VERSION 1

typedef struct chfsi_handle_s* chfsi_handle_t;

int chfsi_abi_version(void);
const char* chfsi_last_error(void);

/* Context: cuSOLVER handle, scratch arenas, stream binding (one per device). */
int chfsi_create(int device, void* stream, chfsi_handle_t* out);
int chfsi_destroy(chfsi_handle_t h);
int chfsi_set_stream(chfsi_handle_t h, void* stream);
int chfsi_synchronize(chfsi_handle_t h);
/* kernels (and cuSOLVER calls) this handle has launched; reset with reset=1 */
long long chfsi_launch_count(chfsi_handle_t h, int reset);

/* C = alpha op(A) op(B) + beta C on the FP64 tensor pipe (DMMA).
 * Replaces linalg.py:198-251 `gemm` (numpy zgemm through OpenBLAS). */
int chfsi_zgemm(chfsi_handle_t h, int opa, int opb, int64_t m, int64_t n, int64_t k,
                double alpha_re, double alpha_im, const void* d_A, int64_t lda,
                const void* d_B, int64_t ldb, double beta_re, double beta_im, void* d_C,
                int64_t ldc);

/* chfsi_zgemm with one triangular operand whose zero triangle holds zeros; the GEMM
 * skips those blocks of the K range (half the work for a square factor). Replaces
 * the ztrmm / ztrsm-via-inverse products of linalg.py:326-366 (`triangular_solve`,
 * `trmm_adjoint`) and core.py:191-195 (`back_transform`). Flags (one of):
 *   1  A lower triangular (opa = N)             4  B lower triangular (opb = N)
 *   2  op(B) = L^H, L lower (opb = C)           8  op(A) = L^H, L lower (opa = C)
 * The factor has order k; C holds its rows (flags 1, 8) or columns (2, 4)
 * [tri_offset, tri_offset + m or n): 0 for a whole factor, the shard start when a
 * rank computes a column range of L^-1 A L^-H (distributed.reduce_sharded).
 * Flag 16 (combinable): C is Hermitian (m == n) and only the tiles touching its lower
 * triangle are computed; the strictly upper part is left undefined. */
#define CHFSI_TRI_A_LOWER 1
#define CHFSI_TRI_B_UPPER 2
#define CHFSI_TRI_B_LOWER 4
#define CHFSI_TRI_A_UPPER 8
#define CHFSI_TRI_C_LOWER 16
int chfsi_zgemm_tri(chfsi_handle_t h, int opa, int opb, int64_t m, int64_t n, int64_t k,
                    double alpha_re, double alpha_im, const void* d_A, int64_t lda,
                    const void* d_B, int64_t ldb, double beta_re, double beta_im, void* d_C,
                    int64_t ldc, int tri, int64_t tri_offset);

/* Scaled degree-m Chebyshev filter p_m(H) Y, core.py:263-284 `_filter_raw`.
 * d_Y (n x k) is clobbered; the result is in d_W when *h_result_in_w == 1,
 * else in d_Y. Exactly `degree` fused GEMM launches (H streamed once each). */
int chfsi_filter(chfsi_handle_t h, int64_t n, int64_t k, int degree, double a, double b,
                 double lam_ref, const void* d_H, int64_t ldh, void* d_Y, int64_t ldy,
                 void* d_W, int64_t ldw, int* h_result_in_w);

/* The same filter when H arrives from HOST memory, core.py:287-311
 * `chebyshev_filter(H, Y, spec)` called with an ndarray H (core.py:304 `_asarray`).
 * h_H (column-major, leading dimension ldh_host >= n) is uploaded into d_H in
 * `panels` row panels (0 = automatic) on a library-owned copy stream while the first
 * degree step runs panel by panel on the handle's stream; steps 2..degree start once
 * the whole of H is resident. d_Y must already hold Y. Pinned h_H overlaps the upload
 * with the first step; pageable h_H is staged panel by panel. Returns once h_H has
 * been read (the filter may still run on the stream); d_H then holds H. */
int chfsi_filter_streamed(chfsi_handle_t h, int64_t n, int64_t k, int degree, double a,
                          double b, double lam_ref, const void* h_H, int64_t ldh_host, void* d_H,
                          int64_t ldh, void* d_Y, int64_t ldy, void* d_W, int64_t ldw, int panels,
                          int* h_result_in_w);

/* chfsi_filter_streamed that also returns the result to the host: the last degree step
 * runs by row panels and each panel of p_m(H) Y is copied to h_out (column-major,
 * ld_out >= n; page-locked for full speed) while the next panel computes. Returns once
 * the result is in h_out (the whole of `chebyshev_filter(ndarray H, ndarray Y, spec)`,
 * core.py:287-311, host to host; d_Y / d_W still hold the device result as flagged). */
int chfsi_filter_streamed_to_host(chfsi_handle_t h, int64_t n, int64_t k, int degree, double a,
                                  double b, double lam_ref, const void* h_H, int64_t ldh_host,
                                  void* d_H, int64_t ldh, void* d_Y, int64_t ldy, void* d_W,
                                  int64_t ldw, int panels, void* h_out, int64_t ld_out,
                                  int* h_result_in_w);

/* One fused degree step C = alpha H Y1 + beta Y1 + gamma Y0 (Y0 may be NULL and may
 * alias C); the unit the filter roofline is measured on (core.py:280-281). */
int chfsi_filter_step(chfsi_handle_t h, int64_t n, int64_t k, const void* d_H, int64_t ldh,
                      const void* d_Y1, int64_t ld1, double alpha, double beta,
                      const void* d_Y0, int64_t ld0, double gamma, void* d_C, int64_t ldc);

/* k-step Lanczos with full reorthogonalisation, core.py:202-256
 * `lanczos_upper_bound`. d_v0 = normalised start vector (drawn by the caller
 * from the reference's Generator stream). Returns alphas/betas (length >= k),
 * the steps taken and b = lambda_max(T) + beta_last + 4 j eps max|lambda(T)|. */
int chfsi_lanczos_bound(chfsi_handle_t h, int64_t n, int k, const void* d_H, int64_t ldh,
                        const void* d_v0, double* h_alphas, double* h_betas, int* h_steps,
                        double* h_bound);

/* core.py:365-382 `_qr_against_locked` (+ linalg.py:273-289 rank test):
 * F <- F - L (L^H F) twice (CGS2), then Q = CholQR2(F) (shifted CholQR3 if the
 * first Cholesky breaks down). d_T is an n x k work block. Returns
 * CHFSI_ERR_RANK with *h_bad_col = first column whose |R_jj| < rank_tol*||F||_F.
 * *h_fro = ||F||_F after projection. */
int chfsi_orthonormalize(chfsi_handle_t h, int64_t n, int64_t k, void* d_F, int64_t ldf,
                         const void* d_L, int64_t ldl, int64_t nl, void* d_T, int64_t ldt,
                         void* d_Q, int64_t ldq, double rank_tol, int64_t* h_bad_col,
                         double* h_fro);

/* core.py:318-330 `_rr_raw`: HQ = H Q, G = Q^H HQ, G <- (G+G^H)/2, (w, W) = eig(G)
 * (cuSOLVER zheevd, ascending), Z = Q W, HZ = HQ W. Ritz values to h_w (k); when h_res
 * is not NULL also the residual norms ||HZ_j - w_j Z_j|| of core.py:477 (one host sync). */
int chfsi_rayleigh_ritz(chfsi_handle_t h, int64_t n, int64_t k, const void* d_H, int64_t ldh,
                        const void* d_Q, int64_t ldq, void* d_HQ, int64_t ldhq, void* d_Z,
                        int64_t ldz, void* d_HZ, int64_t ldhz, double* h_w, double* h_res);

/* Rayleigh-Ritz when the caller already holds HQ = H Q (column-sharded multi-GPU
 * path: each rank computes H Q_p on its shard, then all-gathers HQ). */
int chfsi_rayleigh_ritz_from_hq(chfsi_handle_t h, int64_t n, int64_t k, const void* d_Q,
                                int64_t ldq, const void* d_HQ, int64_t ldhq, void* d_Z,
                                int64_t ldz, void* d_HZ, int64_t ldhz, double* h_w,
                                double* h_res);

/* F <- F - L (L^H F), twice (CGS2): the projection half of core.py:371-372. Column-local,
 * so sharded callers run it on their own columns before the all-gather. */
int chfsi_project_out(chfsi_handle_t h, int64_t n, int64_t k, void* d_F, int64_t ldf,
                      const void* d_L, int64_t ldl, int64_t nl);

/* r_j = ||HY_j - lam_j Y_j||_2, core.py:347-358 `residuals` and core.py:477. */
int chfsi_residual_norms(chfsi_handle_t h, int64_t n, int64_t k, const void* d_HY, int64_t ldhy,
                         const void* d_Y, int64_t ldy, const double* h_lam, double* h_res);

/* linalg.py:104-121 HermitianDenseMatrix: h_out[0] = ||A||_F, h_out[1] = ||A - A^H||_F. */
int chfsi_hermitian_norms(chfsi_handle_t h, int64_t n, const void* d_A, int64_t lda,
                          double* h_out);
/* A <- (A + A^H)/2 with a real diagonal (linalg.py:114-115). */
int chfsi_hermitize(chfsi_handle_t h, int64_t n, void* d_A, int64_t lda);

/* linalg.py:254-270 `cholesky_factor`: in-place lower Cholesky (cuSOLVER zpotrf),
 * upper triangle zeroed and diagonal made real. *h_info = failing pivot (1-based) or 0. */
int chfsi_cholesky(chfsi_handle_t h, int64_t n, void* d_A, int64_t lda, int* h_info);

/* X = L^-1 for lower-triangular L (blocked recursive inverse on the DMMA GEMM);
 * building block of linalg.py:326-366 `triangular_solve` / `trmm_adjoint`. */
int chfsi_trtri_lower(chfsi_handle_t h, int64_t n, const void* d_L, int64_t ldl, void* d_X,
                      int64_t ldx);

/* The replicated k x k step of a column-sharded CholQR pass (the multi-GPU form of
 * core.py:365-382 `_qr_against_locked`, distributed.ShardedPhases): G <- (G + G^H)/2
 * (+ shift I); *h_trace = trace(G); G = L L^H in place (zpotrf, lower); d_Li = L^-1;
 * h_diag[k] = diag(L); *h_info = zpotrf info (0, or the 1-based failing pivot). */
int chfsi_cholesky_inverse(chfsi_handle_t h, int64_t k, void* d_G, int64_t ldg, double shift,
                           void* d_Li, int64_t ldli, double* h_diag, double* h_trace,
                           int* h_info);

/* core.py:172-188 `reduce_to_standard`: H = L^-1 A L^-H given d_Linv = L^-1 (lower
 * triangular with a zero upper triangle, e.g. from chfsi_trtri_lower). Two DMMA GEMMs
 * that skip the zero triangle of Linv; d_W is an n x n work block. H is not
 * re-symmetrised here (chfsi_hermitian_norms / chfsi_hermitize do that). */
int chfsi_reduce_to_standard(chfsi_handle_t h, int64_t n, const void* d_A, int64_t lda,
                             const void* d_Linv, int64_t ldli, void* d_W, int64_t ldw, void* d_H,
                             int64_t ldh);

/* Full Hermitian eigendecomposition in place (cuSOLVER zheevd), ascending.
 * Stands in for linalg.py:292-323 `oracle_eig` / `_jacobi_raw` on the device. */
int chfsi_heevd(chfsi_handle_t h, int64_t n, void* d_A, int64_t lda, double* h_w);

/* Y = alpha X + beta Y on an n x k block (X may be NULL). */
int chfsi_axpby(chfsi_handle_t h, int64_t n, int64_t k, double alpha_re, double alpha_im,
                const void* d_X, int64_t ldx, double beta_re, double beta_im, void* d_Y,
                int64_t ldy);

/* Tuning hooks (process-wide): force GEMM tile config `cfg` (-1 = cost model) and
 * split-K factor (0 = automatic); query the plan the cost model picks for a shape
 * (filter_epilogue: 0 plain product, 1 fused filter step, 2 fused filter step of a
 * chfsi_filter call, which supplies 3M operand-sum planes). */
int chfsi_gemm_override(int cfg, int split);
int chfsi_gemm_plan(chfsi_handle_t h, int opa, int opb, int filter_epilogue, int64_t m,
                    int64_t n, int64_t k, int* h_cfg, int* h_split);

/* Complex-product scheme of the op N x N (TMA) GEMMs, process-wide: 3 = 3M (three real
 * DMMA products per complex multiply-add: Ar Br, Ai Bi, (Ar+Ai)(Br+Bi); default) or
 * 4 = four real products. Replaces the inner kernel of linalg.py:198-251 `gemm`
 * (numpy/OpenBLAS zgemm). Environment CHFSI_COMPLEX_MUL=4 selects 4 at load time.
 * chfsi_get_complex_mul returns the current scheme. */
int chfsi_set_complex_mul(int mul);
int chfsi_get_complex_mul(void);

/* Declare the n x n device operator d_H unchanged until the next declaration on this
 * handle (d_H = NULL clears): its 3M sum plane (Re H + Im H, n^2 doubles of handle
 * scratch) is computed once here and reused by every chfsi_filter call on the same
 * (d_H, n, ldh) instead of once per call. A solve declares H for its duration
 * (core.py:385-546 `chfsi_solve` filters the same H every outer iteration). Writing H
 * while declared, without re-declaring, gives wrong filter results. */
int chfsi_declare_operator(chfsi_handle_t h, int64_t n, const void* d_H, int64_t ldh);

/* Y = H X for an n x n operator and an n x k block (core.py:318-330 `_rr_raw`'s H Q,
 * the re-check H V of core.py:532-544). On the declared operator (above) the product
 * reads H's 3M sum plane; otherwise it is chfsi_zgemm(N, N). */
int chfsi_apply_operator(chfsi_handle_t h, int64_t n, int64_t k, const void* d_H, int64_t ldh,
                         const void* d_X, int64_t ldx, void* d_Y, int64_t ldy);

/* Microbenchmarks that give the roofline denominators on the box:
 * FP64 tensor-pipe (DMMA) and FP64 FMA-pipe (DFMA) peak, TFLOP/s. */
int chfsi_peak_dmma(int device, int iters, double* h_tflops);
int chfsi_peak_dfma(int device, int iters, double* h_tflops);

/* Upload a rows x cols column-major complex block from host memory (ld_src) to the
 * device (ld_dst) on the handle's stream -- the H2D half of every drop-in call that
 * passes numpy arrays (core.py:287-311, :385; linalg.py:89-93 `_asarray`). Page-locked
 * sources take one async 2-D copy; pageable ones go through the handle's pinned staging
 * ring, filled by a host worker pool while the DMA engine drains the previous slot
 * (CHFSI_STAGE_MB per slot, CHFSI_STAGE_THREADS workers). Returns once the source has
 * been read; the device copy completes in stream order. chfsi_filter_streamed uses the
 * same path for the panels of a pageable H. */
int chfsi_upload(chfsi_handle_t h, const void* h_src, int64_t ld_src, int64_t rows,
                 int64_t cols, void* d_dst, int64_t ld_dst);

/* In-process multi-GPU (SURVEY.md section 8b `chfsi_ctx_create(ndev, devices)`): one
 * NCCL clique over `ndev` distinct GPUs of this process (ncclCommInitAll), one rank per
 * device, each driven by its own host thread. The reference takes its parallelism
 * in-process (linalg.py:49-64 `set_workers`, the column tiles of linalg.py:238-243);
 * here the filter columns are sharded over the clique (H replicated) and the shards are
 * all-gathered for QR and Rayleigh-Ritz (distributed.py). NCCL is dlopen'ed at first
 * use; chfsi_comm_available() reports whether it loads (and its version code). */
typedef struct chfsi_comm_s* chfsi_comm_t;
int chfsi_comm_available(int* h_version);
int chfsi_comm_init_all(int ndev, const int* h_devices, chfsi_comm_t* h_out);
int chfsi_comm_destroy(chfsi_comm_t c);
int chfsi_comm_abort(chfsi_comm_t c);
/* d_recv (world * bytes) <- every rank's d_send (bytes) in rank order, on `stream` */
int chfsi_comm_allgather(chfsi_comm_t c, const void* d_send, void* d_recv, size_t bytes,
                         void* stream);
int chfsi_comm_broadcast(chfsi_comm_t c, void* d_buf, size_t bytes, int root, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CHFSI_B200_H */
