// cuSOLVER Hermitian eigensolver variants for the replicated k x k Rayleigh-Ritz step:
// cusolverDnZheevd vs the generic 64-bit cusolverDnXsyevd (CUDA_C_64F), time per call.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 heevd_variants.cu -lcusolver -o hv
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cuComplex.h>

int main() {
  cusolverDnHandle_t h;
  cusolverDnCreate(&h);
  cusolverDnParams_t params;
  cusolverDnCreateParams(&params);
  for (int n : {210, 550, 1100, 2200}) {
    std::vector<cuDoubleComplex> a((size_t)n * n);
    srand(1);
    for (int j = 0; j < n; ++j)
      for (int i = 0; i <= j; ++i) {
        double re = rand() / (double)RAND_MAX - 0.5, im = i == j ? 0.0 : rand() / (double)RAND_MAX - 0.5;
        a[i + (size_t)j * n] = make_cuDoubleComplex(re, im);
        a[j + (size_t)i * n] = make_cuDoubleComplex(re, -im);
      }
    cuDoubleComplex *dA, *dA0;
    double* dW;
    int* dInfo;
    cudaMalloc(&dA, sizeof(cuDoubleComplex) * n * n);
    cudaMalloc(&dA0, sizeof(cuDoubleComplex) * n * n);
    cudaMalloc(&dW, sizeof(double) * n);
    cudaMalloc(&dInfo, sizeof(int));
    cudaMemcpy(dA0, a.data(), sizeof(cuDoubleComplex) * n * n, cudaMemcpyHostToDevice);
    // zheevd
    int lwork = 0;
    cusolverDnZheevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, &lwork);
    cuDoubleComplex* work;
    cudaMalloc(&work, sizeof(cuDoubleComplex) * lwork);
    // Xsyevd
    size_t dws = 0, hws = 0;
    cusolverDnXsyevd_bufferSize(h, params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n,
                                CUDA_C_64F, dA, n, CUDA_R_64F, dW, CUDA_C_64F, &dws, &hws);
    void* dwork;
    cudaMalloc(&dwork, dws + 16);
    std::vector<char> hwork(hws + 16);
    for (int variant = 0; variant < 2; ++variant) {
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaMemcpy(dA, dA0, sizeof(cuDoubleComplex) * n * n, cudaMemcpyDeviceToDevice);
        cudaDeviceSynchronize();
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        if (variant == 0)
          cusolverDnZheevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, work, lwork, dInfo);
        else
          cusolverDnXsyevd(h, params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_C_64F, dA, n,
                           CUDA_R_64F, dW, CUDA_C_64F, dwork, dws, hwork.data(), hws, dInfo);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("n=%d %s %.2f ms\n", n, variant ? "Xsyevd" : "Zheevd", best);
    }
    cudaFree(dA); cudaFree(dA0); cudaFree(dW); cudaFree(dInfo); cudaFree(work); cudaFree(dwork);
  }
  return 0;
}
