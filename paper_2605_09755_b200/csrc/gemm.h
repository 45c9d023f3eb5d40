// Internal GEMM entry points shared by the dispatcher (gemm_dispatch.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace skp {

template <typename T>
int gemm_simt(int ta, int tb, int64_t M, int64_t N, int64_t K, T alpha, const T* A, int64_t lda,
              const T* B, int64_t ldb, T beta, T* C, int64_t ldc, void* ws, int64_t ws_bytes,
              cudaStream_t st);
int64_t gemm_simt_ws_bytes(int64_t M, int64_t N, int64_t K, int elem);

// FP64 on the DMMA tensor cores (gemm_dmma.cu)
int gemm_dmma(int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
              int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
              void* ws, int64_t ws_bytes, cudaStream_t st);
int64_t gemm_dmma_ws_bytes(int64_t M, int64_t N, int64_t K);
int gram_dmma_f32(const float* X, int64_t K, int64_t C, int64_t ldx, double* G, int64_t ldg,
                  void* ws, int64_t ws_bytes, cudaStream_t st);
int64_t gram_dmma_ws_bytes(int64_t K, int64_t C);

// tcgen05 3xTF32 path (gemm_tc.cu).  Returns SKP_ERR_UNSUPPORTED when the
// shape/layout is outside what the kernel handles (caller falls back).
bool tc_available();
int gemm_tc_3xtf32(int ta, int tb, int64_t M, int64_t N, int64_t K, float alpha, const float* A,
                   int64_t lda, const float* B, int64_t ldb, float beta, float* C, int64_t ldc,
                   void* ws, int64_t ws_bytes, cudaStream_t st);
int64_t gemm_tc_ws_bytes(int ta, int tb, int64_t M, int64_t N, int64_t K);

}  // namespace skp
