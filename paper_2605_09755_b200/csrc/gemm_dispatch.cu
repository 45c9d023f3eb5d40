// skp_gemm_* C-ABI: argument checks and dispatch: FP32 to the tcgen05 3xTF32
// kernel (or the SIMT kernel for exact-FP32 mode), FP64 to the DMMA kernel.
#include "common.cuh"
#include "gemm.h"

using namespace skp;

namespace {
int check(int ta, int tb, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldc,
          const void* A, const void* B, const void* C) {
    SKP_ARG(M >= 0 && N >= 0 && K >= 0, "gemm: negative size");
    SKP_ARG(ta == 0 || ta == 1, "gemm: transA must be 0/1");
    SKP_ARG(tb == 0 || tb == 1, "gemm: transB must be 0/1");
    SKP_ARG(lda >= (ta ? M : K) && lda >= 1, "gemm: lda too small");
    SKP_ARG(ldb >= (tb ? K : N) && ldb >= 1, "gemm: ldb too small");
    SKP_ARG(ldc >= N && ldc >= 1, "gemm: ldc too small");
    SKP_ARG((M == 0 || N == 0 || K == 0 || (A && B)) && (M == 0 || N == 0 || C),
            "gemm: null pointer");
    return SKP_OK;
}
}  // namespace

extern "C" int skp_has_tcgen05(void) { return tc_available() ? 1 : 0; }

extern "C" int64_t skp_gemm_ws_bytes(int transA, int transB, int64_t M, int64_t N, int64_t K,
                                     int32_t elem_bytes, int32_t mode) {
    int64_t w = elem_bytes == 8 ? gemm_dmma_ws_bytes(M, N, K) : gemm_simt_ws_bytes(M, N, K, elem_bytes);
    if (elem_bytes == 4 && mode != 2 && tc_available()) {
        int64_t t = gemm_tc_ws_bytes(transA, transB, M, N, K);
        if (t > w) w = t;
    }
    return w;
}

extern "C" int skp_gemm_f32(int transA, int transB, int64_t M, int64_t N, int64_t K, float alpha,
                            const float* A, int64_t lda, const float* B, int64_t ldb, float beta,
                            float* C, int64_t ldc, int32_t mode, void* ws, int64_t ws_bytes,
                            void* stream) {
    int rc = check(transA, transB, M, N, K, lda, ldb, ldc, A, B, C);
    if (rc) return rc;
    SKP_ARG(mode >= 0 && mode <= 2, "gemm_f32: mode must be 0, 1 or 2");
    cudaStream_t st = SKP_STREAM(stream);
    if (mode != 2 && tc_available()) {
        rc = gemm_tc_3xtf32(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws,
                            ws_bytes, st);
        if (rc != SKP_ERR_UNSUPPORTED || mode == 1) return rc;
    } else if (mode == 1) {
        set_error("unsupported: tcgen05 3xTF32 GEMM not available on this device");
        return SKP_ERR_UNSUPPORTED;
    }
    return gemm_simt<float>(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws,
                            ws_bytes, st);
}

extern "C" int skp_gemm_f64(int transA, int transB, int64_t M, int64_t N, int64_t K, double alpha,
                            const double* A, int64_t lda, const double* B, int64_t ldb,
                            double beta, double* C, int64_t ldc, int32_t mode, void* ws,
                            int64_t ws_bytes, void* stream) {
    (void)mode;
    int rc = check(transA, transB, M, N, K, lda, ldb, ldc, A, B, C);
    if (rc) return rc;
    return gemm_dmma(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, ws_bytes,
                     SKP_STREAM(stream));
}
