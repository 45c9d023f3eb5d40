// SIMT GEMM (CUDA cores): the FP64 path and the exact-FP32 mode of
// skp_gemm_f32.  Row-major, op(A) M x K, op(B) K x N, optional split-K into a
// caller workspace reduced deterministically (fixed summation order).
// The FP32 hot path is the tcgen05 3xTF32 kernel (gemm_tc.cu); this file is
// also its fallback when the tcgen05 path does not apply.
#include "common.cuh"
#include "gemm.h"

namespace skp {
namespace {

constexpr int BM = 64, BN = 64, THREADS = 256;

template <typename T>
struct Bk;
template <>
struct Bk<float> { static constexpr int v = 16; };
template <>
struct Bk<double> { static constexpr int v = 8; };

template <typename T>
__global__ void __launch_bounds__(THREADS)
gemm_simt_kernel(int ta, int tb, int64_t M, int64_t N, int64_t K, int64_t kchunk, T alpha,
                 const T* __restrict__ A, int64_t lda, const T* __restrict__ B, int64_t ldb,
                 T beta, T* __restrict__ C, int64_t ldc, T* __restrict__ ws) {
    constexpr int BK = Bk<T>::v;
    __shared__ __align__(16) T As[BK][BM + 4];
    __shared__ __align__(16) T Bs[BK][BN + 4];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
    const int64_t kb = (int64_t)blockIdx.z * kchunk;
    const int64_t ke = kb + kchunk < K ? kb + kchunk : K;
    T acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
    for (int64_t k0 = kb; k0 < ke; k0 += BK) {
#pragma unroll
        for (int it = 0; it < (BM * BK) / THREADS; ++it) {
            int idx = tid + it * THREADS;
            int mm, kk;
            if (!ta) { mm = idx / BK; kk = idx % BK; } else { kk = idx / BM; mm = idx % BM; }
            int64_t gm = m0 + mm, gk = k0 + kk;
            T v = T(0);
            if (gm < M && gk < ke) v = ta ? A[gk * lda + gm] : A[gm * lda + gk];
            As[kk][mm] = v;
        }
#pragma unroll
        for (int it = 0; it < (BN * BK) / THREADS; ++it) {
            int idx = tid + it * THREADS;
            int nn, kk;
            if (tb) { nn = idx / BK; kk = idx % BK; } else { kk = idx / BN; nn = idx % BN; }
            int64_t gn = n0 + nn, gk = k0 + kk;
            T v = T(0);
            if (gn < N && gk < ke) v = tb ? B[gn * ldb + gk] : B[gk * ldb + gn];
            Bs[kk][nn] = v;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            T a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int64_t gm = m0 + ty * 4 + i;
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int64_t gn = n0 + tx * 4 + j;
            if (gn >= N) continue;
            if (ws) {
                ws[((int64_t)blockIdx.z * M + gm) * N + gn] = acc[i][j];
            } else {
                T* c = C + gm * ldc + gn;
                *c = beta == T(0) ? alpha * acc[i][j] : alpha * acc[i][j] + beta * *c;
            }
        }
    }
}

template <typename T>
__global__ void splitk_reduce_kernel(const T* __restrict__ ws, int splits, int64_t M, int64_t N,
                                     T alpha, T beta, T* __restrict__ C, int64_t ldc) {
    const int64_t total = M * N;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        T s = T(0);
        for (int z = 0; z < splits; ++z) s += ws[(int64_t)z * total + t];
        int64_t i = t / N, j = t - i * N;
        T* c = C + i * ldc + j;
        *c = beta == T(0) ? alpha * s : alpha * s + beta * *c;
    }
}

template <typename T>
int choose_splits(int64_t M, int64_t N, int64_t K, int64_t ws_bytes) {
    int64_t tiles = cdiv(M, BM) * cdiv(N, BN);
    int64_t target = 2 * 148;
    if (tiles >= target || K < 512) return 1;
    int64_t s = cdiv(target, tiles);
    int64_t maxs = K / 256;
    if (s > maxs) s = maxs;
    if (s > 64) s = 64;
    int64_t cap = ws_bytes / (int64_t)(M * N * sizeof(T));
    if (s > cap) s = cap;
    return s < 1 ? 1 : (int)s;
}

}  // namespace

template <typename T>
int gemm_simt(int ta, int tb, int64_t M, int64_t N, int64_t K, T alpha, const T* A, int64_t lda,
              const T* B, int64_t ldb, T beta, T* C, int64_t ldc, void* ws, int64_t ws_bytes,
              cudaStream_t st) {
    constexpr int BK = Bk<T>::v;
    if (M == 0 || N == 0) return SKP_OK;
    int splits = choose_splits<T>(M, N, K, ws ? ws_bytes : 0);
    int64_t kchunk = cdiv(cdiv(K, BK), splits) * BK;
    if (K == 0) kchunk = BK;
    splits = (int)(K == 0 ? 1 : cdiv(K, kchunk));
    SKP_ARG(cdiv(M, BM) < 65536, "gemm: M too large for the SIMT path");
    dim3 grid((unsigned)cdiv(N, BN), (unsigned)cdiv(M, BM), (unsigned)splits);
    T* wsp = splits > 1 ? reinterpret_cast<T*>(ws) : nullptr;
    gemm_simt_kernel<T><<<grid, THREADS, 0, st>>>(ta, tb, M, N, K, kchunk, alpha, A, lda, B, ldb,
                                                 beta, C, ldc, wsp);
    SKP_LAUNCHED(gemm_simt_kernel);
    if (splits > 1) {
        int64_t blocks = cdiv(M * N, 256);
        if (blocks > 148 * 16) blocks = 148 * 16;
        splitk_reduce_kernel<T><<<(unsigned)blocks, 256, 0, st>>>(wsp, splits, M, N, alpha, beta,
                                                                  C, ldc);
        SKP_LAUNCHED(splitk_reduce_kernel);
    }
    return SKP_OK;
}

int64_t gemm_simt_ws_bytes(int64_t M, int64_t N, int64_t K, int elem) {
    int64_t s = elem == 8 ? choose_splits<double>(M, N, K, INT64_MAX)
                          : choose_splits<float>(M, N, K, INT64_MAX);
    return s > 1 ? s * M * N * elem : 0;
}

template int gemm_simt<float>(int, int, int64_t, int64_t, int64_t, float, const float*, int64_t,
                              const float*, int64_t, float, float*, int64_t, void*, int64_t,
                              cudaStream_t);
template int gemm_simt<double>(int, int, int64_t, int64_t, int64_t, double, const double*,
                               int64_t, const double*, int64_t, double, double*, int64_t, void*,
                               int64_t, cudaStream_t);

}  // namespace skp

// ---- G = X^T X in fp64 from fp32 X (randsvd's B B^T via B^T) ----------------
// fp32 x fp32 products are exact in fp64, so the fp64 Gram of fp32 data needs
// no widened copy: gemm_dmma.cu widens X as it stages the tiles and
// accumulates on the DMMA tensor cores (lower tiles only, mirrored; split-K
// partials reduced in a fixed order).
using namespace skp;
extern "C" int64_t skp_gram_f32_f64_ws_bytes(int64_t K, int64_t C) {
    return skp::gram_dmma_ws_bytes(K, C);
}
extern "C" int skp_gram_f32_f64(const float* X, int64_t K, int64_t C, int64_t ldx, double* G,
                                int64_t ldg, void* ws, int64_t ws_bytes, void* stream) {
    SKP_ARG(K >= 1 && C >= 1 && ldx >= C && ldg >= C, "gram_f32_f64: bad sizes");
    SKP_ARG(ws_bytes >= skp_gram_f32_f64_ws_bytes(K, C) && (ws || ws_bytes == 0),
            "gram_f32_f64: workspace too small");
    return skp::gram_dmma_f32(X, K, C, ldx, G, ldg, ws, ws_bytes, SKP_STREAM(stream));
}
