// K4d: FP64 GEMM on the FP64 tensor cores (DMMA, mma.sync m8n8k4.f64) -- the
// FP64 path (C1, the psd Nystrom core, fp64 operands of the facade).
// tcgen05 has no f64 kind; the B200's FP64 rate (~37 TFLOP/s, cuBLAS DGEMM
// 35.5 measured: scripts/peaks_probe.py) is reached through DMMA, which the
// SIMT kernel (gemm_simt.cu: 9.1 TFLOP/s) cannot approach.
//
// CTA tile 128 x 64 x 16 (8 warps, 4 along M x 2 along N; warp tile 32 x 32 =
// 4 x 4 DMMA tiles, 32 fp64 accumulators per lane).  Operands are staged
// k-major in shared memory (As[k][m], Bs[k][n]) with a 4-double pad, so a
// fragment load -- lane reads (k = lane % 4, m = lane / 4) -- touches 16
// distinct banks per half warp.  The next K tile is fetched into registers
// while the current one is multiplied.  Split-K over a caller workspace,
// reduced in a fixed order (deterministic), as the SIMT kernel.
//   DMMA m8n8k4 (row.col): a = A[lane/4][lane%4], b = B[lane%4][lane/4],
//   c = C[lane/4][2 (lane%4) + {0, 1}].
#include <algorithm>

#include "common.cuh"
#include "gemm.h"

namespace skp {
namespace {

constexpr int DM = 128, DN = 64, DK = 16, DTHREADS = 256;
constexpr int DMP = DM + 4, DNP = DN + 4;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// TIn = float: fp32 operands widened to fp64 as they are staged (exact), e.g.
// randsvd's B B^T from fp32 B^T.  sym: C = A^T A (A == B), only the tiles
// meeting the lower triangle run; the caller mirrors the strict upper one.
template <typename TIn>
__global__ void __launch_bounds__(DTHREADS)
gemm_dmma_kernel(int ta, int tb, int64_t M, int64_t N, int64_t K, int64_t kchunk, double alpha,
                 const TIn* __restrict__ A, int64_t lda, const TIn* __restrict__ B,
                 int64_t ldb, double beta, double* __restrict__ C, int64_t ldc,
                 double* __restrict__ ws, int sym) {
    __shared__ __align__(16) double As[DK][DMP];
    __shared__ __align__(16) double Bs[DK][DNP];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 3, wn = warp >> 2;
    const int64_t m0 = (int64_t)blockIdx.y * DM, n0 = (int64_t)blockIdx.x * DN;
    if (sym && n0 >= m0 + DM) return;  // strictly upper tile: mirrored by the caller
    const int64_t kb = (int64_t)blockIdx.z * kchunk;
    const int64_t ke = kb + kchunk < K ? kb + kchunk : K;

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    double ra[(DM * DK) / DTHREADS], rb[(DN * DK) / DTHREADS];
    auto fetch = [&](int64_t k0) {
#pragma unroll
        for (int it = 0; it < (DM * DK) / DTHREADS; ++it) {
            const int idx = tid + it * DTHREADS;
            int mm, kk;
            if (!ta) { mm = idx / DK; kk = idx % DK; } else { kk = idx / DM; mm = idx % DM; }
            const int64_t gm = m0 + mm, gk = k0 + kk;
            ra[it] = (gm < M && gk < ke) ? (double)(ta ? A[gk * lda + gm] : A[gm * lda + gk]) : 0.0;
        }
#pragma unroll
        for (int it = 0; it < (DN * DK) / DTHREADS; ++it) {
            const int idx = tid + it * DTHREADS;
            int nn, kk;
            if (tb) { nn = idx / DK; kk = idx % DK; } else { kk = idx / DN; nn = idx % DN; }
            const int64_t gn = n0 + nn, gk = k0 + kk;
            rb[it] = (gn < N && gk < ke) ? (double)(tb ? B[gn * ldb + gk] : B[gk * ldb + gn]) : 0.0;
        }
    };
    auto stash = [&]() {
#pragma unroll
        for (int it = 0; it < (DM * DK) / DTHREADS; ++it) {
            const int idx = tid + it * DTHREADS;
            int mm, kk;
            if (!ta) { mm = idx / DK; kk = idx % DK; } else { kk = idx / DM; mm = idx % DM; }
            As[kk][mm] = ra[it];
        }
#pragma unroll
        for (int it = 0; it < (DN * DK) / DTHREADS; ++it) {
            const int idx = tid + it * DTHREADS;
            int nn, kk;
            if (tb) { nn = idx / DK; kk = idx % DK; } else { kk = idx / DN; nn = idx % DN; }
            Bs[kk][nn] = rb[it];
        }
    };

    if (kb < ke) fetch(kb);
    for (int64_t k0 = kb; k0 < ke; k0 += DK) {
        __syncthreads();  // the previous tile's fragments are consumed
        stash();
        __syncthreads();
        if (k0 + DK < ke) fetch(k0 + DK);  // next tile in flight during the MMAs
#pragma unroll
        for (int k4 = 0; k4 < DK; k4 += 4) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[k4 + (lane & 3)][wm * 32 + i * 8 + (lane >> 2)];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[k4 + (lane & 3)][wn * 32 + j * 8 + (lane >> 2)];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t gm = m0 + wm * 32 + i * 8 + (lane >> 2);
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t gn = n0 + wn * 32 + j * 8 + 2 * (lane & 3) + h;
                if (gn >= N) continue;
                const double v = acc[i][j][h];
                if (ws) {
                    ws[((int64_t)blockIdx.z * M + gm) * N + gn] = v;
                } else {
                    double* c = C + gm * ldc + gn;
                    *c = beta == 0.0 ? alpha * v : alpha * v + beta * *c;
                }
            }
        }
    }
}

__global__ void dmma_splitk_reduce(const double* __restrict__ ws, int splits, int64_t M, int64_t N,
                                   double alpha, double beta, double* __restrict__ C, int64_t ldc) {
    const int64_t total = M * N;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int z = 0; z < splits; ++z) s += ws[(int64_t)z * total + t];
        const int64_t i = t / N, j = t - i * N;
        double* c = C + i * ldc + j;
        *c = beta == 0.0 ? alpha * s : alpha * s + beta * *c;
    }
}

int dmma_splits(int64_t M, int64_t N, int64_t K, int64_t ws_bytes) {
    const int64_t tiles = cdiv(M, DM) * cdiv(N, DN);
    const int64_t target = 2 * 148;
    if (tiles >= target || K < 512) return 1;
    int64_t s = cdiv(target, tiles);
    s = std::min<int64_t>(s, K / 256);
    s = std::min<int64_t>(s, 64);
    s = std::min<int64_t>(s, ws_bytes / (M * N * (int64_t)sizeof(double)));
    return s < 1 ? 1 : (int)s;
}

}  // namespace

int64_t gemm_dmma_ws_bytes(int64_t M, int64_t N, int64_t K) {
    const int s = dmma_splits(M, N, K, INT64_MAX);
    return s > 1 ? (int64_t)s * M * N * (int64_t)sizeof(double) : 0;
}

int gemm_dmma(int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
              int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
              void* ws, int64_t ws_bytes, cudaStream_t st) {
    if (M == 0 || N == 0) return SKP_OK;
    int splits = dmma_splits(M, N, K, ws ? ws_bytes : 0);
    int64_t kchunk = cdiv(cdiv(K, DK), splits) * DK;
    if (K == 0) kchunk = DK;
    splits = (int)(K == 0 ? 1 : cdiv(K, kchunk));
    SKP_ARG(cdiv(M, DM) < 65536, "gemm: M too large for the fp64 path");
    dim3 grid((unsigned)cdiv(N, DN), (unsigned)cdiv(M, DM), (unsigned)splits);
    double* wsp = splits > 1 ? reinterpret_cast<double*>(ws) : nullptr;
    gemm_dmma_kernel<double><<<grid, DTHREADS, 0, st>>>(ta, tb, M, N, K, kchunk, alpha, A, lda,
                                                        B, ldb, beta, C, ldc, wsp, 0);
    SKP_LAUNCHED(gemm_dmma_kernel);
    if (splits > 1) {
        const int64_t blocks = std::min<int64_t>(cdiv(M * N, 256), 148 * 16);
        dmma_splitk_reduce<<<(unsigned)blocks, 256, 0, st>>>(wsp, splits, M, N, alpha, beta, C,
                                                             ldc);
        SKP_LAUNCHED(dmma_splitk_reduce);
    }
    return SKP_OK;
}

__global__ void mirror_lower_f64(double* __restrict__ C, int64_t n, int64_t ldc) {
    __shared__ double t[32][33];
    const int64_t bi = blockIdx.y, bj = blockIdx.x;  // source tile (bi, bj), bi >= bj
    if (bj > bi) return;
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int r = ty; r < 32; r += 8) {
        const int64_t i = bi * 32 + r, j = bj * 32 + tx;
        t[r][tx] = (i < n && j < n) ? C[i * ldc + j] : 0.0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int64_t i = bj * 32 + r, j = bi * 32 + tx;
        if (i < n && j < n && j > i) C[i * ldc + j] = t[tx][r];
    }
}

int gram_splits(int64_t K, int64_t Cc, int64_t ws_bytes);
int64_t gram_dmma_ws_bytes(int64_t K, int64_t C) {
    const int s = gram_splits(K, C, INT64_MAX);
    return s > 1 ? (int64_t)s * C * C * (int64_t)sizeof(double) : 0;
}

// G = X^T X (C x C, fp64, exactly symmetric) of fp32 X (K x C): exact fp32
// products, fp64 DMMA accumulation, lower tiles only, then mirrored
// split-K count for the Gram: the lower tiles x s slices over the SMs (one
// 224-register CTA each) in as few waves per slice as possible
int gram_splits(int64_t K, int64_t Cc, int64_t ws_bytes) {
    int64_t lower = 0;
    for (int64_t bm = 0; bm < cdiv(Cc, DM); ++bm)
        lower += std::min<int64_t>(cdiv(Cc, DN), cdiv((bm + 1) * DM, DN));
    int best = 1;
    double best_t = 1e30;
    for (int s = 1; s <= 32 && (s == 1 || K / s >= 512); ++s) {
        if (s > 1 && (int64_t)s * Cc * Cc * (int64_t)sizeof(double) > ws_bytes) break;
        const double t = (double)cdiv(lower * s, (int64_t)148) / s;
        if (t < best_t - 1e-9) {
            best_t = t;
            best = s;
        }
    }
    return best;
}

int gram_dmma_f32(const float* X, int64_t K, int64_t Cc, int64_t ldx, double* G, int64_t ldg,
                  void* ws, int64_t ws_bytes, cudaStream_t st) {
    int splits = gram_splits(K, Cc, ws ? ws_bytes : 0);
    int64_t kchunk = cdiv(cdiv(K, DK), splits) * DK;
    splits = (int)cdiv(K, kchunk);
    SKP_ARG(cdiv(Cc, DM) < 65536, "gram: too many columns");
    dim3 grid((unsigned)cdiv(Cc, DN), (unsigned)cdiv(Cc, DM), (unsigned)splits);
    double* wsp = splits > 1 ? reinterpret_cast<double*>(ws) : nullptr;
    gemm_dmma_kernel<float><<<grid, DTHREADS, 0, st>>>(1, 0, Cc, Cc, K, kchunk, 1.0, X, ldx, X, ldx,
                                                       0.0, G, ldg, wsp, 1);
    SKP_LAUNCHED(gemm_dmma_kernel);
    if (splits > 1) {
        const int64_t blocks = std::min<int64_t>(cdiv(Cc * Cc, 256), 148 * 16);
        dmma_splitk_reduce<<<(unsigned)blocks, 256, 0, st>>>(wsp, splits, Cc, Cc, 1.0, 0.0, G, ldg);
        SKP_LAUNCHED(dmma_splitk_reduce);
    }
    const unsigned nt = (unsigned)cdiv(Cc, 32);
    mirror_lower_f64<<<dim3(nt, nt), dim3(32, 8), 0, st>>>(G, Cc, ldg);
    SKP_LAUNCHED(mirror_lower_f64);
    return SKP_OK;
}

}  // namespace skp
