// One-sided Jacobi SVD (Hestenes) in fp64 for the public thin_svd / pinv
// (replaces LAPACK gesdd, reference linalg.py:84-106).
//
// The Gram route the range finder uses for its small cores (eigen-decompose
// B B^T) resolves singular values only down to ~1e-8 sigma_1: squaring the
// matrix squares its condition number.  Here the columns of A (m x n, m >= n)
// are orthogonalised directly by plane rotations, so every sigma_i comes out
// with an absolute error ~eps sigma_1 (a cond 1e12 matrix keeps its small
// singular values), and the right vectors accumulate the same rotations.
//
// Layout: the columns live contiguously in a workspace (A^T, n x m), V^T
// (n x n) beside it.  One persistent cooperative kernel: each sweep is n' - 1
// rounds of a round-robin tournament (n' = n rounded up to even); in a round
// the n'/2 column pairs are disjoint, so CTAs take pairs independently (a CTA
// reduces the three dot products of its pair over m, then rotates both
// columns of A and of V) and one grid barrier separates rounds.  A sweep that
// rotates no pair ends the iteration.  Rotation (Hestenes / Rutishauser):
//   zeta = (b - a) / (2 g),  t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)),
//   c = 1 / sqrt(1 + t^2),  s = c t;  a_p <- c a_p - s a_q,  a_q <- s a_p + c a_q
// with a = |a_p|^2, b = |a_q|^2, g = a_p . a_q; a pair is rotated while
// |g| > tol sqrt(a b), tol = sqrt(m) eps (LAPACK dgesvj's threshold).
#include <cooperative_groups.h>
#include <math.h>

#include <algorithm>

#include "common.cuh"

namespace skp {
namespace {

namespace cg = cooperative_groups;

constexpr int kJThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x < kJThreads / 32) t = red[threadIdx.x];
    if (w == 0) {
#pragma unroll
        for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (l == 0) red[0] = t;
    }
    __syncthreads();
    return red[0];
}

// round-robin pair k of round r among np players (np even): player np-1 is
// fixed, the rest rotate
__device__ __forceinline__ void rr_pair(int r, int k, int np, int& p, int& q) {
    const int m = np - 1;
    if (k == 0) {
        p = r;
        q = m;
    } else {
        p = (r + k) % m;
        q = (r - k + m) % m;
    }
    if (p > q) {
        const int t = p;
        p = q;
        q = t;
    }
}

__global__ void __launch_bounds__(kJThreads)
gesvj_kernel(double* __restrict__ At, int64_t m, int n, double* __restrict__ Vt, int max_sweeps,
             double tol, unsigned long long* __restrict__ rot_count, int32_t* __restrict__ sweeps) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[kJThreads / 32];
    const int np = n + (n & 1);
    const int pairs = np / 2;
    int sw = 0;
    for (; sw < max_sweeps; ++sw) {
        for (int r = 0; r < np - 1; ++r) {
            for (int k = blockIdx.x; k < pairs; k += gridDim.x) {
                int p, q;
                rr_pair(r, k, np, p, q);
                if (q >= n) continue;  // the padding player
                double* ap = At + (int64_t)p * m;
                double* aq = At + (int64_t)q * m;
                double sa = 0.0, sb = 0.0, sg = 0.0;
                for (int64_t i = threadIdx.x; i < m; i += kJThreads) {
                    const double x = ap[i], y = aq[i];
                    sa = fma(x, x, sa);
                    sb = fma(y, y, sb);
                    sg = fma(x, y, sg);
                }
                const double a = block_sum(sa, red);
                const double b = block_sum(sb, red);
                const double g = block_sum(sg, red);
                if (!(fabs(g) > tol * sqrt(a) * sqrt(b)) || g == 0.0) continue;
                const double zeta = (b - a) / (2.0 * g);
                const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t);
                const double s = c * t;
                for (int64_t i = threadIdx.x; i < m; i += kJThreads) {
                    const double x = ap[i], y = aq[i];
                    ap[i] = c * x - s * y;
                    aq[i] = s * x + c * y;
                }
                double* vp = Vt + (int64_t)p * n;
                double* vq = Vt + (int64_t)q * n;
                for (int i = threadIdx.x; i < n; i += kJThreads) {
                    const double x = vp[i], y = vq[i];
                    vp[i] = c * x - s * y;
                    vq[i] = s * x + c * y;
                }
                if (threadIdx.x == 0) atomicAdd(&rot_count[sw], 1ull);
            }
            grid.sync();
        }
        // every CTA reads the same count after the barrier
        if (*reinterpret_cast<volatile unsigned long long*>(&rot_count[sw]) == 0) break;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *sweeps = sw + 1;
}

__global__ void vt_identity_kernel(double* __restrict__ Vt, int n) {
    const int64_t nn = (int64_t)n * n;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nn;
         t += (int64_t)gridDim.x * blockDim.x)
        Vt[t] = (t / n == t % n) ? 1.0 : 0.0;
}

// A (row-major, lda) -> A^T (n x m, columns contiguous)
template <typename T>
__global__ void to_cols_kernel(const T* __restrict__ A, int64_t m, int n, int64_t lda,
                               double* __restrict__ At) {
    __shared__ double tile[32][33];
    const int64_t i0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t i = i0 + r, j = j0 + threadIdx.x;
        tile[r][threadIdx.x] = (i < m && j < n) ? (double)A[i * lda + j] : 0.0;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t j = j0 + r, i = i0 + threadIdx.x;
        if (j < n && i < m) At[j * m + i] = tile[threadIdx.x][r];
    }
}

// sigma_j = |a_j| (one thread per column); gesvj_scatter_kernel then orders
// them descending (ties by index) with U[:, rank] = a_j / sigma_j (0 for
// sigma_j = 0) and V[:, rank] = v_j
__global__ void gesvj_norms_kernel(const double* __restrict__ At, int64_t m, int n,
                                   double* __restrict__ norms) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        double s = 0.0;
        const double* a = At + (int64_t)j * m;
        for (int64_t i = 0; i < m; ++i) s = fma(a[i], a[i], s);
        norms[j] = sqrt(s);
    }
}
__global__ void gesvj_scatter_kernel(const double* __restrict__ At, int64_t m, int n,
                                     const double* __restrict__ Vt,
                                     const double* __restrict__ norms, double* __restrict__ S,
                                     double* __restrict__ U, int64_t ldu, double* __restrict__ V,
                                     int64_t ldv) {
    // block per column j
    const int j = blockIdx.x;
    if (j >= n) return;
    const double sj = norms[j];
    int rank = 0;
    for (int k = 0; k < n; ++k) {
        const double sk = norms[k];
        rank += (sk > sj) || (sk == sj && k < j);
    }
    if (threadIdx.x == 0) S[rank] = sj;
    const double inv = sj > 0.0 ? 1.0 / sj : 0.0;
    const double* a = At + (int64_t)j * m;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) U[i * ldu + rank] = a[i] * inv;
    const double* v = Vt + (int64_t)j * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) V[(int64_t)i * ldv + rank] = v[i];
}

template <typename T>
int gesvj(const T* A, int64_t m, int64_t n, int64_t lda, double* S, double* U, int64_t ldu,
          double* V, int64_t ldv, int max_sweeps, void* ws, int64_t ws_bytes, int32_t* sweeps,
          cudaStream_t st);

}  // namespace

int64_t gesvj_ws_bytes(int64_t m, int64_t n) {
    return (int64_t)sizeof(double) * (n * m + n * n + n) + 64 * (int64_t)sizeof(unsigned long long) +
           256;
}

namespace {
template <typename T>
int gesvj(const T* A, int64_t m, int64_t n, int64_t lda, double* S, double* U, int64_t ldu,
          double* V, int64_t ldv, int max_sweeps, void* ws, int64_t ws_bytes, int32_t* sweeps,
          cudaStream_t st) {
    SKP_ARG(m >= n && n >= 1 && n <= (1 << 20) && lda >= n && ldu >= n && ldv >= n,
            "gesvj: needs m >= n >= 1 (transpose a wide matrix)");
    SKP_ARG(max_sweeps >= 1 && max_sweeps <= 60, "gesvj: max_sweeps in [1, 60]");
    SKP_ARG(ws && ws_bytes >= gesvj_ws_bytes(m, n), "gesvj needs %lld bytes of workspace",
            (long long)gesvj_ws_bytes(m, n));
    double* At = reinterpret_cast<double*>(ws);
    double* Vt = At + n * m;
    double* norms = Vt + n * n;
    auto* cnt = reinterpret_cast<unsigned long long*>(norms + n);
    SKP_CUDA(cudaMemsetAsync(cnt, 0, 64 * sizeof(unsigned long long), st));
    {
        dim3 grid((unsigned)cdiv(n, 32), (unsigned)cdiv(m, 32));
        to_cols_kernel<T><<<grid, dim3(32, 8), 0, st>>>(A, m, (int)n, lda, At);
        SKP_LAUNCHED(to_cols_kernel);
        vt_identity_kernel<<<(unsigned)std::min<int64_t>(cdiv(n * n, 256), 4096), 256, 0, st>>>(
            Vt, (int)n);
        SKP_LAUNCHED(vt_identity_kernel);
    }
    int dev = 0, sms = 148, per_sm = 0;
    SKP_CUDA(cudaGetDevice(&dev));
    SKP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    SKP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gesvj_kernel, kJThreads, 0));
    SKP_ARG(per_sm >= 1, "gesvj: cooperative kernel cannot be resident");
    const int pairs = (int)((n + (n & 1)) / 2);
    int blocks = std::max(1, std::min(sms * per_sm, pairs));
    int64_t mm = m;
    int nn = (int)n;
    int mx = std::min(max_sweeps, 64);
    double tol = sqrt((double)m) * 2.220446049250313e-16;
    void* args[] = {&At, &mm, &nn, &Vt, &mx, &tol, &cnt, &sweeps};
    SKP_CUDA(cudaLaunchCooperativeKernel((void*)gesvj_kernel, dim3(blocks), dim3(kJThreads), args,
                                         0, st));
    count_launch();
    gesvj_norms_kernel<<<(unsigned)cdiv(n, 128), 128, 0, st>>>(At, m, nn, norms);
    SKP_LAUNCHED(gesvj_norms_kernel);
    gesvj_scatter_kernel<<<(unsigned)n, 256, 0, st>>>(At, m, nn, Vt, norms, S, U, ldu, V, ldv);
    SKP_LAUNCHED(gesvj_scatter_kernel);
    return SKP_OK;
}
}  // namespace
}  // namespace skp

using namespace skp;

extern "C" int64_t skp_gesvj_ws_bytes(int64_t m, int64_t n) { return gesvj_ws_bytes(m, n); }

extern "C" int skp_gesvj_f64(const double* A, int64_t m, int64_t n, int64_t lda, double* S,
                             double* U, int64_t ldu, double* V, int64_t ldv, int32_t max_sweeps,
                             void* ws, int64_t ws_bytes, int32_t* sweeps, void* stream) {
    return skp::gesvj<double>(A, m, n, lda, S, U, ldu, V, ldv, max_sweeps, ws, ws_bytes, sweeps,
                              SKP_STREAM(stream));
}
extern "C" int skp_gesvj_f32(const float* A, int64_t m, int64_t n, int64_t lda, double* S,
                             double* U, int64_t ldu, double* V, int64_t ldv, int32_t max_sweeps,
                             void* ws, int64_t ws_bytes, int32_t* sweeps, void* stream) {
    return skp::gesvj<float>(A, m, n, lda, S, U, ldu, V, ldv, max_sweeps, ws, ws_bytes, sweeps,
                             SKP_STREAM(stream));
}
