// K6 v2: symmetric eigensolver via tridiagonal reduction (fp64), for the
// r2 x r2 cores (randsvd's B B^T, Nystrom's W) with 112 < n <= 8192.
//
//   1. sytrd_kernel   cooperative Householder tridiagonalisation, 2 grid
//                     syncs per column (p = tau A v, then A -= v w^T + w v^T);
//                     every CTA rebuilds the reflector redundantly from the
//                     untouched column, so no extra sync is needed for it.
//   2. bisect_kernel  one thread per eigenvalue: Sturm-count bisection on T
//                     (d, e staged in smem) -> eigenvalues already sorted
//                     (index i = (i+1)-th largest), absolute accuracy
//                     ~eps * ||T||.
//   3. inviter_kernel one thread per eigenvector: 3 steps of inverse iteration
//                     with a partially pivoted tridiagonal LU (LAPACK dlagtf /
//                     dlagts scheme), vectors stored column-interleaved so the
//                     threads of a warp touch consecutive addresses.
//   4. reorth_kernel  modified Gram-Schmidt inside clusters of eigenvalues
//                     closer than 1e-10 * ||T|| (degenerate / zero clusters).
//   5. backtr_kernel  x <- H_0 ... H_{n-3} x per eigenvector, one warp per
//                     column; columns are independent, so no grid syncs.
// ~2 * n grid syncs in total vs ~13 * n for cyclic Jacobi.
#include <cooperative_groups.h>
#include <math.h>

#include <algorithm>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace skp {
namespace {

constexpr int kTriThreads = 512;

__device__ double block_reduce_sum_all(double v, double* scratch) {
    // all threads receive the sum
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) scratch[w] = v;
    __syncthreads();
    double r = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r += scratch[i];
    __syncthreads();
    return r;
}

// A: n x n symmetric (full storage, row-major, overwritten).  Outputs d[n],
// e[n-1], tau[n-1], Hv (n x n; row i holds v_i on columns i+1.., v_i[i+1]=1).
__global__ void __launch_bounds__(kTriThreads)
sytrd_kernel(double* A, int n, double* d, double* e, double* tau, double* Hv, double* pbuf) {
    __shared__ double scratch[32];
    cg::grid_group grid = cg::this_grid();
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
    const int warp_g = (int)(gtid >> 5), lane = threadIdx.x & 31;
    const int nwarps_g = (int)(gstride >> 5);
    for (int i = 0; i + 2 < n; ++i) {
        const int r0 = i + 1, k = n - r0;
        // (a) reflector from x = A[r0:, i] (column i below the diagonal is not
        //     touched by this step's update, so every CTA can read it)
        double ss = 0.0;
        for (int t = 1 + threadIdx.x; t < k; t += blockDim.x) {
            const double x = A[(int64_t)(r0 + t) * n + i];
            ss += x * x;
        }
        const double xnorm2 = block_reduce_sum_all(ss, scratch);
        const double alpha = A[(int64_t)r0 * n + i];
        double t_, beta, scal;
        if (xnorm2 == 0.0) {
            t_ = 0.0;
            beta = alpha;
            scal = 0.0;
        } else {
            beta = -copysign(sqrt(alpha * alpha + xnorm2), alpha);
            t_ = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        // v_c (c = r0 + t): t == 0 -> 1, else x_t * scal
        auto vat = [&](int t) -> double {
            return t == 0 ? 1.0 : A[(int64_t)(r0 + t) * n + i] * scal;
        };
        // (b) p = tau * A' v, one warp per row of A' = A[r0:, r0:]
        if (t_ != 0.0) {
            for (int rr = warp_g; rr < k; rr += nwarps_g) {
                const double* row = A + (int64_t)(r0 + rr) * n + r0;
                double acc = 0.0;
                for (int t = lane; t < k; t += 32) acc += row[t] * vat(t);
                acc = warp_sum(acc);
                if (lane == 0) pbuf[rr] = t_ * acc;
            }
        }
        if (gtid == 0) {
            d[i] = A[(int64_t)i * n + i];
            e[i] = beta;
            tau[i] = t_;
        }
        grid.sync();
        if (t_ != 0.0) {
            // (c) K = tau/2 * p.v ; w = p - K v   (redundant per CTA)
            double pv = 0.0;
            for (int t = threadIdx.x; t < k; t += blockDim.x) pv += pbuf[t] * vat(t);
            const double K = 0.5 * t_ * block_reduce_sum_all(pv, scratch);
            // (d) A' -= v w^T + w v^T
            for (int64_t q = gtid; q < (int64_t)k * k; q += gstride) {
                const int rr = (int)(q / k), cc = (int)(q % k);
                const double vr = vat(rr), vc = vat(cc);
                const double wr = pbuf[rr] - K * vr, wc = pbuf[cc] - K * vc;
                A[(int64_t)(r0 + rr) * n + r0 + cc] -= vr * wc + wr * vc;
            }
        }
        // store v_i for the back-transformation (row i of Hv)
        for (int64_t t = gtid; t < k; t += gstride) Hv[(int64_t)i * n + r0 + t] = vat((int)t);
        grid.sync();
    }
    if (gtid == 0) {
        if (n >= 2) {
            d[n - 2] = A[(int64_t)(n - 2) * n + n - 2];
            e[n - 2] = A[(int64_t)(n - 1) * n + n - 2];
            tau[n - 2] = 0.0;
        }
        d[n - 1] = A[(int64_t)(n - 1) * n + n - 1];
    }
}

// #eigenvalues of T strictly less than x (Sturm sequence via LDL^T)
__device__ __forceinline__ int sturm_count(const double* d, const double* e2, int n, double x,
                                           double pivmin) {
    int cnt = 0;
    double q = d[0] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
    for (int j = 1; j < n; ++j) {
        q = (d[j] - x) - e2[j - 1] / q;
        if (fabs(q) < pivmin) q = -pivmin;
        cnt += q < 0.0;
    }
    return cnt;
}

__global__ void bisect_kernel(const double* __restrict__ dg, const double* __restrict__ eg, int n,
                              double* __restrict__ W, double* __restrict__ tnorm_out) {
    extern __shared__ double sm[];
    double* d = sm;
    double* e2 = sm + n;
    __shared__ double lo_s, hi_s;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        d[j] = dg[j];
        if (j < n - 1) e2[j] = eg[j] * eg[j];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double lo = INFINITY, hi = -INFINITY;
        for (int j = 0; j < n; ++j) {
            const double r = (j > 0 ? fabs(eg[j - 1]) : 0.0) + (j < n - 1 ? fabs(eg[j]) : 0.0);
            lo = fmin(lo, d[j] - r);
            hi = fmax(hi, d[j] + r);
        }
        const double tn = fmax(fabs(lo), fabs(hi));
        lo_s = lo - 4e-16 * tn - 1e-300;
        hi_s = hi + 4e-16 * tn + 1e-300;
        if (blockIdx.x == 0) *tnorm_out = tn;
    }
    __syncthreads();
    const double tn = fmax(fabs(lo_s), fabs(hi_s));
    const double pivmin = 1e-290;
    const double width = 4.0 * 2.220446049250313e-16 * tn + 1e-300;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        // (i+1)-th largest: the value x with count(x) <= n-1-i < count(x')
        const int target = n - 1 - i;  // number of eigenvalues below it
        double lo = lo_s, hi = hi_s;
        for (int it = 0; it < 200; ++it) {
            const double mid = 0.5 * (lo + hi);
            if (mid == lo || mid == hi || hi - lo <= width) break;
            if (sturm_count(d, e2, n, mid, pivmin) > target) hi = mid;
            else lo = mid;
        }
        W[i] = 0.5 * (lo + hi);
    }
}

// Inverse iteration: thread j computes eigenvector j of T for lambda = W[j].
// Scratch per thread (interleaved [row][j]): u1, u2, u3 (upper bands), mult,
// piv (as double 0/1), x.  Z (n x n) receives column j.
__global__ void inviter_kernel(const double* __restrict__ d, const double* __restrict__ e, int n,
                               const double* __restrict__ W, const double* __restrict__ tnorm_p,
                               double* __restrict__ scr, double* __restrict__ Z) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int64_t N = n;
    double* U1 = scr;
    double* U2 = scr + N * N;
    double* U3 = scr + 2 * N * N;
    double* ML = scr + 3 * N * N;
    double* PV = scr + 4 * N * N;
    const double tn = fmax(*tnorm_p, 1e-300);
    const double lam = W[j];
    const double eps_piv = 2.2e-16 * tn;
    // LU with partial pivoting of (T - lam I), rows r, r+1 interchange
    // column layout: row r has u1 (diag), u2 (super 1), u3 (super 2)
    double a = d[0] - lam;              // current diag candidate of row r
    double b = n > 1 ? e[0] : 0.0;      // super diag of row r
    double c3 = 0.0;                    // 2nd super of row r (from a previous swap)
    for (int r = 0; r < n - 1; ++r) {
        const double sub = e[r];                  // T[r+1][r]
        const double dnext = d[r + 1] - lam;      // T[r+1][r+1]
        const double snext = r + 1 < n - 1 ? e[r + 1] : 0.0;  // T[r+1][r+2]
        if (fabs(a) >= fabs(sub)) {
            // no swap: row r stays pivot
            double piv = a;
            if (fabs(piv) < eps_piv) piv = copysign(eps_piv, piv == 0.0 ? 1.0 : piv);
            const double m = sub / piv;
            U1[r * N + j] = piv;
            U2[r * N + j] = b;
            U3[r * N + j] = c3;
            ML[r * N + j] = m;
            PV[r * N + j] = 0.0;
            a = dnext - m * b;
            b = snext - m * c3;
            c3 = 0.0;
        } else {
            // swap rows r and r+1: pivot row is (sub, dnext, snext)
            const double m = a / sub;
            U1[r * N + j] = sub;
            U2[r * N + j] = dnext;
            U3[r * N + j] = snext;
            ML[r * N + j] = m;
            PV[r * N + j] = 1.0;
            a = b - m * dnext;
            b = c3 - m * snext;
            c3 = 0.0;
        }
    }
    {
        double piv = a;
        if (fabs(piv) < eps_piv) piv = copysign(eps_piv, piv == 0.0 ? 1.0 : piv);
        U1[(N - 1) * N + j] = piv;
        U2[(N - 1) * N + j] = 0.0;
        U3[(N - 1) * N + j] = 0.0;
    }
    // start vector: deterministic pseudo-random
    uint64_t st = 0x9E3779B97F4A7C15ULL * (uint64_t)(j + 1);
    for (int r = 0; r < n; ++r) {
        st ^= st << 13; st ^= st >> 7; st ^= st << 17;
        Z[r * N + j] = 0.5 + (double)(st >> 11) * 0x1p-53;
    }
    for (int iter = 0; iter < 3; ++iter) {
        // forward: apply L^{-1} (with the recorded interchanges)
        for (int r = 0; r < n - 1; ++r) {
            double xr = Z[r * N + j], xn = Z[(r + 1) * N + j];
            if (PV[r * N + j] != 0.0) { const double t = xr; xr = xn; xn = t; }
            Z[r * N + j] = xr;
            Z[(r + 1) * N + j] = xn - ML[r * N + j] * xr;
        }
        // backward: U x = y
        for (int r = n - 1; r >= 0; --r) {
            double s = Z[r * N + j];
            if (r + 1 < n) s -= U2[r * N + j] * Z[(r + 1) * N + j];
            if (r + 2 < n) s -= U3[r * N + j] * Z[(r + 2) * N + j];
            Z[r * N + j] = s / U1[r * N + j];
        }
        // normalise
        double nrm = 0.0;
        for (int r = 0; r < n; ++r) nrm += Z[r * N + j] * Z[r * N + j];
        nrm = 1.0 / sqrt(nrm);
        for (int r = 0; r < n; ++r) Z[r * N + j] *= nrm;
    }
}

// MGS inside clusters: one warp per cluster start (eigenvalue j that begins a
// run of values within tol of each other).
__global__ void reorth_kernel(const double* __restrict__ W, int n, const double* tnorm_p,
                              double* Z) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= n) return;
    const double tol = 1e-10 * fmax(*tnorm_p, 1e-300);
    const int j0 = warp;
    if (j0 > 0 && fabs(W[j0 - 1] - W[j0]) <= tol) return;  // not a cluster start
    int j1 = j0 + 1;
    while (j1 < n && fabs(W[j1 - 1] - W[j1]) <= tol) ++j1;
    if (j1 - j0 < 2) return;
    const int64_t N = n;
    for (int a = j0; a < j1; ++a) {
        for (int b = j0; b < a; ++b) {
            double dot = 0.0;
            for (int r = lane; r < n; r += 32) dot += Z[r * N + a] * Z[r * N + b];
            dot = warp_sum(dot);
            for (int r = lane; r < n; r += 32) Z[r * N + a] -= dot * Z[r * N + b];
        }
        double nrm = 0.0;
        for (int r = lane; r < n; r += 32) nrm += Z[r * N + a] * Z[r * N + a];
        nrm = warp_sum(nrm);
        nrm = 1.0 / sqrt(nrm);
        for (int r = lane; r < n; r += 32) Z[r * N + a] *= nrm;
    }
}

// V[:, j] = H_0 ... H_{n-3} Z[:, j]; one warp per column, reflectors applied
// from the last to the first (H_i = I - tau_i v_i v_i^T on rows i+1..n-1).
__global__ void backtr_kernel(const double* __restrict__ Z, int n, const double* __restrict__ tau,
                              const double* __restrict__ Hv, double* __restrict__ scr,
                              double* __restrict__ V) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= n) return;
    const int64_t N = n;
    const int j = warp;
    double* x = scr + (int64_t)j * N;  // contiguous working copy of column j
    for (int r = lane; r < n; r += 32) x[r] = Z[r * N + j];
    __syncwarp();
    for (int i = n - 3; i >= 0; --i) {
        const double t = tau[i];
        if (t == 0.0) continue;
        const double* v = Hv + (int64_t)i * N;
        double dot = 0.0;
        for (int r = i + 1 + lane; r < n; r += 32) dot += v[r] * x[r];
        dot = warp_sum(dot) * t;
        for (int r = i + 1 + lane; r < n; r += 32) x[r] -= dot * v[r];
        __syncwarp();
    }
    for (int r = lane; r < n; r += 32) V[r * N + j] = x[r];
}

}  // namespace

int64_t syev_tri_ws_bytes(int64_t n) {
    // A copy, Hv, 5 n^2 inverse-iteration scratch, Z, backtr scratch, vectors
    return (int64_t)sizeof(double) * (2 * n * n + 5 * n * n + n * n + n * n + 8 * n + 64) + 256;
}

int syev_tri(const double* A, int64_t n, double* W, double* V, void* ws, int64_t ws_bytes,
             int32_t* sweeps, cudaStream_t st) {
    if (ws_bytes < syev_tri_ws_bytes(n)) {
        set_error("syev_tri: workspace too small");
        return SKP_ERR_ARG;
    }
    double* Ac = reinterpret_cast<double*>(ws);
    double* Hv = Ac + n * n;
    double* scr = Hv + n * n;          // 5 n^2
    double* Z = scr + 5 * n * n;       // n^2
    double* bscr = Z + n * n;          // n^2
    double* d = bscr + n * n;
    double* e = d + n;
    double* tau = e + n;
    double* pbuf = tau + n;
    double* tnorm = pbuf + n;
    SKP_CUDA(cudaMemcpyAsync(Ac, A, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st));
    SKP_CUDA(cudaMemsetAsync(Hv, 0, sizeof(double) * n * n, st));
    int dev = 0, sms = 148, per_sm = 0;
    SKP_CUDA(cudaGetDevice(&dev));
    SKP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    SKP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sytrd_kernel, kTriThreads, 0));
    if (per_sm < 1) {
        set_error("syev_tri: cooperative kernel cannot be resident");
        return SKP_ERR_CUDA;
    }
    int nn = (int)n;
    void* args[] = {&Ac, &nn, &d, &e, &tau, &Hv, &pbuf};
    SKP_CUDA(cudaLaunchCooperativeKernel((void*)sytrd_kernel, dim3(sms), dim3(kTriThreads), args, 0,
                                         st));
    count_launch();
    const size_t bsm = 2 * (size_t)n * sizeof(double);
    SKP_CUDA(cudaFuncSetAttribute(bisect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)std::max<size_t>(bsm, 1)));
    bisect_kernel<<<(unsigned)cdiv(n, 128), 128, bsm, st>>>(d, e, nn, W, tnorm);
    SKP_LAUNCHED(bisect_kernel);
    inviter_kernel<<<(unsigned)cdiv(n, 64), 64, 0, st>>>(d, e, nn, W, tnorm, scr, Z);
    SKP_LAUNCHED(inviter_kernel);
    reorth_kernel<<<(unsigned)cdiv(n * 32, 256), 256, 0, st>>>(W, nn, tnorm, Z);
    SKP_LAUNCHED(reorth_kernel);
    backtr_kernel<<<(unsigned)cdiv(n * 32, 256), 256, 0, st>>>(Z, nn, tau, Hv, bscr, V);
    SKP_LAUNCHED(backtr_kernel);
    if (sweeps) SKP_CUDA(cudaMemsetAsync(sweeps, 0, sizeof(int32_t), st));
    return SKP_OK;
}

}  // namespace skp
