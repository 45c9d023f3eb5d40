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
#include <stdlib.h>

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
// Per column i, 2 grid syncs:
//   every CTA stages column i (below the diagonal) in smem and builds the
//   reflector v there (redundantly -- no sync); p = tau A' v, one warp per row
//   (coalesced rows, v from smem); sync; every CTA forms w = p - K v in smem;
//   the rank-2 update A' -= v w^T + w v^T by rows (row -> CTA, columns ->
//   threads: no index division); sync.
// smem: v[n], w[n] (dynamic).
__global__ void __launch_bounds__(kTriThreads)
sytrd_kernel(double* A, int n, int i_end, double* d, double* e, double* tau, double* Hv,
             double* pbuf) {
    extern __shared__ double tsm[];
    double* vs = tsm;         // v over rows r0.. (index t = row - r0)
    double* ws = tsm + n;     // w
    __shared__ double scratch[32];
    cg::grid_group grid = cg::this_grid();
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int warp_g = (int)(gtid >> 5), lane = threadIdx.x & 31;
    const int nwarps_g = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
    for (int i = 0; i < i_end && i + 2 < n; ++i) {
        const int r0 = i + 1, k = n - r0;
        // (a) reflector from x = A[r0:, i] (untouched by this step's update)
        double ss = 0.0;
        for (int t = threadIdx.x; t < k; t += blockDim.x) {
            const double x = A[(int64_t)(r0 + t) * n + i];
            vs[t] = x;
            if (t > 0) ss += x * x;
        }
        const double xnorm2 = block_reduce_sum_all(ss, scratch);   // (syncs the block)
        const double alpha = vs[0];
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
        for (int t = threadIdx.x; t < k; t += blockDim.x) vs[t] = t == 0 ? 1.0 : vs[t] * scal;
        __syncthreads();
        // (b) p = tau * A' v, one warp per row of A' = A[r0:, r0:]
        if (t_ != 0.0) {
            for (int rr = warp_g; rr < k; rr += nwarps_g) {
                const double* row = A + (int64_t)(r0 + rr) * n + r0;
                double acc = 0.0;
                for (int t = lane; t < k; t += 32) acc += row[t] * vs[t];
                acc = warp_sum(acc);
                if (lane == 0) pbuf[rr] = t_ * acc;
            }
        }
        if (gtid == 0) {
            d[i] = A[(int64_t)i * n + i];
            e[i] = beta;
            tau[i] = t_;
        }
        // store v_i for the back-transformation (row i of Hv)
        for (int64_t t = gtid; t < k; t += (int64_t)gridDim.x * blockDim.x)
            Hv[(int64_t)i * n + r0 + t] = vs[t];
        grid.sync();
        if (t_ != 0.0) {
            // (c) K = tau/2 * p.v ; w = p - K v   (redundant per CTA, into smem)
            double pv = 0.0;
            for (int t = threadIdx.x; t < k; t += blockDim.x) {
                const double pt = pbuf[t];
                ws[t] = pt;
                pv += pt * vs[t];
            }
            const double K = 0.5 * t_ * block_reduce_sum_all(pv, scratch);
            for (int t = threadIdx.x; t < k; t += blockDim.x) ws[t] -= K * vs[t];
            __syncthreads();
            // (d) A' -= v w^T + w v^T: rows over CTAs, columns over threads
            for (int rr = blockIdx.x; rr < k; rr += gridDim.x) {
                double* row = A + (int64_t)(r0 + rr) * n + r0;
                const double vr = vs[rr], wr = ws[rr];
                for (int cc = threadIdx.x; cc < k; cc += blockDim.x)
                    row[cc] -= vr * ws[cc] + wr * vs[cc];
            }
        }
        grid.sync();
    }
    if (gtid == 0 && i_end >= n - 2) {  // (else the cluster kernel finishes the trailing block)
        if (n >= 2) {
            d[n - 2] = A[(int64_t)(n - 2) * n + n - 2];
            e[n - 2] = A[(int64_t)(n - 1) * n + n - 2];
            tau[n - 2] = 0.0;
        }
        d[n - 1] = A[(int64_t)(n - 1) * n + n - 1];
    }
}

// ---- cluster tridiagonalisation: the whole matrix in distributed smem -------
// A cluster of kCl CTAs (one per SM) holds A row-interleaved in shared memory
// (row r -> CTA r % kCl, local row r / kCl); per column: the owners broadcast
// column i and their norm partials by DSMEM stores, cluster barrier, every CTA
// builds v and computes p for its rows, broadcasts p and p.v partials, cluster
// barrier, every CTA forms w and updates its rows.  No global-memory round
// trips and hardware cluster barriers instead of grid syncs.  Exchange buffers
// alternate with the column parity (a CTA is never more than one phase ahead).
constexpr int kCl = 16;
constexpr int kClThreads = 512;

__device__ __forceinline__ uint32_t cl_smem(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cl_mapa(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void cl_st(uint32_t a, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
// remote store that completes `8 bytes` on the destination's mbarrier
__device__ __forceinline__ void cl_st_async(uint32_t a, double v, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(a),
                 "d"(v), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void cl_arm(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void cl_wait(uint32_t bar, uint32_t parity) {
    long long t0 = 0;
    for (int it = 0;; ++it) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
        if (ok) return;
        // watchdog: a protocol bug becomes a trap (error), never a hung GPU
        if (it == 64) t0 = clock64();
        if (it > 64 && (it & 1023) == 0 && clock64() - t0 > (long long)40e9) __trap();
    }
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" :::
                     "memory");
}

__global__ void __launch_bounds__(kClThreads, 1)
sytrd_cluster_kernel(const double* __restrict__ Ag, int lda, int n, int rpc, double* d,
                     double* e, double* tau, double* Hv, int ldh) {
    extern __shared__ __align__(16) double csm[];
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    // layout: A rows [rpc][n] | xv[2][n] | pv[2][n] | ssp[2][kCl] | pvp[2][kCl] | vs[n] | ws[n]
    double* Al = csm;
    double* xv = Al + (size_t)rpc * n;
    double* pvv = xv + 2 * (size_t)n;
    double* ssp = pvv + 2 * (size_t)n;
    double* pvp = ssp + 2 * kCl;
    double* vs = pvp + 2 * kCl;
    double* wsv = vs + n;
    __shared__ double scratch[32];
    // exchange completion: xbar[par] (column i's entries + norm partials),
    // pbar[par] (p and p.v partials); each CTA arms its own for the bytes it
    // will receive and the senders' st.async complete them -- no cluster
    // barrier per exchange.  A sender is never more than one column ahead of a
    // receiver's reads of a buffer: to send column i + 2 it needs every CTA's
    // p of column i + 1, sent after that CTA finished column i.
    __shared__ __align__(8) uint64_t xbar[2], pbar[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    auto xbytes = [&](int i) { return (uint32_t)(8 * ((n - 1 - i) + kCl)); };
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cl_smem(&xbar[b])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cl_smem(&pbar[b])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < 2 && i + 2 < n; ++i) {  // columns 0 and 1
            cl_arm(cl_smem(&xbar[i]), xbytes(i));
            cl_arm(cl_smem(&pbar[i]), xbytes(i));
        }
    }
    // load owned rows
    for (int lr = 0; lr < rpc; ++lr) {
        const int r = lr * kCl + (int)rank;
        for (int c = tid; c < n; c += blockDim.x) Al[(size_t)lr * n + c] = r < n ? Ag[(int64_t)r * lda + c] : 0.0;
    }
    cl_sync();  // every CTA's rows loaded and barriers armed
    const uint32_t xv_a = cl_smem(xv), pv_a = cl_smem(pvv), ssp_a = cl_smem(ssp), pvp_a = cl_smem(pvp);
    const uint32_t xb_a = cl_smem(&xbar[0]), pb_a = cl_smem(&pbar[0]);
    for (int i = 0; i + 2 < n; ++i) {
        const int par = i & 1;
        const uint32_t ph = (uint32_t)((i >> 1) & 1);  // use i / 2 of each barrier
        const int r0 = i + 1, k = n - r0;
        // (1) broadcast column i of my rows r > i, and sum_{r > r0} x_r^2
        double ss = 0.0;
        for (int q = tid; q < rpc * kCl; q += blockDim.x) {
            const int lr = q / kCl, dst = q % kCl;
            const int r = lr * kCl + (int)rank;
            if (r <= i || r >= n) continue;
            const double x = Al[(size_t)lr * n + i];
            if (dst == 0 && r > r0) ss += x * x;
            cl_st_async(cl_mapa(xv_a + 8u * (uint32_t)(par * n + r), (uint32_t)dst), x,
                        cl_mapa(xb_a + 8u * par, (uint32_t)dst));
        }
        ss = warp_sum(ss);
        if (lane == 0) scratch[warp] = ss;
        __syncthreads();
        if (tid < kCl) {
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += scratch[w];
            cl_st_async(cl_mapa(ssp_a + 8u * (uint32_t)(par * kCl + (int)rank), (uint32_t)tid), t,
                        cl_mapa(xb_a + 8u * par, (uint32_t)tid));
        }
        cl_wait(xb_a + 8u * par, ph);
        if (tid == 0 && i + 4 < n) cl_arm(xb_a + 8u * par, xbytes(i + 2));  // column i + 2
        // (2) reflector (every CTA), p for my rows, broadcast p and p.v partials
        double xnorm2 = 0.0;
        for (int c = 0; c < kCl; ++c) xnorm2 += ssp[par * kCl + c];
        const double* xcol = xv + (size_t)par * n;
        const double alpha = xcol[r0];
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
        for (int c = r0 + tid; c < n; c += blockDim.x) vs[c] = c == r0 ? 1.0 : xcol[c] * scal;
        if (rank == 0) {
            if (tid == 0) {
                e[i] = beta;
                tau[i] = t_;
            }
            for (int c = r0 + tid; c < n; c += blockDim.x)
                Hv[(int64_t)i * ldh + c] = c == r0 ? 1.0 : xcol[c] * scal;
        }
        if ((i % kCl) == (int)rank && tid == 0) d[i] = Al[(size_t)(i / kCl) * n + i];
        __syncthreads();
        double pvpart = 0.0;
        for (int lr = warp; lr < rpc; lr += nw) {
            const int r = lr * kCl + (int)rank;
            if (r < r0 || r >= n) continue;
            const double* row = Al + (size_t)lr * n;
            double acc = 0.0;
            for (int c = r0 + lane; c < n; c += 32) acc += row[c] * vs[c];
            acc = warp_sum(acc) * t_;
            if (lane < kCl)
                cl_st_async(cl_mapa(pv_a + 8u * (uint32_t)(par * n + r), (uint32_t)lane), acc,
                            cl_mapa(pb_a + 8u * par, (uint32_t)lane));
            pvpart += acc * vs[r];
        }
        if (lane == 0) scratch[warp] = pvpart;
        __syncthreads();
        if (tid < kCl) {
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += scratch[w];
            cl_st_async(cl_mapa(pvp_a + 8u * (uint32_t)(par * kCl + (int)rank), (uint32_t)tid), t,
                        cl_mapa(pb_a + 8u * par, (uint32_t)tid));
        }
        cl_wait(pb_a + 8u * par, ph);
        if (tid == 0 && i + 4 < n) cl_arm(pb_a + 8u * par, xbytes(i + 2));
        // (3) w = p - K v ; update my rows  A[r][c] -= v_r w_c + w_r v_c  (r, c > i)
        if (t_ != 0.0) {
            double pv = 0.0;
            for (int c = 0; c < kCl; ++c) pv += pvp[par * kCl + c];
            const double K = 0.5 * t_ * pv;
            const double* pcol = pvv + (size_t)par * n;
            for (int c = r0 + tid; c < n; c += blockDim.x) wsv[c] = pcol[c] - K * vs[c];
            __syncthreads();
            for (int lr = warp; lr < rpc; lr += nw) {
                const int r = lr * kCl + (int)rank;
                if (r < r0 || r >= n) continue;
                double* row = Al + (size_t)lr * n;
                const double vr = vs[r], wr = wsv[r];
                for (int c = r0 + lane; c < n; c += 32) row[c] -= vr * wsv[c] + wr * vs[c];
            }
        }
        __syncthreads();
    }
    cl_sync();
    if (n >= 2) {
        if (((n - 2) % kCl) == (int)rank && tid == 0) {
            d[n - 2] = Al[(size_t)((n - 2) / kCl) * n + n - 2];
            tau[n - 2] = 0.0;
        }
        if (((n - 1) % kCl) == (int)rank && tid == 0) e[n - 2] = Al[(size_t)((n - 1) / kCl) * n + n - 2];
    }
    if (((n - 1) % kCl) == (int)rank && tid == 0) d[n - 1] = Al[(size_t)((n - 1) / kCl) * n + n - 1];
}

size_t sytrd_cluster_smem(int n) {
    const int rpc = (n + kCl - 1) / kCl;
    return sizeof(double) * ((size_t)rpc * n + 4 * (size_t)n + 4 * kCl + 2 * (size_t)n);
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

// One WARP per eigenvalue: 32 lanes evaluate Sturm counts at 32 interior
// points of the bracket, which then shrinks 33x per round (~11 rounds to
// machine precision instead of ~55 bisection steps).
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
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    for (int i = blockIdx.x * wpb + (threadIdx.x >> 5); i < n; i += gridDim.x * wpb) {
        // (i+1)-th largest: the value x with count(x) <= n-1-i < count(x')
        const int target = n - 1 - i;  // number of eigenvalues below it
        double lo = lo_s, hi = hi_s;
        for (int it = 0; it < 64; ++it) {
            if (hi - lo <= width) break;
            const double step = (hi - lo) / 33.0;
            const double x = lo + step * (lane + 1);
            const bool above = x < hi && x > lo && sturm_count(d, e2, n, x, pivmin) > target;
            // first lane whose point already has more than `target` below it
            const unsigned mask = __ballot_sync(0xffffffffu, above);
            const int k = mask ? __ffs(mask) - 1 : 32;   // points 0..k-1 are "not above"
            const double nlo = k > 0 ? lo + step * k : lo;
            const double nhi = k < 32 ? lo + step * (k + 1) : hi;
            if (!(nlo > lo || nhi < hi)) break;          // no progress at this resolution
            lo = nlo;
            hi = nhi;
        }
        if (lane == 0) W[i] = 0.5 * (lo + hi);
    }
}

// Inverse iteration: thread j computes eigenvector j of T for lambda = W[j].
// Scratch per thread (interleaved [row][j], coalesced across a warp): 1/u1,
// u2, u3 (the U bands), the multiplier and the interchange flag of a
// partially pivoted tridiagonal LU (LAPACK dlagtf / dlagts scheme).  Every
// recurrence carries its running values in REGISTERS -- global memory only
// holds the previous pass's vector, whose loads do not depend on the chain (a
// store-then-reload per step made each step a global round trip).  The
// normalisation is folded into the next pass.  Z (n x n) receives column j.
__global__ void __launch_bounds__(64)
inviter_kernel(const double* __restrict__ d, const double* __restrict__ e, int n,
               const double* __restrict__ W, const double* __restrict__ tnorm_p,
               double* __restrict__ scr, double* __restrict__ Z) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int64_t N = n;
    double* IU1 = scr;
    double* U2 = scr + N * N;
    double* U3 = scr + 2 * N * N;
    double* ML = scr + 3 * N * N;
    double* PV = scr + 4 * N * N;
    const double tn = fmax(*tnorm_p, 1e-300);
    const double lam = W[j];
    const double eps_piv = 2.2e-16 * tn;
    // LU with partial pivoting of (T - lam I), rows r, r+1 interchange
    double a = d[0] - lam;              // current diag candidate of row r
    double b = n > 1 ? e[0] : 0.0;      // super diag of row r
    double c3 = 0.0;                    // 2nd super of row r (from a previous swap)
    for (int r = 0; r < n - 1; ++r) {
        const double sub = e[r];                  // T[r+1][r]
        const double dnext = d[r + 1] - lam;      // T[r+1][r+1]
        const double snext = r + 1 < n - 1 ? e[r + 1] : 0.0;  // T[r+1][r+2]
        if (fabs(a) >= fabs(sub)) {
            double piv = a;
            if (fabs(piv) < eps_piv) piv = copysign(eps_piv, piv == 0.0 ? 1.0 : piv);
            const double ip = 1.0 / piv;
            const double m = sub * ip;
            IU1[r * N + j] = ip;
            U2[r * N + j] = b;
            U3[r * N + j] = c3;
            ML[r * N + j] = m;
            PV[r * N + j] = 0.0;
            a = dnext - m * b;
            b = snext - m * c3;
            c3 = 0.0;
        } else {
            const double m = a / sub;
            IU1[r * N + j] = 1.0 / sub;
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
        IU1[(N - 1) * N + j] = 1.0 / piv;
        U2[(N - 1) * N + j] = 0.0;
        U3[(N - 1) * N + j] = 0.0;
    }
    // start vector: deterministic pseudo-random
    uint64_t st = 0x9E3779B97F4A7C15ULL * (uint64_t)(j + 1);
    for (int r = 0; r < n; ++r) {
        st ^= st << 13; st ^= st >> 7; st ^= st << 17;
        Z[r * N + j] = 0.5 + (double)(st >> 11) * 0x1p-53;
    }
    // The recurrences below are sequential in r, but their operands are not:
    // each group of kIvG rows is loaded up front (independent loads in
    // flight together) and then consumed -- one L2 round trip per group
    // instead of per row (1.1 ms -> ~0.1 ms at n = 520).
    constexpr int kIvG = 16;
    double scale = 1.0;
    for (int iter = 0; iter < 3; ++iter) {
        // forward: apply L^{-1} with the recorded interchanges (scale folded in)
        double carry = Z[j] * scale;
        for (int r0 = 0; r0 < n - 1; r0 += kIvG) {
            double zn[kIvG], pv[kIvG], ml[kIvG];
#pragma unroll
            for (int u = 0; u < kIvG; ++u) {
                const int r = r0 + u;
                if (r < n - 1) {
                    zn[u] = Z[(r + 1) * N + j];
                    pv[u] = PV[r * N + j];
                    ml[u] = ML[r * N + j];
                }
            }
#pragma unroll
            for (int u = 0; u < kIvG; ++u) {
                const int r = r0 + u;
                if (r < n - 1) {
                    double xr = carry, xn = zn[u] * scale;
                    if (pv[u] != 0.0) { const double t = xr; xr = xn; xn = t; }
                    Z[r * N + j] = xr;
                    carry = xn - ml[u] * xr;
                }
            }
        }
        Z[(N - 1) * N + j] = carry;
        // backward: U x = y, carrying x_{r+1}, x_{r+2}; sum of squares on the fly
        double x1 = 0.0, x2 = 0.0, nrm = 0.0;
        for (int r1 = n - 1; r1 >= 0; r1 -= kIvG) {
            double zr[kIvG], u2[kIvG], u3[kIvG], iu[kIvG];
#pragma unroll
            for (int u = 0; u < kIvG; ++u) {
                const int r = r1 - u;
                if (r >= 0) {
                    zr[u] = Z[r * N + j];
                    u2[u] = U2[r * N + j];
                    u3[u] = U3[r * N + j];
                    iu[u] = IU1[r * N + j];
                }
            }
#pragma unroll
            for (int u = 0; u < kIvG; ++u) {
                const int r = r1 - u;
                if (r >= 0) {
                    const double x = (zr[u] - u2[u] * x1 - u3[u] * x2) * iu[u];
                    Z[r * N + j] = x;
                    nrm += x * x;
                    x2 = x1;
                    x1 = x;
                }
            }
        }
        scale = 1.0 / sqrt(nrm);
    }
#pragma unroll 8
    for (int r = 0; r < n; ++r) Z[r * N + j] *= scale;
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
// The column lives in registers (lane holds rows lane + 32 m); the reflectors
// (2 MB for n = 520) are read from L2 by every warp.
constexpr int kBtMaxM = 34;  // rows per lane: n <= 1088 in registers (C5: r2 = 1050)
template <int M>
__global__ void __launch_bounds__(256)
backtr_kernel(const double* __restrict__ Z, int n, const double* __restrict__ tau,
              const double* __restrict__ Hv, double* __restrict__ V) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= n) return;
    const int64_t N = n;
    const int j = warp;
    double x[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const int r = lane + 32 * m;
        x[m] = r < n ? Z[r * N + j] : 0.0;
    }
    // software-pipelined: reflector i-1 is loaded while reflector i is applied
    // (each load was an exposed L2 round trip per reflector: 455 us at n = 520)
    double vn[M];
    double tn = 0.0;
    auto load = [&](int i) {
        const double* v = Hv + (int64_t)i * N;
        tn = __ldg(tau + i);
#pragma unroll
        for (int m = 0; m < M; ++m) {
            const int r = lane + 32 * m;
            vn[m] = (r > i && r < n) ? __ldg(v + r) : 0.0;
        }
    };
    if (n >= 3) load(n - 3);
    for (int i = n - 3; i >= 0; --i) {
        double vv[M];
#pragma unroll
        for (int m = 0; m < M; ++m) vv[m] = vn[m];
        const double t = tn;
        if (i > 0) load(i - 1);
        if (t == 0.0) continue;
        double d0 = 0.0, d1 = 0.0;  // two chains: the fp64 FMA latency, not the rate
#pragma unroll
        for (int m = 0; m < M; m += 2) {
            d0 += vv[m] * x[m];
            if (m + 1 < M) d1 += vv[m + 1] * x[m + 1];
        }
        const double dot = warp_sum(d0 + d1) * t;
#pragma unroll
        for (int m = 0; m < M; ++m) x[m] -= dot * vv[m];
    }
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const int r = lane + 32 * m;
        if (r < n) V[r * N + j] = x[m];
    }
}

// generic fallback (n > 32 * kBtMaxM): column in global scratch
__global__ void backtr_kernel_big(const double* __restrict__ Z, int n, const double* __restrict__ tau,
                                  const double* __restrict__ Hv, double* __restrict__ scr,
                                  double* __restrict__ V) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= n) return;
    const int64_t N = n;
    const int j = warp;
    double* x = scr + (int64_t)j * N;
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
    const size_t tsm = 2 * (size_t)n * sizeof(double);
    SKP_CUDA(cudaFuncSetAttribute(sytrd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)std::max<size_t>(tsm, 1)));
    SKP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sytrd_kernel, kTriThreads, tsm));
    if (per_sm < 1) {
        set_error("syev_tri: cooperative kernel cannot be resident");
        return SKP_ERR_CUDA;
    }
    int nn = (int)n;
    // The trailing block of the reduction runs in a 16-CTA cluster's shared
    // memory (DSMEM exchanges and mbarriers instead of grid syncs: ~2x faster
    // per column): the whole matrix when it fits, else the grid kernel reduces
    // the leading columns until the trailing block fits (C5's r2 = 1050: 410
    // columns on the grid, the last 640 in the cluster).
    int nc = 0;  // trailing block size for the cluster (0: none)
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    {
        int cand = nn;
        while (cand > 2 && sytrd_cluster_smem(cand) > 220 * 1024) --cand;
        const size_t csm = sytrd_cluster_smem(cand);
        cudaError_t ea = cudaFuncSetAttribute(sytrd_cluster_kernel,
                                              cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaError_t eb = cudaFuncSetAttribute(sytrd_cluster_kernel,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
        if (cand > 2 && ea == cudaSuccess && eb == cudaSuccess) {
            cfg.gridDim = dim3(kCl);
            cfg.blockDim = dim3(kClThreads);
            cfg.dynamicSmemBytes = csm;
            cfg.stream = st;
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = kCl;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            int ncl = 0;
            if (cudaOccupancyMaxActiveClusters(&ncl, sytrd_cluster_kernel, &cfg) == cudaSuccess &&
                ncl >= 1)
                nc = cand;
        }
        cudaGetLastError();  // clear a refused attribute / occupancy query
    }
    const int i0 = nc ? nn - nc : nn;  // columns reduced by the grid kernel
    if (i0 > 0) {
        int iend = i0;
        void* args[] = {&Ac, &nn, &iend, &d, &e, &tau, &Hv, &pbuf};
        SKP_CUDA(cudaLaunchCooperativeKernel((void*)sytrd_kernel, dim3(sms), dim3(kTriThreads), args,
                                             tsm, st));
        count_launch();
    }
    if (nc) {
        const int rpc = (nc + kCl - 1) / kCl;
        const int64_t off = (int64_t)i0 * nn + i0;
        SKP_CUDA(cudaLaunchKernelEx(&cfg, sytrd_cluster_kernel, (const double*)(Ac + off), nn, nc,
                                    rpc, d + i0, e + i0, tau + i0, Hv + off, nn));
        SKP_LAUNCHED(sytrd_cluster_kernel);
    }
    const size_t bsm = 2 * (size_t)n * sizeof(double);
    SKP_CUDA(cudaFuncSetAttribute(bisect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)std::max<size_t>(bsm, 1)));
    // 2 warps (eigenvalues) per block: the launch spreads over all SMs
    bisect_kernel<<<(unsigned)cdiv(n, 2), 64, bsm, st>>>(d, e, nn, W, tnorm);
    SKP_LAUNCHED(bisect_kernel);
    inviter_kernel<<<(unsigned)cdiv(n, 32), 32, 0, st>>>(d, e, nn, W, tnorm, scr, Z);
    SKP_LAUNCHED(inviter_kernel);
    reorth_kernel<<<(unsigned)cdiv(n * 32, 256), 256, 0, st>>>(W, nn, tnorm, Z);
    SKP_LAUNCHED(reorth_kernel);
    {
        const unsigned bgrid = (unsigned)cdiv(n * 32, 64);  // 2 columns per block: all SMs
        if (n <= 32 * 17) backtr_kernel<17><<<bgrid, 64, 0, st>>>(Z, nn, tau, Hv, V);
        else if (n <= 32 * kBtMaxM) backtr_kernel<kBtMaxM><<<bgrid, 64, 0, st>>>(Z, nn, tau, Hv, V);
        else backtr_kernel_big<<<bgrid, 64, 0, st>>>(Z, nn, tau, Hv, bscr, V);
        SKP_LAUNCHED(backtr_kernel);
    }
    if (sweeps) SKP_CUDA(cudaMemsetAsync(sweeps, 0, sizeof(int32_t), st));
    return SKP_OK;
}

}  // namespace skp
