// K5 v2: fused Cholesky + rank check + triangular inverse (fp64), one
// cooperative kernel, for CholeskyQR's r2 x r2 Gram matrices.
//
//   G = L L^T  ->  X = L^{-1}   (X dense n x n, strict upper zero)
//
// 32-wide panels on a zero/identity-padded copy (npad = 32 * nb):
//   per panel p  (1) CTA 0 factors the 32x32 diagonal block in smem and
//                    inverts it (L_pp, L_pp^{-1}), tracking min/max pivots;
//                (2) all CTAs: L_ip = A_ip L_pp^{-T} for the rows below;
//                (3) all CTAs: trailing update A_IJ -= L_Ip L_Jp^T (32x32 tiles).
//   then the inverse by block columns: one CTA per block column J keeps
//   X[:, J] in shared memory and sweeps down it,
//                X_IJ = -L_II^{-1} sum_{K=J}^{I-1} L_IK X_KJ,
//   independent of the other columns (no grid syncs).
// ~3 nb grid syncs in total instead of ~30 launches + a serial inverse.
// shift_rel > 0: factor G + shift_rel * max_i G_ii * I instead (shifted
// CholeskyQR: a Gram whose noise floor would give a non-positive pivot still
// factors, and range(Y L^{-T}) = range(Y) is kept; see _engine.orthonormalize).
// info: left untouched on success; set to k+1 if pivot k is not
// positive/finite, -1 if min L_ii < rel_tol * max L_ii (numerically rank
// deficient -> eigen-based path).  Callers zero it; failures accumulate, so one
// flag can cover a whole sync-free sequence of factorisations.
#include <cooperative_groups.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace skp {
namespace {

constexpr int CB = 32;
constexpr int kCIThreads = 256;

struct CIShared {
    double a[CB][CB + 1];
    double b[CB][CB + 1];
    double c[CB][CB + 1];
    double e[CB][CB + 1];
    double xpp[CB][CB + 1];  // CTA 0: L_pp^{-1} of its last factorisation (no reload)
    double dmn, dmx;         // CTA 0: running pivot range (written to dinfo at the end)
    int info0;               // CTA 0: first failing pivot
    double invd[CB];
    int bad;
};

// C[32x32] (smem) -= X[32x32] * Y^T  (op 0) or  C = X * Y (op 1); 256 threads, 4 outputs each
__device__ __forceinline__ void tile_mm(double (*C)[CB + 1], double (*X)[CB + 1],
                                        double (*Y)[CB + 1], int op, double alpha, bool accumulate) {
    const int tr = threadIdx.x / 8, tc = (threadIdx.x % 8) * 4;
    double acc[4] = {0, 0, 0, 0};
    for (int k = 0; k < CB; ++k) {
        const double x = X[tr][k];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] += x * (op == 0 ? Y[tc + j][k] : Y[k][tc + j]);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 4; ++j)
        C[tr][tc + j] = accumulate ? C[tr][tc + j] + alpha * acc[j] : alpha * acc[j];
    __syncthreads();
}

// 1/sqrt(d) to fp64 accuracy: the fp32 estimate (MUFU, ~23 bits) and two
// Newton steps (46 -> full); the IEEE sqrt + divide chain costs ~10x more and
// sits on the factorisation's critical path 64 times per 32x32 tile
__device__ __forceinline__ double rsqrt64(double d) {   // d > 0, finite, normal
    // d = m * 4^h with m in [1, 4): exact power-of-four scaling from the
    // exponent bits keeps the fp32 estimate in range with no calls or branches
    // (an out-of-line sqrt / divide forced register spills around the loop)
    const int e = ((__double2hiint(d) >> 20) & 0x7ff) - 1023;
    const int h = e >> 1;
    const double m = d * __hiloint2double((1023 - 2 * h) << 20, 0);
    double y = (double)rsqrtf((float)m);
    const double hm = 0.5 * m;
    y = y * fma(-hm * y, y, 1.5);
    y = y * fma(-hm * y, y, 1.5);
    return y * __hiloint2double((1023 - h) << 20, 0);
}

// 32x32 SPD tile T (smem, lower part) -> L into T (lower, upper zeroed) and
// L^{-1} into Li, by the whole block (block-uniform; 256 threads):
//   Cholesky, right-looking on the UNSCALED columns: step k reads the pivot
//   d_k = T[k][k] and updates T[i][j] -= T[i][k] T[j][k] / d_k for
//   k < j <= i -- column k is never written again, so one block barrier per
//   step suffices; each thread owns <= 3 fixed (i, j) entries of the lower
//   triangle (no per-step index arithmetic).  Afterwards L_ij = T_ij / sqrt(d_j)
//   in one pass.  (Scaling the column in place took 3 barriers per step and a
//   triangular index decode per entry: 18.8 us per tile.)
//   inverse by recursive doubling: with the diagonal 1/L_ii, level b = 1..16
//   fills every off-diagonal block of the inverse at once,
//   X21 = -X22 (L21 X11), one output entry per thread, 2 barriers per level.
// Returns the first bad pivot (1-based in the tile, 0 if none) and the pivot
// range via *mn / *mx.
__device__ __forceinline__ int tile_chol_inv(double (*T)[CB + 1], double (*Li)[CB + 1],
                                             double (*W)[CB + 1], double* invd, double* mn,
                                             double* mx) {
    __shared__ int s_bad;
    __shared__ double s_mn, s_mx;
    __shared__ double s_d[CB];
    const int tid = threadIdx.x;
    // owned lower-triangle entries (i >= j), linear index t = i (i + 1) / 2 + j
    int oi[3], oj[3];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
        const int t = tid + u * 256;
        int r = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
        while (r * (r + 1) / 2 > t) --r;
        while ((r + 1) * (r + 2) / 2 <= t) ++r;
        oi[u] = t < CB * (CB + 1) / 2 ? r : -1;
        oj[u] = t - r * (r + 1) / 2;
    }
    if (tid == 0) s_bad = 0;
    for (int k = 0; k < CB; ++k) {
        __syncthreads();  // step k-1's updates (and the pivot T[k][k]) are visible
        double d = T[k][k];
        const bool ok = d > 1e-300 && isfinite(d);
        if (!ok) d = 1.0;  // keep going; the caller discards the result
        if (tid == 0) {
            if (!ok && !s_bad) s_bad = k + 1;
            s_d[k] = d;
        }
        const double rd = 1.0 / d;
#pragma unroll
        for (int u = 0; u < 3; ++u) {
            const int i = oi[u], j = oj[u];
            if (i >= 0 && j > k) T[i][j] -= (T[i][k] * rd) * T[j][k];
        }
    }
    __syncthreads();
    if (tid < CB) {
        const double is = rsqrt64(s_d[tid]);
        invd[tid] = is;  // 1 / L_jj
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 3; ++u) {
        const int i = oi[u], j = oj[u];
        if (i >= 0) T[i][j] = (i == j) ? s_d[j] * invd[j] : T[i][j] * invd[j];
    }
    if (tid == 0) {
        double lo = INFINITY, hi = 0.0;
        for (int k = 0; k < CB; ++k) {
            const double l = s_d[k] * invd[k];
            lo = fmin(lo, l);
            hi = fmax(hi, l);
        }
        s_mn = lo;
        s_mx = hi;
    }
    __syncthreads();
    for (int q = tid; q < CB * CB; q += blockDim.x) {
        const int i = q / CB, j = q % CB;
        if (j > i) T[i][j] = 0.0;
        Li[i][j] = i == j ? invd[i] : 0.0;
    }
    __syncthreads();
    for (int b = 1; b < CB; b *= 2) {
        // pairs of b x b diagonal blocks (s0, s0 + b): W = L21 X11, then X21 = -X22 W
        const int per = b * b, npairs = CB / (2 * b);
        for (int t = tid; t < npairs * per; t += blockDim.x) {
            const int q = t / per, e = t % per, r = e / b, c = e % b;
            const int s0 = q * 2 * b, s1 = s0 + b;
            double acc = 0.0;
            for (int k = 0; k < b; ++k) acc += T[s1 + r][s0 + k] * Li[s0 + k][s0 + c];
            W[s1 + r][s0 + c] = acc;
        }
        __syncthreads();
        for (int t = tid; t < npairs * per; t += blockDim.x) {
            const int q = t / per, e = t % per, r = e / b, c = e % b;
            const int s0 = q * 2 * b, s1 = s0 + b;
            double acc = 0.0;
            for (int k = 0; k < b; ++k) acc += Li[s1 + r][s1 + k] * W[s1 + k][s0 + c];
            Li[s1 + r][s0 + c] = -acc;
        }
        __syncthreads();
    }
    *mn = s_mn;
    *mx = s_mx;
    return s_bad;
}

// One cooperative kernel, ONE grid sync per 32-wide panel:
//   before panel p: L_pp and L_pp^{-1} are final (factored by CTA 0 as a
//   lookahead at the end of panel p-1); the trailing matrix holds all updates
//   through panel p-1.
//   panel p tasks (any CTA):
//     trailing tile (I, J), p < J <= I:  L_Ip = A_Ip L_pp^{-T}, L_Jp likewise
//       (recomputed per task: no separate panel solve and no extra sync),
//       A_IJ -= L_Ip L_Jp^T; the task with J = p+1 stores L_Ip;
//     inverse, one layer per panel (row p-1 of X became final in panel p-1):
//       rows r > p, J < p:  S_rJ += L_{r,p-1} X_{p-1,J};
//       row p, J < p:       X_pJ = -L_pp^{-1} (S_pJ + L_{p,p-1} X_{p-1,J})
//     (X_pJ = -L_pp^{-1} sum_{K=J}^{p-1} L_pK X_KJ, accumulated across panels
//     so every task is ONE tile product and each S tile has one writer).
//   CTA 0 takes task (p+1, p+1) first and factors the result right away.
__global__ void __launch_bounds__(kCIThreads, 1)
cholinv_kernel(const double* __restrict__ G, int n, int64_t ldg, int nb, double rel_tol,
               double shift_rel, double* A, double* Lb, double* X, double* S, double* dinfo, int32_t* info,
               unsigned long long* prof) {
    auto stamp = [&](int slot) {
        if (prof && blockIdx.x == 0 && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            prof[slot] = t;
        }
    };
    extern __shared__ __align__(16) unsigned char smraw[];
    CIShared& sh = *reinterpret_cast<CIShared*>(smraw);
    double (*sd)[CB + 1] = reinterpret_cast<double (*)[CB + 1]>(smraw + sizeof(CIShared));
    cg::grid_group grid = cg::this_grid();
    const int np = nb * CB;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
    // diagonal shift: every CTA reduces max_i G_ii itself (n loads, no sync)
    double shift = 0.0;
    if (shift_rel > 0.0) {
        __shared__ double s_red[kCIThreads / 32];
        double mx = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) mx = fmax(mx, G[(int64_t)i * ldg + i]);
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = mx;
        __syncthreads();
        mx = 0.0;
        for (int w = 0; w < kCIThreads / 32; ++w) mx = fmax(mx, s_red[w]);
        shift = shift_rel * mx;
    }
    // padded copy: [[G + shift I, 0], [0, I]]; X = 0
    for (int64_t t = gtid; t < (int64_t)np * np; t += gstride) {
        const int i = (int)(t / np), j = (int)(t % np);
        A[t] = (i < n && j < n) ? G[(int64_t)i * ldg + j] + (i == j ? shift : 0.0)
                                : (i == j ? 1.0 : 0.0);
        X[t] = 0.0;
        S[t] = 0.0;
    }
    grid.sync();
    auto tload = [&](double (*T)[CB + 1], const double* M, int r0, int c0) {
        for (int q = threadIdx.x; q < CB * CB; q += blockDim.x)
            T[q / CB][q % CB] = M[(int64_t)(r0 + q / CB) * np + c0 + q % CB];
    };
    auto tstore = [&](double* M, int r0, int c0, double (*T)[CB + 1]) {
        for (int q = threadIdx.x; q < CB * CB; q += blockDim.x)
            M[(int64_t)(r0 + q / CB) * np + c0 + q % CB] = T[q / CB][q % CB];
    };
    // factor tile (p, p) held in T (smem) into Lb / X, pivot statistics (CTA 0)
    auto factor = [&](int p, double (*T)[CB + 1]) {
        __syncthreads();
        {
            double mn, mx;
            for (int q = threadIdx.x; q < CB * CB; q += blockDim.x)  // factor a copy in sh.a
                sh.a[q / CB][q % CB] = T[q / CB][q % CB];
            __syncthreads();
            const int bad = tile_chol_inv(sh.a, sh.b, sh.c, sh.invd, &mn, &mx);
            if (threadIdx.x == 0) {
                // (pivot bookkeeping in shared memory: a global read here was a
                // round trip on the per-panel critical path)
                const int p0 = p * CB;
                if (bad && sh.info0 == 0) sh.info0 = p0 + bad;
                // pivots of the identity padding are 1: count only real rows
                if (p0 < n) {
                    if (p0 + CB <= n) {
                        sh.dmn = fmin(sh.dmn, mn);
                        sh.dmx = fmax(sh.dmx, mx);
                    } else {
                        for (int k = 0; p0 + k < n; ++k) {
                            sh.dmn = fmin(sh.dmn, sh.a[k][k]);
                            sh.dmx = fmax(sh.dmx, sh.a[k][k]);
                        }
                    }
                }
            }
        }
        __syncthreads();
        for (int q = threadIdx.x; q < CB * CB; q += blockDim.x)
            sh.xpp[q / CB][q % CB] = sh.b[q / CB][q % CB];
        tstore(Lb, p * CB, p * CB, sh.a);
        tstore(X, p * CB, p * CB, sh.b);
    };
    if (blockIdx.x == 0) {
        if (threadIdx.x == 0) {
            sh.dmn = INFINITY;
            sh.dmx = 0.0;
            sh.info0 = 0;
        }
        tload(sh.c, A, 0, 0);
        factor(0, sh.c);
    }
    for (int p = 0; p < nb; ++p) {
        stamp(4 * p + 0);
        grid.sync();
        stamp(4 * p + 1);
        const int p0 = p * CB;
        const int m = nb - 1 - p;
        const int ntrail = m * (m + 1) / 2;
        const int ntask = ntrail + (nb - p) * p;   // + inverse layer: rows p..nb-1 x J < p
        for (int t = blockIdx.x; t < ntask; t += gridDim.x) {
            if (t < ntrail) {
                // trailing tile: t = 0 is (p+1, p+1); then row-major over J <= I
                int I = 0, rem = t;
                while (rem > I) {
                    rem -= I + 1;
                    ++I;
                }
                int J = rem;
                // remap so task 0 is the lookahead tile (p+1, p+1): tile order
                // (0,0),(1,0),(1,1),... -> (I, J) relative to p+1
                const int I0 = (p + 1 + I) * CB, J0 = (p + 1 + J) * CB;
                // all operand tiles in flight at once (one global round trip);
                // CTA 0 factored L_pp itself and still holds its inverse (its
                // later tasks of this panel run after factor(p+1) replaced it)
                if (t == 0) {
                    for (int q = threadIdx.x; q < CB * CB; q += blockDim.x)
                        sh.b[q / CB][q % CB] = sh.xpp[q / CB][q % CB];
                } else {
                    tload(sh.b, X, p0, p0);             // L_pp^{-1}
                }
                tload(sh.a, A, I0, p0);                 // A_Ip
                if (I != J) tload(sd, A, J0, p0);       // A_Jp
                tload(sh.e, A, I0, J0);                 // A_IJ
                __syncthreads();
                tile_mm(sh.c, sh.a, sh.b, 0, 1.0, false);   // L_Ip = A_Ip L_pp^{-T}
                if (J == 0) tstore(Lb, I0, p0, sh.c);
                if (I != J) tile_mm(sh.a, sd, sh.b, 0, 1.0, false);  // L_Jp
                tile_mm(sh.e, sh.c, I != J ? sh.a : sh.c, 0, -1.0, true);  // A_IJ -= L_Ip L_Jp^T
                tstore(A, I0, J0, sh.e);
                if (t == 0 && blockIdx.x == 0) {
                    stamp(4 * p + 2);
                    factor(p + 1, sh.e);  // lookahead
                    stamp(4 * p + 3);
                }
                __syncthreads();
            } else {
                // inverse layer K = p-1 for tile (r, J), r >= p, J < p
                const int u = t - ntrail;
                const int r = p + u / p, J = u % p;
                const int R0 = r * CB, J0 = J * CB, K0 = (p - 1) * CB;
                tload(sh.a, Lb, R0, K0);                // L_{r,p-1}
                tload(sh.b, X, K0, J0);                 // X_{p-1,J}
                tload(sd, S, R0, J0);                   // S_rJ
                __syncthreads();
                tile_mm(sd, sh.a, sh.b, 1, 1.0, true);  // S_rJ += L_{r,p-1} X_{p-1,J}
                if (r > p) {
                    tstore(S, R0, J0, sd);
                } else {
                    tload(sh.a, X, p0, p0);             // L_pp^{-1}
                    __syncthreads();
                    tile_mm(sh.c, sh.a, sd, 1, -1.0, false);
                    tstore(X, p0, J0, sh.c);
                }
                __syncthreads();
            }
        }
    }
    grid.sync();
    if (gtid == 0) {
        dinfo[0] = sh.dmn;
        dinfo[1] = sh.dmx;
        if (sh.info0 != 0 && *info == 0) *info = sh.info0;
        else if (*info == 0 && sh.dmn < rel_tol * sh.dmx) *info = -1;
    }
}

__global__ void unpad_kernel(const double* __restrict__ Xp, int np, int n, double* __restrict__ X) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)n * n;
         t += (int64_t)gridDim.x * blockDim.x)
        X[t] = Xp[(t / n) * np + t % n];
}

}  // namespace
}  // namespace skp

using namespace skp;

extern "C" int64_t skp_cholinv_ws_bytes(int64_t n) {
    const int64_t np = cdiv(n, CB) * CB;
    return 4 * np * np * (int64_t)sizeof(double) + 64;
}

extern "C" int skp_cholinv_f64(const double* G, int64_t n, int64_t ld, double rel_tol,
                               double shift_rel, double* X, int32_t* info, void* ws, int64_t ws_bytes, void* stream) {
    SKP_ARG(n >= 1 && n <= 16384 && ld >= n && G && X && info && shift_rel >= 0.0,
            "cholinv: bad arguments");
    SKP_ARG(ws && ws_bytes >= skp_cholinv_ws_bytes(n), "cholinv needs %lld bytes of workspace",
            (long long)skp_cholinv_ws_bytes(n));
    cudaStream_t st = SKP_STREAM(stream);
    const int nb = (int)cdiv(n, CB);
    const int np = nb * CB;
    double* A = reinterpret_cast<double*>(ws);
    double* Lb = A + (int64_t)np * np;
    double* Xp = Lb + (int64_t)np * np;
    double* Sp = Xp + (int64_t)np * np;
    // 2 doubles of pivot statistics live in the 64-byte tail of the workspace
    double* dinfo = reinterpret_cast<double*>(
        (reinterpret_cast<uintptr_t>(Sp + (int64_t)np * np) + 15) & ~uintptr_t(15));
    int dev = 0, sms = 148, per_sm = 0;
    SKP_CUDA(cudaGetDevice(&dev));
    SKP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const size_t smem = sizeof(CIShared) + sizeof(double) * CB * (CB + 1) + 16;
    SKP_CUDA(cudaFuncSetAttribute(cholinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    SKP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cholinv_kernel, kCIThreads, smem));
    SKP_ARG(per_sm >= 1, "cholinv: cooperative kernel cannot be resident");
    int maxtask = 1;
    for (int p = 0; p < nb; ++p)
        maxtask = std::max(maxtask, (nb - 1 - p) * (nb - p) / 2 + (nb - p) * p);
    int blocks = std::min(sms, std::max(maxtask, 1));
    int nn = (int)n;
    int64_t ldg = ld;
    unsigned long long* prof_arg = nullptr;  // (per-panel timestamps: unused)
    void* args[] = {(void*)&G, &nn, &ldg, (void*)&nb, &rel_tol, &shift_rel, &A, &Lb, &Xp, &Sp, &dinfo, &info, &prof_arg};
    SKP_CUDA(cudaLaunchCooperativeKernel((void*)cholinv_kernel, dim3(blocks), dim3(kCIThreads), args,
                                         smem, st));
    count_launch();
    if (np == n) {
        SKP_CUDA(cudaMemcpyAsync(X, Xp, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st));
    } else {
        unpad_kernel<<<(unsigned)std::min<int64_t>(cdiv(n * n, 256), 4096), 256, 0, st>>>(Xp, np,
                                                                                        nn, X);
        SKP_LAUNCHED(unpad_kernel);
    }
    return SKP_OK;
}
