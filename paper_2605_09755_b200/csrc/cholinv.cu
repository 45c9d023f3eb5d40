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
// info: left untouched on success; set to k+1 if pivot k is not
// positive/finite, -1 if min L_ii < rel_tol * max L_ii (numerically rank
// deficient -> eigen-based path).  Callers zero it; failures accumulate, so one
// flag can cover a whole sync-free sequence of factorisations.
#include <cooperative_groups.h>
#include <math.h>

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

__global__ void __launch_bounds__(kCIThreads)
cholinv_kernel(const double* __restrict__ G, int n, int64_t ldg, int nb, double rel_tol,
               double* A, double* X, double* dinfo, int32_t* info, int col_in_smem) {
    extern __shared__ __align__(16) unsigned char smraw[];
    CIShared& sh = *reinterpret_cast<CIShared*>(smraw);
    cg::grid_group grid = cg::this_grid();
    const int np = nb * CB;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
    // padded copy: [[G, 0], [0, I]]
    for (int64_t t = gtid; t < (int64_t)np * np; t += gstride) {
        const int i = (int)(t / np), j = (int)(t % np);
        A[t] = (i < n && j < n) ? G[(int64_t)i * ldg + j] : (i == j ? 1.0 : 0.0);
        X[t] = 0.0;
    }
    if (gtid == 0) {                 // *info is only ever SET (failures accumulate)
        dinfo[0] = INFINITY;   // min pivot of L
        dinfo[1] = 0.0;        // max pivot of L
    }
    grid.sync();
    for (int p = 0; p < nb; ++p) {
        const int p0 = p * CB;
        // (1) diagonal block: factor + invert (CTA 0)
        if (blockIdx.x == 0) {
            for (int t = threadIdx.x; t < CB * CB; t += blockDim.x)
                sh.a[t / CB][t % CB] = A[(int64_t)(p0 + t / CB) * np + p0 + t % CB];
            if (threadIdx.x == 0) sh.bad = 0;
            __syncthreads();
            for (int k = 0; k < CB; ++k) {
                if (threadIdx.x == 0) {
                    const double dkk = sh.a[k][k];
                    if (!(dkk > 0.0) || !isfinite(dkk)) {
                        if (!sh.bad) sh.bad = p0 + k + 1;
                        sh.a[k][k] = 1.0;  // keep going; result is discarded
                    } else {
                        sh.a[k][k] = sqrt(dkk);
                    }
                }
                __syncthreads();
                const double dk = sh.a[k][k];
                for (int i = k + 1 + threadIdx.x; i < CB; i += blockDim.x) sh.a[i][k] /= dk;
                __syncthreads();
                for (int t = threadIdx.x; t < (CB - k - 1) * (CB - k - 1); t += blockDim.x) {
                    const int i = k + 1 + t / (CB - k - 1), j = k + 1 + t % (CB - k - 1);
                    if (j <= i) sh.a[i][j] -= sh.a[i][k] * sh.a[j][k];
                }
                __syncthreads();
            }
            // zero the strict upper part, invert (column-parallel forward substitution)
            for (int t = threadIdx.x; t < CB * CB; t += blockDim.x)
                if (t % CB > t / CB) sh.a[t / CB][t % CB] = 0.0;
            __syncthreads();
            if (threadIdx.x < CB) {
                const int j = threadIdx.x;
                for (int i = 0; i < CB; ++i) {
                    double s = (i == j) ? 1.0 : 0.0;
                    for (int k = j; k < i; ++k) s -= sh.a[i][k] * sh.b[k][j];
                    sh.b[i][j] = i >= j ? s / sh.a[i][i] : 0.0;
                }
            }
            __syncthreads();
            for (int t = threadIdx.x; t < CB * CB; t += blockDim.x) {
                const int i = t / CB, j = t % CB;
                A[(int64_t)(p0 + i) * np + p0 + j] = sh.a[i][j];
                X[(int64_t)(p0 + i) * np + p0 + j] = sh.b[i][j];
            }
            if (threadIdx.x == 0) {
                if (sh.bad && *info == 0) *info = sh.bad;
                double mn = dinfo[0], mx = dinfo[1];
                for (int k = 0; k < CB; ++k)
                    if (p0 + k < n) { mn = fmin(mn, sh.a[k][k]); mx = fmax(mx, sh.a[k][k]); }
                dinfo[0] = mn;
                dinfo[1] = mx;
            }
        }
        grid.sync();
        if (p + 1 < nb) {
            // (2) L_ip = A_ip L_pp^{-T}: one warp per row below the panel
            const int warp_g = (int)(gtid >> 5), nw = (int)(gstride >> 5), lane = threadIdx.x & 31;
            for (int i = p0 + CB + warp_g; i < np; i += nw) {
                double* row = A + (int64_t)i * np + p0;
                const double* Li = X + (int64_t)p0 * np + p0;  // L_pp^{-1}, row-major
                const double a_l = row[lane];
                double acc = 0.0;
                // L_ip[c] = sum_k A_ip[k] * Linv[c][k]
                for (int k = 0; k < CB; ++k) acc += __shfl_sync(0xffffffffu, a_l, k) * Li[(int64_t)lane * np + k];
                __syncwarp();
                row[lane] = acc;
            }
            grid.sync();
            // (3) trailing update of tiles (I, J), p < J <= I
            const int m = nb - p - 1;
            const int ntile = m * (m + 1) / 2;
            for (int t = blockIdx.x; t < ntile; t += gridDim.x) {
                int I = 0, rem = t;
                while (rem > I) { rem -= I + 1; ++I; }
                const int J = rem;
                const int I0 = (p + 1 + I) * CB, J0 = (p + 1 + J) * CB;
                for (int q = threadIdx.x; q < CB * CB; q += blockDim.x) {
                    const int r = q / CB, c = q % CB;
                    sh.a[r][c] = A[(int64_t)(I0 + r) * np + p0 + c];   // L_Ip
                    sh.b[r][c] = A[(int64_t)(J0 + r) * np + p0 + c];   // L_Jp
                    sh.c[r][c] = A[(int64_t)(I0 + r) * np + J0 + c];
                }
                __syncthreads();
                tile_mm(sh.c, sh.a, sh.b, 0, -1.0, true);
                for (int q = threadIdx.x; q < CB * CB; q += blockDim.x)
                    A[(int64_t)(I0 + q / CB) * np + J0 + q % CB] = sh.c[q / CB][q % CB];
                __syncthreads();
            }
            grid.sync();
        }
    }
    // X = L^{-1} by block columns: block column J depends only on itself
    // (X_IJ = -L_II^{-1} sum_{K=J}^{I-1} L_IK X_KJ), so one CTA sweeps down one
    // column with it resident in shared memory -- no grid syncs.
    // resident copy in smem when np x 32 doubles fit, else read X (L1/L2)
    double* colS = reinterpret_cast<double*>(smraw + sizeof(CIShared));  // np x CB
    for (int J = blockIdx.x; J < nb; J += gridDim.x) {
        const int J0 = J * CB;
        double* colX = col_in_smem ? colS : X + J0;
        const int64_t cld = col_in_smem ? CB : np;   // leading dim of the column view
        if (col_in_smem) {
            for (int q = threadIdx.x; q < CB * CB; q += blockDim.x)
                colS[(q / CB) * CB + q % CB] = X[(int64_t)(J0 + q / CB) * np + J0 + q % CB];
        }
        __syncthreads();
        for (int I = J + 1; I < nb; ++I) {
            const int I0 = I * CB;
            // T = sum_K L_IK X_KJ : thread (r, c4) accumulates 4 outputs
            const int tr = threadIdx.x / 8, tc = (threadIdx.x % 8) * 4;
            double acc[4] = {0, 0, 0, 0};
            const double* Lrow = A + (int64_t)(I0 + tr) * np;
            for (int k = J0; k < I0; ++k) {
                const double l = Lrow[k];
                const double* xr = colX + (int64_t)(col_in_smem ? k - J0 : k) * cld + tc;
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[j] += l * xr[j];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) sh.c[tr][tc + j] = acc[j];
            for (int q = threadIdx.x; q < CB * CB; q += blockDim.x)
                sh.a[q / CB][q % CB] = X[(int64_t)(I0 + q / CB) * np + I0 + q % CB];  // L_II^{-1}
            __syncthreads();
            tile_mm(sh.b, sh.a, sh.c, 1, -1.0, false);
            for (int q = threadIdx.x; q < CB * CB; q += blockDim.x) {
                const double v = sh.b[q / CB][q % CB];
                if (col_in_smem) colS[(int64_t)(I0 - J0 + q / CB) * CB + q % CB] = v;
                X[(int64_t)(I0 + q / CB) * np + J0 + q % CB] = v;
            }
            __syncthreads();
        }
    }
    grid.sync();
    if (gtid == 0 && *info == 0 && dinfo[0] < rel_tol * dinfo[1]) *info = -1;
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
    return 2 * np * np * (int64_t)sizeof(double) + 64;
}

extern "C" int skp_cholinv_f64(const double* G, int64_t n, int64_t ld, double rel_tol, double* X,
                               int32_t* info, void* ws, int64_t ws_bytes, void* stream) {
    SKP_ARG(n >= 1 && n <= 16384 && ld >= n && G && X && info, "cholinv: bad arguments");
    SKP_ARG(ws && ws_bytes >= skp_cholinv_ws_bytes(n), "cholinv needs %lld bytes of workspace",
            (long long)skp_cholinv_ws_bytes(n));
    cudaStream_t st = SKP_STREAM(stream);
    const int nb = (int)cdiv(n, CB);
    const int np = nb * CB;
    double* A = reinterpret_cast<double*>(ws);
    double* Xp = A + (int64_t)np * np;
    // 2 doubles of pivot statistics live in the 64-byte tail of the workspace
    double* dinfo = reinterpret_cast<double*>(
        (reinterpret_cast<uintptr_t>(Xp + (int64_t)np * np) + 15) & ~uintptr_t(15));
    int dev = 0, sms = 148, per_sm = 0;
    SKP_CUDA(cudaGetDevice(&dev));
    SKP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // CIShared + one resident block column of L^{-1} (np x 32 doubles) if it fits
    const size_t col_bytes = (size_t)np * CB * sizeof(double);
    int col_in_smem = sizeof(CIShared) + col_bytes + 16 <= 200 * 1024 ? 1 : 0;
    const size_t smem = sizeof(CIShared) + (col_in_smem ? col_bytes : 0) + 16;
    SKP_CUDA(cudaFuncSetAttribute(cholinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    SKP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cholinv_kernel, kCIThreads, smem));
    SKP_ARG(per_sm >= 1, "cholinv: cooperative kernel cannot be resident");
    int blocks = std::min(sms, std::max(nb * (nb + 1) / 2, 1));
    int nn = (int)n;
    int64_t ldg = ld;
    void* args[] = {(void*)&G, &nn, &ldg, (void*)&nb, &rel_tol, &A, &Xp, &dinfo, &info, &col_in_smem};
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
