// K5 / K6: small dense FP64 kernels for the r2 x r2 cores, plus utilities and
// the C-ABI error plumbing.
//   * blocked right-looking Cholesky (diag factor in smem -> panel TRSM ->
//     trailing SYRK through the SIMT DGEMM), status in a device int;
//   * lower-triangular inverse (column-parallel forward substitution);
//   * parallel cyclic Jacobi eigensolver (round-robin pairing, in-place 2x2
//     block updates), single-CTA shared-memory variant for n <= 112 and a
//     cooperative grid-synchronised variant above.
#include <algorithm>
#include <atomic>
#include <cooperative_groups.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "gemm.h"

namespace cg = cooperative_groups;

// ----------------------------------------------------------- errors ------
namespace skp {
int64_t syev_tri_ws_bytes(int64_t n);
int syev_tri(const double* A, int64_t n, double* W, double* V, void* ws, int64_t ws_bytes,
             int32_t* sweeps, cudaStream_t st);
static thread_local char g_err[512] = "";
void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
int cuda_fail(cudaError_t e, const char* what) {
    set_error("CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e), what);
    return SKP_ERR_CUDA;
}
}  // namespace skp

namespace skp {
static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace skp

extern "C" const char* skp_last_error(void) { return skp::g_err; }
extern "C" int64_t skp_launch_count(void) { return skp::g_launches.load(); }
extern "C" int skp_abi_version(void) { return 1; }

namespace skp {
namespace {

// ------------------------------------------------------------ Cholesky ---
constexpr int NB = 64;

__global__ void chol_diag_kernel(double* G, int64_t ld, int64_t k0, int b, int32_t* info) {
    __shared__ double L[NB][NB + 1];
    __shared__ int bad;
    if (*info != 0) return;
    for (int t = threadIdx.x; t < b * b; t += blockDim.x) {
        int i = t / b, j = t % b;
        L[i][j] = G[(k0 + i) * ld + k0 + j];
    }
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    for (int k = 0; k < b; ++k) {
        if (threadIdx.x == 0) {
            double d = L[k][k];
            if (!(d > 0.0) || !isfinite(d)) bad = k + 1;
            else L[k][k] = sqrt(d);
        }
        __syncthreads();
        if (bad) break;
        double dk = L[k][k];
        for (int i = k + 1 + threadIdx.x; i < b; i += blockDim.x) L[i][k] /= dk;
        __syncthreads();
        for (int t = threadIdx.x; t < (b - k - 1) * (b - k - 1); t += blockDim.x) {
            int i = k + 1 + t / (b - k - 1), j = k + 1 + t % (b - k - 1);
            if (j <= i) L[i][j] -= L[i][k] * L[j][k];
        }
        __syncthreads();
    }
    if (bad) {
        if (threadIdx.x == 0) *info = (int32_t)(k0 + bad);
        return;
    }
    for (int t = threadIdx.x; t < b * b; t += blockDim.x) {
        int i = t / b, j = t % b;
        if (j <= i) G[(k0 + i) * ld + k0 + j] = L[i][j];
    }
}

// rows i >= k0 + b: G[i][k0:k0+b] <- G[i][k0:k0+b] . L_kk^{-T}
__global__ void chol_trsm_kernel(double* G, int64_t ld, int64_t n, int64_t k0, int b,
                                 const int32_t* info) {
    __shared__ double L[NB][NB + 1];
    if (*info != 0) return;
    for (int t = threadIdx.x; t < b * b; t += blockDim.x) {
        int i = t / b, j = t % b;
        L[i][j] = G[(k0 + i) * ld + k0 + j];
    }
    __syncthreads();
    int64_t i = k0 + b + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double x[NB];
    double* row = G + i * ld + k0;
#pragma unroll
    for (int j = 0; j < NB; ++j)
        if (j < b) x[j] = row[j];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
        if (j < b) {
            double s = x[j];
#pragma unroll
            for (int t = 0; t < j; ++t) s -= x[t] * L[j][t];
            x[j] = s / L[j][j];
        }
    }
#pragma unroll
    for (int j = 0; j < NB; ++j)
        if (j < b) row[j] = x[j];
}

// X = L^{-1}: one warp per column j, forward substitution down the column.
// x_i = (delta_ij - sum_{k=j}^{i-1} L_ik x_k) / L_ii; the dot product is split
// across the 32 lanes (warp shuffle reduction), x lives in shared memory.
constexpr int kTrinvWarps = 8;
__global__ void __launch_bounds__(kTrinvWarps * 32)
trinv_kernel(const double* __restrict__ L, int64_t ldl, int64_t n, double* __restrict__ X) {
    extern __shared__ double xs_all[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t j = (int64_t)blockIdx.x * kTrinvWarps + warp;
    if (j >= n) return;
    double* xs = xs_all + (int64_t)warp * n;
    for (int64_t i = lane; i < j; i += 32) X[i * n + j] = 0.0;
    for (int64_t i = j; i < n; ++i) {
        const double* li = L + i * ldl;
        double acc = 0.0;
        for (int64_t k = j + lane; k < i; k += 32) acc += li[k] * xs[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        const double xi = ((i == j ? 1.0 : 0.0) - acc) / li[i];
        if (lane == 0) xs[i] = xi;
        __syncwarp();
        if (lane == (int)(i & 31)) X[i * n + j] = xi;
    }
}

// ------------------------------------------------------------- Jacobi ----
// Round-robin schedule over np (= n rounded up to even) slots: slot 0 fixed,
// slots 1..np-1 rotate.  Round k pairs slot i with slot np-1-i.
__device__ __forceinline__ int rr_slot(int t, int k, int np) {
    return t == 0 ? 0 : ((t - 1 + k) % (np - 1)) + 1;
}

struct JacobiShared {
    double* c;   // [np/2]
    double* s;   // [np/2]
    int* p;      // [np/2]
    int* q;      // [np/2]
};

// Rotation threshold: skip when |a_pq| <= max(eps * sqrt(|a_pp a_qq|), tol_abs)
// with tol_abs = 2^-47 * max_i |a_ii| of the input.  The absolute floor stops
// the sweeps once every eigenvalue is accurate relative to lambda_max (what
// sigma parity needs) instead of chasing noise-floor eigenvalues to full
// relative accuracy (13-14 sweeps -> ~7 at n = 520).
__device__ __forceinline__ bool jacobi_rotate(double apq, double app, double aqq, double tol_abs) {
    return apq != 0.0 && fabs(apq) > 0x1p-52 * sqrt(fabs(app * aqq)) && fabs(apq) > tol_abs &&
           fabs(apq) > 1e-300;
}
// block-wide max |A_ii| (all threads get the value)
__device__ double diag_absmax(const double* A, int64_t n, int64_t ld) {
    __shared__ double red[32];
    double m = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, fabs(A[i * ld + i]));
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    double r = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, red[w]);
    __syncthreads();
    return r;
}

// Every CTA computes all rotations of round k (redundantly) into smem.
// Returns the number of non-trivial rotations (valid in thread 0 only).
__device__ int jacobi_rotations(const double* A, int64_t ld, int n, int np, int k,
                                JacobiShared sh, int* cnt_smem, double tol_abs) {
    if (threadIdx.x == 0) *cnt_smem = 0;
    __syncthreads();
    int local = 0;
    for (int i = threadIdx.x; i < np / 2; i += blockDim.x) {
        int a = rr_slot(i, k, np), b = rr_slot(np - 1 - i, k, np);
        int p = a < b ? a : b, q = a < b ? b : a;
        double c = 1.0, s = 0.0;
        if (q < n) {
            double apq = A[(int64_t)p * ld + q];
            double app = A[(int64_t)p * ld + p], aqq = A[(int64_t)q * ld + q];
            if (jacobi_rotate(apq, app, aqq, tol_abs)) {
                double theta = (aqq - app) / (2.0 * apq);
                double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
                if (!isfinite(theta)) t = 0.5 / theta;  // huge theta
                c = 1.0 / sqrt(1.0 + t * t);
                s = t * c;
                ++local;
            }
        }
        sh.c[i] = c;
        sh.s[i] = s;
        sh.p[i] = p;
        sh.q[i] = q;
    }
    if (local) atomicAdd(cnt_smem, local);
    __syncthreads();
    return *cnt_smem;
}

// In-place 2x2 block update A' = J^T A J for blocks [tid0, total) stride, and V' = V J.
__device__ void jacobi_apply(double* A, int64_t ld, double* V, int64_t ldv, int n, int np,
                             JacobiShared sh, int64_t tid0, int64_t stride) {
    const int64_t P = np / 2;
    for (int64_t t = tid0; t < P * P; t += stride) {
        int u = (int)(t / P), v = (int)(t % P);
        int pu = sh.p[u], qu = sh.q[u], pv = sh.p[v], qv = sh.q[v];
        double cu = sh.c[u], su = sh.s[u], cv = sh.c[v], sv = sh.s[v];
        if (su == 0.0 && sv == 0.0) continue;
        bool qu_ok = qu < n, qv_ok = qv < n;
        double a00 = A[(int64_t)pu * ld + pv];
        double a01 = qv_ok ? A[(int64_t)pu * ld + qv] : 0.0;
        double a10 = qu_ok ? A[(int64_t)qu * ld + pv] : 0.0;
        double a11 = (qu_ok && qv_ok) ? A[(int64_t)qu * ld + qv] : 0.0;
        // rows: R = J_u^T [a]: J_u = [[c, s], [-s, c]] on (p, q)
        double r00 = cu * a00 - su * a10, r01 = cu * a01 - su * a11;
        double r10 = su * a00 + cu * a10, r11 = su * a01 + cu * a11;
        // cols: R J_v
        double b00 = r00 * cv - r01 * sv, b01 = r00 * sv + r01 * cv;
        double b10 = r10 * cv - r11 * sv, b11 = r10 * sv + r11 * cv;
        if (u == v) { b01 = 0.0; b10 = 0.0; }
        A[(int64_t)pu * ld + pv] = b00;
        if (qv_ok) A[(int64_t)pu * ld + qv] = b01;
        if (qu_ok) A[(int64_t)qu * ld + pv] = b10;
        if (qu_ok && qv_ok) A[(int64_t)qu * ld + qv] = b11;
    }
    for (int64_t t = tid0; t < (int64_t)n * P; t += stride) {
        int row = (int)(t / P), u = (int)(t % P);
        double su = sh.s[u];
        if (su == 0.0 || sh.q[u] >= n) continue;
        double cu = sh.c[u];
        double* vr = V + (int64_t)row * ldv;
        double vp = vr[sh.p[u]], vq = vr[sh.q[u]];
        vr[sh.p[u]] = cu * vp - su * vq;
        vr[sh.q[u]] = su * vp + cu * vq;
    }
}

__device__ void jacobi_shared_carve(JacobiShared& sh, unsigned char* base, int np) {
    int P = np / 2;
    sh.c = reinterpret_cast<double*>(base);
    sh.s = sh.c + P;
    sh.p = reinterpret_cast<int*>(sh.s + P);
    sh.q = sh.p + P;
}

// Single CTA, A and V resident in shared memory (n <= 112).
__global__ void syevj_smem_kernel(const double* __restrict__ Ain, int64_t n, double* Vout_ws,
                                  double* Aout_ws, int max_sweeps, int32_t* sweeps) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int nn = (int)n, np = nn + (nn & 1);
    double* A = reinterpret_cast<double*>(sm);
    double* V = A + nn * nn;
    JacobiShared sh;
    jacobi_shared_carve(sh, reinterpret_cast<unsigned char*>(V + nn * nn), np);
    __shared__ int cnt;
    for (int t = threadIdx.x; t < nn * nn; t += blockDim.x) {
        A[t] = Ain[t];
        V[t] = (t / nn == t % nn) ? 1.0 : 0.0;
    }
    __syncthreads();
    const double tol_abs = 0x1p-47 * diag_absmax(A, nn, nn);
    int sw = 0;
    for (; sw < max_sweeps; ++sw) {
        int total = 0;
        for (int k = 0; k < np - 1; ++k) {
            total += jacobi_rotations(A, nn, nn, np, k, sh, &cnt, tol_abs);
            jacobi_apply(A, nn, V, nn, nn, np, sh, threadIdx.x, blockDim.x);
            __syncthreads();
        }
        if (total == 0) break;
    }
    for (int t = threadIdx.x; t < nn * nn; t += blockDim.x) {
        Aout_ws[t] = A[t];
        Vout_ws[t] = V[t];
    }
    if (threadIdx.x == 0) *sweeps = sw + 1;
}

// Double-buffered variant for the cooperative kernel: reads Ain (stable for
// the whole round), writes every 2x2 block of Aout.
__device__ void jacobi_apply_db(const double* Ain, double* Aout, int n, int np, JacobiShared sh,
                                double* V, int64_t tid0, int64_t stride) {
    const int64_t P = np / 2;
    for (int64_t t = tid0; t < P * P; t += stride) {
        int u = (int)(t / P), v = (int)(t % P);
        int pu = sh.p[u], qu = sh.q[u], pv = sh.p[v], qv = sh.q[v];
        double cu = sh.c[u], su = sh.s[u], cv = sh.c[v], sv = sh.s[v];
        bool qu_ok = qu < n, qv_ok = qv < n;
        double a00 = Ain[(int64_t)pu * n + pv];
        double a01 = qv_ok ? Ain[(int64_t)pu * n + qv] : 0.0;
        double a10 = qu_ok ? Ain[(int64_t)qu * n + pv] : 0.0;
        double a11 = (qu_ok && qv_ok) ? Ain[(int64_t)qu * n + qv] : 0.0;
        double r00 = cu * a00 - su * a10, r01 = cu * a01 - su * a11;
        double r10 = su * a00 + cu * a10, r11 = su * a01 + cu * a11;
        double b00 = r00 * cv - r01 * sv, b01 = r00 * sv + r01 * cv;
        double b10 = r10 * cv - r11 * sv, b11 = r10 * sv + r11 * cv;
        if (u == v && su != 0.0) { b01 = 0.0; b10 = 0.0; }
        Aout[(int64_t)pu * n + pv] = b00;
        if (qv_ok) Aout[(int64_t)pu * n + qv] = b01;
        if (qu_ok) Aout[(int64_t)qu * n + pv] = b10;
        if (qu_ok && qv_ok) Aout[(int64_t)qu * n + qv] = b11;
    }
    for (int64_t t = tid0; t < (int64_t)n * P; t += stride) {
        int row = (int)(t / P), u = (int)(t % P);
        double su = sh.s[u];
        if (su == 0.0 || sh.q[u] >= n) continue;
        double cu = sh.c[u];
        double* vr = V + (int64_t)row * n;
        double vp = vr[sh.p[u]], vq = vr[sh.q[u]];
        vr[sh.p[u]] = cu * vp - su * vq;
        vr[sh.q[u]] = su * vp + cu * vq;
    }
}

// eigenvalues = diag(A) sorted descending (ties by index); permute V columns.
__global__ void eig_sort_kernel(const double* __restrict__ A, int64_t n,
                                const double* __restrict__ V, double* __restrict__ W,
                                double* __restrict__ Vout) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double li = A[i * n + i];
        int64_t rank = 0;
        for (int64_t j = 0; j < n; ++j) {
            double lj = A[j * n + j];
            rank += (lj > li) || (lj == li && j < i);
        }
        W[rank] = li;
        for (int64_t r = 0; r < n; ++r) Vout[r * n + rank] = V[r * n + i];
    }
}

// -------------------------------------------------------------- misc -----
__global__ void cast_f32_f64_kernel(const float* x, double* y, int64_t cnt) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x)
        y[t] = (double)x[t];
}
__global__ void cast_f64_f32_kernel(const double* x, float* y, int64_t cnt) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x)
        y[t] = (float)x[t];
}

template <typename S, typename D>
__global__ void cast2d_kernel(const S* __restrict__ x, int64_t ldx, D* __restrict__ y, int64_t ldy,
                              int64_t rows, int64_t cols) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < rows * cols;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = t / cols, j = t - i * cols;
        y[i * ldy + j] = (D)x[i * ldx + j];
    }
}

// y[v, :] = x[perm[v], :] (row gather; one block-row per output row)
template <typename T>
__global__ void permute_rows_kernel(const T* __restrict__ x, int64_t ldx, const int32_t* __restrict__ perm,
                                    T* __restrict__ y, int64_t ldy, int64_t rows, int64_t cols) {
    for (int64_t v = blockIdx.x; v < rows; v += gridDim.x) {
        const T* src = x + (int64_t)perm[v] * ldx;
        T* dst = y + v * ldy;
        for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) dst[j] = src[j];
    }
}

template <typename T>
__global__ void symmetrize_kernel(T* W, int64_t n, int64_t ld) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * n;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = t / n, j = t % n;
        if (j <= i) continue;
        T a = W[i * ld + j], b = W[j * ld + i];
        T m = (a + b) / T(2);
        W[i * ld + j] = m;
        W[j * ld + i] = m;
    }
}

template <typename T>
__global__ void scale_cols_kernel(T* X, int64_t rows, int64_t cols, int64_t ld,
                                  const double* __restrict__ sc) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < rows * cols;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = t / cols, j = t % cols;
        X[i * ld + j] = (T)((double)X[i * ld + j] * sc[j]);
    }
}

__global__ void orth_dev_kernel(const double* G, int64_t n, int64_t ld, double* out) {
    __shared__ double red[32];
    double mx = 0.0;
    for (int64_t t = threadIdx.x; t < n * n; t += blockDim.x) {
        int64_t i = t / n, j = t % n;
        double d = fabs(G[i * ld + j] - (i == j ? 1.0 : 0.0));
        if (!(d <= mx)) mx = d;  // propagates NaN
    }
    for (int o = 16; o > 0; o >>= 1) {
        double x = __shfl_xor_sync(0xffffffffu, mx, o);
        if (!(x <= mx)) mx = x;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
            if (!(red[w] <= m)) m = red[w];
        *out = m;
    }
}

__global__ void eig_orth_kernel(const double* W, const double* V, int64_t n, double rel_tol,
                                double* T, int32_t* k_out) {
    double w0 = W[0];
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * n;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = t / n, j = t % n;
        double wj = W[j];
        bool keep = wj > 0.0 && w0 > 0.0 && wj > rel_tol * w0;
        T[t] = keep ? V[t] / sqrt(wj) : 0.0;
        if (t == 0) {
            int k = 0;
            for (int64_t q = 0; q < n; ++q)
                k += (W[q] > 0.0 && w0 > 0.0 && W[q] > rel_tol * w0);
            *k_out = k;
        }
        (void)i;
    }
}

__global__ void sqrt_eigs_kernel(const double* W, int64_t n, double* sigma, double* inv) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double s = W[i] > 0.0 ? sqrt(W[i]) : 0.0;
        if (sigma) sigma[i] = s;
        if (inv) inv[i] = s > 0.0 ? 1.0 / s : 0.0;
    }
}

__global__ void chol_pivot_check_kernel(const double* L, int64_t n, int64_t ld, double rel_tol,
                                        int32_t* info) {
    __shared__ double smin[32], smax[32];
    if (*info != 0) return;
    double mn = INFINITY, mx = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        double d = fabs(L[i * ld + i]);
        mn = fmin(mn, d);
        mx = fmax(mx, d);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) { smin[threadIdx.x >> 5] = mn; smax[threadIdx.x >> 5] = mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { mn = fmin(mn, smin[w]); mx = fmax(mx, smax[w]); }
        mn = fmin(mn, smin[0]);
        mx = fmax(mx, smax[0]);
        if (mn < rel_tol * mx) *info = -1;
    }
}

inline unsigned grid_for(int64_t cnt, int threads = 256) {
    int64_t b = cdiv(cnt, threads);
    if (b > 148 * 32) b = 148 * 32;
    return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace
}  // namespace skp

using namespace skp;

extern "C" int skp_cholesky_f64(double* G, int64_t n, int64_t ld, int32_t* info, void* stream) {
    SKP_ARG(n >= 1 && n <= 16384 && ld >= n, "cholesky: bad sizes n=%lld ld=%lld", (long long)n,
            (long long)ld);
    SKP_ARG(G && info, "cholesky: null pointer");
    cudaStream_t st = SKP_STREAM(stream);
    SKP_CUDA(cudaMemsetAsync(info, 0, sizeof(int32_t), st));
    for (int64_t k0 = 0; k0 < n; k0 += NB) {
        int b = (int)(n - k0 < NB ? n - k0 : NB);
        chol_diag_kernel<<<1, 256, 0, st>>>(G, ld, k0, b, info);
        SKP_LAUNCHED(chol_diag_kernel);
        int64_t rest = n - k0 - b;
        if (rest <= 0) break;
        chol_trsm_kernel<<<(unsigned)cdiv(rest, 128), 128, 0, st>>>(G, ld, n, k0, b, info);
        SKP_LAUNCHED(chol_trsm_kernel);
        double* P = G + (k0 + b) * ld + k0;
        double* T = G + (k0 + b) * ld + k0 + b;
        int rc = gemm_simt<double>(0, 1, rest, rest, b, -1.0, P, ld, P, ld, 1.0, T, ld, nullptr,
                                   0, st);
        if (rc) return rc;
    }
    return SKP_OK;
}

extern "C" int skp_chol_pivot_check_f64(const double* L, int64_t n, int64_t ld, double rel_tol,
                                        int32_t* info, void* stream) {
    SKP_ARG(n >= 1 && ld >= n && L && info, "chol_pivot_check: bad arguments");
    chol_pivot_check_kernel<<<1, 256, 0, SKP_STREAM(stream)>>>(L, n, ld, rel_tol, info);
    SKP_LAUNCHED(chol_pivot_check);
    return SKP_OK;
}

extern "C" int skp_trinv_lower_f64(const double* L, int64_t ldl, int64_t n, double* X,
                                   void* stream) {
    SKP_ARG(n >= 1 && n <= 3000 && ldl >= n && L && X, "trinv: bad arguments (n <= 3000)");
    const size_t smem = (size_t)kTrinvWarps * n * sizeof(double);
    SKP_CUDA(cudaFuncSetAttribute(trinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    trinv_kernel<<<(unsigned)cdiv(n, kTrinvWarps), kTrinvWarps * 32, smem, SKP_STREAM(stream)>>>(
        L, ldl, n, X);
    SKP_LAUNCHED(trinv_kernel);
    return SKP_OK;
}

extern "C" int64_t skp_syevj_ws_bytes(int64_t n) {
    const int64_t small = 2 * n * n * (int64_t)sizeof(double);
    int64_t b = small;
    const int64_t tri = syev_tri_ws_bytes(n);
    b = b > tri ? b : tri;
    return b + 64 * sizeof(int32_t) + 256;
}

extern "C" int skp_syevj_f64(double* A, int64_t n, double* W, double* V, int32_t max_sweeps,
                             void* ws, int64_t ws_bytes, int32_t* sweeps, void* stream) {
    SKP_ARG(n >= 1 && n <= 8192 && A && W && V && sweeps, "syevj: bad arguments");
    SKP_ARG(ws && ws_bytes >= skp_syevj_ws_bytes(n), "syevj needs %lld bytes of workspace",
            (long long)skp_syevj_ws_bytes(n));
    SKP_ARG(max_sweeps >= 1 && max_sweeps <= 60, "syevj: max_sweeps in [1, 60]");
    cudaStream_t st = SKP_STREAM(stream);
    double* Vws = reinterpret_cast<double*>(ws);
    double* Aws = Vws + n * n;
    const int np = (int)(n + (n & 1));
    const size_t rot_bytes = (size_t)(np / 2) * (2 * sizeof(double) + 2 * sizeof(int));
    if (n <= 112) {
        size_t smem = 2 * (size_t)n * n * sizeof(double) + rot_bytes;
        SKP_CUDA(cudaFuncSetAttribute(syevj_smem_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        syevj_smem_kernel<<<1, 512, smem, st>>>(A, n, Vws, Aws, max_sweeps, sweeps);
        SKP_LAUNCHED(syevj_smem_kernel);
        eig_sort_kernel<<<grid_for(n), 256, 0, st>>>(Aws, n, Vws, W, V);
        SKP_LAUNCHED(eig_sort_kernel);
        return SKP_OK;
    }
    // n > 112: tridiagonal reduction + bisection + inverse iteration (eig_tri.cu)
    return syev_tri(A, n, W, V, ws, ws_bytes, sweeps, st);
}

// _check_psd's symmetry test (power.py:242-255) at any n: out[0] = max
// |a_ij - a_ji|, out[1] = max |a_ij| (fp64 bit patterns of non-negative
// values, so an integer atomicMax orders them; the caller zeroes out).  One
// CTA per 64 x 64 tile pair (bi >= bj) at a time: tile (bi, bj) is read into
// registers and tile (bj, bi) into shared memory with 16-byte loads (16
// elements in flight per thread and tile), so the matrix is read exactly once
// (C4: 17.2 GB, HBM-bound) with no n x n temporaries.
constexpr int kSymT = 64;
template <typename T>
__global__ void __launch_bounds__(256)
sym_check_kernel(const T* __restrict__ A, int64_t n, int64_t ld, int64_t tiles, int vec_ok,
                 unsigned long long* __restrict__ out) {
    constexpr int V = 16 / sizeof(T);        // elements per 16-byte load
    constexpr int RV = kSymT / V;            // vectors per tile row
    constexpr int NV = kSymT * kSymT / V / 256;  // vectors per thread per tile
    __shared__ T t1[kSymT][kSymT + 1];
    double dmax = 0.0, amax = 0.0;
    for (int64_t p = blockIdx.x; p < tiles * (tiles + 1) / 2; p += gridDim.x) {
        // p -> (bi, bj), bi >= bj: p = bi (bi + 1) / 2 + bj
        int64_t bi = (int64_t)((sqrt(8.0 * (double)p + 1.0) - 1.0) * 0.5);
        while (bi * (bi + 1) / 2 > p) --bi;
        while ((bi + 1) * (bi + 2) / 2 <= p) ++bi;
        const int64_t bj = p - bi * (bi + 1) / 2;
        const bool full = vec_ok && (bi + 1) * kSymT <= n;
        T a[NV][V];
        __syncthreads();
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const int u = threadIdx.x + 256 * q, r = u / RV, c = (u % RV) * V;
            const int64_t i = bi * kSymT + r, j = bj * kSymT + c;   // tile (bi, bj)
            const int64_t i2 = bj * kSymT + r, j2 = bi * kSymT + c; // tile (bj, bi)
            if (full) {
                const uint4 x = *reinterpret_cast<const uint4*>(A + i * ld + j);
                const uint4 y = *reinterpret_cast<const uint4*>(A + i2 * ld + j2);
                const T* xs = reinterpret_cast<const T*>(&x);
                const T* ys = reinterpret_cast<const T*>(&y);
#pragma unroll
                for (int e = 0; e < V; ++e) {
                    a[q][e] = xs[e];
                    t1[r][c + e] = ys[e];
                }
            } else {
#pragma unroll
                for (int e = 0; e < V; ++e) {
                    a[q][e] = (i < n && j + e < n) ? A[i * ld + j + e] : T(0);
                    t1[r][c + e] = (i2 < n && j2 + e < n) ? A[i2 * ld + j2 + e] : T(0);
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const int u = threadIdx.x + 256 * q, r = u / RV, c = (u % RV) * V;
#pragma unroll
            for (int e = 0; e < V; ++e) {
                const double x = (double)a[q][e], y = (double)t1[c + e][r];  // a_ij, a_ji
                dmax = fmax(dmax, fabs(x - y));
                amax = fmax(amax, fmax(fabs(x), fabs(y)));
            }
        }
    }
    for (int o = 16; o; o >>= 1) {
        dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&out[0], (unsigned long long)__double_as_longlong(dmax));
        atomicMax(&out[1], (unsigned long long)__double_as_longlong(amax));
    }
}

template <typename T>
static int sym_check(const T* A, int64_t n, int64_t ld, double* out, void* stream) {
    SKP_ARG(n >= 0 && ld >= n && out && (n == 0 || A), "sym_check: bad arguments");
    cudaStream_t st = SKP_STREAM(stream);
    SKP_CUDA(cudaMemsetAsync(out, 0, 2 * sizeof(double), st));
    if (!n) return SKP_OK;
    const int64_t tiles = cdiv(n, (int64_t)kSymT);
    const int vec_ok = (reinterpret_cast<uintptr_t>(A) % 16 == 0) && (ld * sizeof(T)) % 16 == 0;
    int dev = 0, sms = 148;
    SKP_CUDA(cudaGetDevice(&dev));
    SKP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int64_t pairs = tiles * (tiles + 1) / 2;
    const unsigned grid = (unsigned)std::min<int64_t>(pairs, (int64_t)sms * 8);
    sym_check_kernel<T><<<grid, 256, 0, st>>>(A, n, ld, tiles, vec_ok,
                                             reinterpret_cast<unsigned long long*>(out));
    SKP_LAUNCHED(sym_check_kernel);
    return SKP_OK;
}
extern "C" int skp_sym_check_f32(const float* A, int64_t n, int64_t ld, double* out,
                                 void* stream) {
    return sym_check<float>(A, n, ld, out, stream);
}
extern "C" int skp_sym_check_f64(const double* A, int64_t n, int64_t ld, double* out,
                                 void* stream) {
    return sym_check<double>(A, n, ld, out, stream);
}

extern "C" int skp_cast_f32_f64(const float* x, double* y, int64_t count, void* stream) {
    SKP_ARG(count >= 0, "cast: bad count");
    if (!count) return SKP_OK;
    cast_f32_f64_kernel<<<grid_for(count), 256, 0, SKP_STREAM(stream)>>>(x, y, count);
    SKP_LAUNCHED(cast);
    return SKP_OK;
}
extern "C" int skp_cast_f64_f32(const double* x, float* y, int64_t count, void* stream) {
    SKP_ARG(count >= 0, "cast: bad count");
    if (!count) return SKP_OK;
    cast_f64_f32_kernel<<<grid_for(count), 256, 0, SKP_STREAM(stream)>>>(x, y, count);
    SKP_LAUNCHED(cast);
    return SKP_OK;
}
extern "C" int skp_cast2d_f32_f64(const float* x, int64_t ldx, double* y, int64_t ldy,
                                  int64_t rows, int64_t cols, void* stream) {
    SKP_ARG(rows >= 0 && cols >= 0 && ldx >= cols && ldy >= cols, "cast2d: bad sizes");
    if (!rows || !cols) return SKP_OK;
    cast2d_kernel<float, double><<<grid_for(rows * cols), 256, 0, SKP_STREAM(stream)>>>(
        x, ldx, y, ldy, rows, cols);
    SKP_LAUNCHED(cast2d);
    return SKP_OK;
}
template <typename T>
static int permute_rows(const T* x, int64_t ldx, const int32_t* perm, T* y, int64_t ldy,
                        int64_t rows, int64_t cols, void* stream) {
    SKP_ARG(rows >= 0 && cols >= 0 && ldx >= cols && ldy >= cols, "permute_rows: bad sizes");
    if (!rows || !cols) return SKP_OK;
    const int64_t grid = rows < 65535 ? rows : 65535;
    permute_rows_kernel<T><<<(unsigned)grid, 128, 0, SKP_STREAM(stream)>>>(x, ldx, perm, y, ldy,
                                                                           rows, cols);
    SKP_LAUNCHED(permute_rows);
    return SKP_OK;
}
extern "C" int skp_permute_rows_f32(const float* x, int64_t ldx, const int32_t* perm, float* y,
                                    int64_t ldy, int64_t rows, int64_t cols, void* stream) {
    return permute_rows<float>(x, ldx, perm, y, ldy, rows, cols, stream);
}
extern "C" int skp_permute_rows_f64(const double* x, int64_t ldx, const int32_t* perm, double* y,
                                    int64_t ldy, int64_t rows, int64_t cols, void* stream) {
    return permute_rows<double>(x, ldx, perm, y, ldy, rows, cols, stream);
}
extern "C" int skp_cast2d_f64_f32(const double* x, int64_t ldx, float* y, int64_t ldy,
                                  int64_t rows, int64_t cols, void* stream) {
    SKP_ARG(rows >= 0 && cols >= 0 && ldx >= cols && ldy >= cols, "cast2d: bad sizes");
    if (!rows || !cols) return SKP_OK;
    cast2d_kernel<double, float><<<grid_for(rows * cols), 256, 0, SKP_STREAM(stream)>>>(
        x, ldx, y, ldy, rows, cols);
    SKP_LAUNCHED(cast2d);
    return SKP_OK;
}

extern "C" int skp_symmetrize_f32(float* W, int64_t n, int64_t ld, void* stream) {
    SKP_ARG(n >= 1 && ld >= n, "symmetrize: bad sizes");
    symmetrize_kernel<float><<<grid_for(n * n), 256, 0, SKP_STREAM(stream)>>>(W, n, ld);
    SKP_LAUNCHED(symmetrize);
    return SKP_OK;
}
extern "C" int skp_symmetrize_f64(double* W, int64_t n, int64_t ld, void* stream) {
    SKP_ARG(n >= 1 && ld >= n, "symmetrize: bad sizes");
    symmetrize_kernel<double><<<grid_for(n * n), 256, 0, SKP_STREAM(stream)>>>(W, n, ld);
    SKP_LAUNCHED(symmetrize);
    return SKP_OK;
}
extern "C" int skp_scale_cols_f32(float* X, int64_t rows, int64_t cols, int64_t ld,
                                  const double* scale, void* stream) {
    SKP_ARG(rows >= 0 && cols >= 0 && ld >= cols, "scale_cols: bad sizes");
    if (!rows || !cols) return SKP_OK;
    scale_cols_kernel<float><<<grid_for(rows * cols), 256, 0, SKP_STREAM(stream)>>>(X, rows, cols,
                                                                                   ld, scale);
    SKP_LAUNCHED(scale_cols);
    return SKP_OK;
}
extern "C" int skp_scale_cols_f64(double* X, int64_t rows, int64_t cols, int64_t ld,
                                  const double* scale, void* stream) {
    SKP_ARG(rows >= 0 && cols >= 0 && ld >= cols, "scale_cols: bad sizes");
    if (!rows || !cols) return SKP_OK;
    scale_cols_kernel<double><<<grid_for(rows * cols), 256, 0, SKP_STREAM(stream)>>>(
        X, rows, cols, ld, scale);
    SKP_LAUNCHED(scale_cols);
    return SKP_OK;
}
extern "C" int skp_orth_dev_f64(const double* G, int64_t n, int64_t ld, double* out,
                                void* stream) {
    SKP_ARG(n >= 1 && ld >= n, "orth_dev: bad sizes");
    orth_dev_kernel<<<1, 1024, 0, SKP_STREAM(stream)>>>(G, n, ld, out);
    SKP_LAUNCHED(orth_dev);
    return SKP_OK;
}
extern "C" int skp_eig_orth_f64(const double* W, const double* V, int64_t n, double rel_tol,
                                double* T, int32_t* k_out, void* stream) {
    SKP_ARG(n >= 1, "eig_orth: bad size");
    eig_orth_kernel<<<grid_for(n * n), 256, 0, SKP_STREAM(stream)>>>(W, V, n, rel_tol, T, k_out);
    SKP_LAUNCHED(eig_orth);
    return SKP_OK;
}
extern "C" int skp_sqrt_eigs_f64(const double* W, int64_t n, double* sigma, double* inv,
                                 void* stream) {
    SKP_ARG(n >= 1, "sqrt_eigs: bad size");
    sqrt_eigs_kernel<<<grid_for(n), 256, 0, SKP_STREAM(stream)>>>(W, n, sigma, inv);
    SKP_LAUNCHED(sqrt_eigs);
    return SKP_OK;
}
