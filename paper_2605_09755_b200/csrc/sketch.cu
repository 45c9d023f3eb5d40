// K2 / K3: applying the CountSketch S (n x r, s nonzeros +-1/sqrt(s) per row).
//
// K2  out = A . S  (reference sketching.py:163-164, scipy csc_matvecs)
//     Gather formulation over the CSC of S: out[i][c] = sum_{(j,sg) in col c}
//     sg * A[i][j] / sqrt(s).  A row slab (R rows x n) is staged in shared
//     memory once (one HBM read of A, fused ||A||_F^2 + non-finite count);
//     each thread then owns output columns and gathers ~n*s/r entries per
//     column from the slab.  When a single row does not fit (n*sizeof(T) >
//     ~200 KB) a slab-free variant gathers straight from L2.
// K3  out = S^T . X  (reference sketching.py:181-182)
//     Row gather: out[c][:] = sum_{(j,sg) in col c} sg * X[j][:] / sqrt(s).
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"

namespace skp {

template <typename T>
int sketch_right_rows(const T* A, int64_t lda, int64_t m, int64_t n, const int32_t* colptr,
                      const int32_t* entries, int32_t s, int64_t r, T* out, int64_t ldo,
                      double* fro2, int64_t* nonfinite, void* ws, int64_t ws_bytes,
                      cudaStream_t st);
int64_t sketch_rows_ws_bytes(int64_t n, int32_t s, int64_t r, int elem);

namespace {

constexpr int kSketchThreads = 512;
constexpr int kMaxRows = 8;
constexpr int64_t kSlabBytes = 200 * 1024;

template <typename T>
__device__ __forceinline__ bool finite_v(T x) { return isfinite(x); }

template <typename T>
__global__ void __launch_bounds__(kSketchThreads)
sketch_right_slab_kernel(const T* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                         const int32_t* __restrict__ colptr, const int32_t* __restrict__ entries,
                         T scale, int64_t r, int rows_per_cta, T* __restrict__ out, int64_t ldo,
                         double* fro2, long long* nonfinite) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* slab = reinterpret_cast<T*>(smem_raw);
    __shared__ double red_d[32];
    __shared__ long long red_i[32];
    const int64_t i0 = (int64_t)blockIdx.x * rows_per_cta;
    const int R = (int)((m - i0) < rows_per_cta ? (m - i0) : rows_per_cta);
    // stage R rows (dense, row stride n), fused sum of squares / finiteness
    double ss = 0.0;
    long long bad = 0;
    for (int rr = 0; rr < R; ++rr) {
        const T* src = A + (i0 + rr) * lda;
        T* dst = slab + (int64_t)rr * n;
        for (int64_t j = threadIdx.x; j < n; j += kSketchThreads) {
            T v = __ldg(src + j);
            dst[j] = v;
            ss += (double)v * (double)v;
            bad += !finite_v(v);
        }
    }
    if (fro2 || nonfinite) {
        double bs = block_sum<double>(ss, red_d);
        long long bb = block_sum<long long>(bad, red_i);
        if (threadIdx.x == 0) {
            if (fro2) atomicAdd(fro2, bs);
            if (nonfinite && bb) atomicAdd((unsigned long long*)nonfinite, (unsigned long long)bb);
        }
    }
    __syncthreads();
    for (int64_t c = threadIdx.x; c < r; c += kSketchThreads) {
        T acc[kMaxRows];
#pragma unroll
        for (int k = 0; k < kMaxRows; ++k) acc[k] = T(0);
        const int eb = __ldg(colptr + c), ee = __ldg(colptr + c + 1);
        for (int e = eb; e < ee; ++e) {
            uint32_t v = (uint32_t)__ldg(entries + e);
            int64_t j = v & 0x7fffffffu;
            T sg = (v >> 31) ? T(-1) : T(1);
#pragma unroll
            for (int k = 0; k < kMaxRows; ++k)
                if (k < R) acc[k] += sg * slab[(int64_t)k * n + j];
        }
#pragma unroll
        for (int k = 0; k < kMaxRows; ++k)
            if (k < R) out[(i0 + k) * ldo + c] = acc[k] * scale;
    }
}

// n too large for a one-row slab: one thread per (row, column), gathering from L2.
template <typename T>
__global__ void sketch_right_direct_kernel(const T* __restrict__ A, int64_t lda, int64_t m,
                                           const int32_t* __restrict__ colptr,
                                           const int32_t* __restrict__ entries, T scale,
                                           int64_t r, T* __restrict__ out, int64_t ldo) {
    const int64_t cblocks = (r + blockDim.x - 1) / blockDim.x;
    const int64_t i = (int64_t)blockIdx.x / cblocks;
    const int64_t c = ((int64_t)blockIdx.x % cblocks) * blockDim.x + threadIdx.x;
    if (c >= r || i >= m) return;
    const T* row = A + i * lda;
    T acc = T(0);
    const int eb = __ldg(colptr + c), ee = __ldg(colptr + c + 1);
    for (int e = eb; e < ee; ++e) {
        uint32_t v = (uint32_t)__ldg(entries + e);
        T a = __ldg(row + (v & 0x7fffffffu));
        acc += (v >> 31) ? -a : a;
    }
    out[i * ldo + c] = acc * scale;
}

__device__ __forceinline__ void sq_acc(float v, double& ss, long long& bad) {
    ss = fma((double)v, (double)v, ss);  // fp64 squares: finite inputs cannot overflow
    bad += (__float_as_uint(v) & 0x7f800000u) == 0x7f800000u;
}
__device__ __forceinline__ void sq_acc(double v, double& ss, long long& bad) {
    ss = fma(v, v, ss);
    bad += !isfinite(v);
}

// ||X||_F^2 (fp64) and #non-finite entries: blocks walk rows, threads walk a
// row with 16-byte vector loads (HBM-bound; no per-element index arithmetic)
template <typename T>
__global__ void __launch_bounds__(256)
sumsq_kernel(const T* __restrict__ X, int64_t rows, int64_t cols, int64_t ld, double* out,
             long long* nonfinite) {
    typedef typename std::conditional<sizeof(T) == 4, float4, double2>::type V;
    constexpr int VE = sizeof(V) / sizeof(T);
    __shared__ double red_d[32];
    __shared__ long long red_i[32];
    double ss = 0.0;
    long long bad = 0;
    const bool vec = (reinterpret_cast<uintptr_t>(X) % sizeof(V) == 0) && (ld % VE == 0);
    const int64_t nv = vec ? cols / VE : 0;
    for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) {
        const T* row = X + i * ld;
        const V* rv = reinterpret_cast<const V*>(row);
        for (int64_t j = threadIdx.x; j < nv; j += blockDim.x) {
            const V v = __ldg(rv + j);
            const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
            for (int k = 0; k < VE; ++k) sq_acc(e[k], ss, bad);
        }
        for (int64_t j = nv * VE + threadIdx.x; j < cols; j += blockDim.x) sq_acc(row[j], ss, bad);
    }
    double bs = block_sum<double>(ss, red_d);
    long long bb = block_sum<long long>(bad, red_i);
    if (threadIdx.x == 0) {
        if (out) atomicAdd(out, bs);
        if (nonfinite && bb) atomicAdd((unsigned long long*)nonfinite, (unsigned long long)bb);
    }
}

template <typename T>
__global__ void sketch_left_t_kernel(const T* __restrict__ X, int64_t ldx, int64_t c,
                                     const int32_t* __restrict__ colptr,
                                     const int32_t* __restrict__ entries, T scale,
                                     T* __restrict__ out, int64_t ldo) {
    const int64_t row = blockIdx.x;  // output row = sketch column
    const int eb = __ldg(colptr + row), ee = __ldg(colptr + row + 1);
    for (int64_t q = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; q < c;
         q += (int64_t)gridDim.y * blockDim.x) {
        T acc = T(0);
        for (int e = eb; e < ee; ++e) {
            uint32_t v = (uint32_t)__ldg(entries + e);
            T x = __ldg(X + (int64_t)(v & 0x7fffffffu) * ldx + q);
            acc += (v >> 31) ? -x : x;
        }
        out[row * ldo + q] = acc * scale;
    }
}

template <typename T>
int sketch_right(const T* A, int64_t lda, int64_t m, int64_t n, const int32_t* colptr,
                 const int32_t* entries, int32_t s, int64_t r, T* out, int64_t ldo, double* fro2,
                 int64_t* nonfinite, void* ws, int64_t ws_bytes, void* stream) {
    SKP_ARG(m >= 1 && n >= 1 && r >= 1 && s >= 1, "sketch_right: bad sizes");
    SKP_ARG(lda >= n && ldo >= r, "sketch_right: bad leading dimension");
    cudaStream_t st = SKP_STREAM(stream);
    if (ws) {
        int rc = sketch_right_rows<T>(A, lda, m, n, colptr, entries, s, r, out, ldo, fro2,
                                      nonfinite, ws, ws_bytes, st);
        if (rc != SKP_ERR_UNSUPPORTED) return rc;
    }
    const T scale = T(1) / sqrt(T(s));
    const int64_t row_bytes = n * (int64_t)sizeof(T);
    if (row_bytes <= kSlabBytes) {
        int R = (int)(kSlabBytes / row_bytes);
        if (R > kMaxRows) R = kMaxRows;
        int64_t smem = (int64_t)R * row_bytes;
        SKP_CUDA(cudaFuncSetAttribute(sketch_right_slab_kernel<T>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int64_t grid = cdiv(m, R);
        sketch_right_slab_kernel<T><<<(unsigned)grid, kSketchThreads, smem, st>>>(
            A, lda, m, n, colptr, entries, scale, r, R, out, ldo, fro2,
            reinterpret_cast<long long*>(nonfinite));
        SKP_LAUNCHED(sketch_right_slab_kernel);
        return SKP_OK;
    }
    SKP_ARG(cdiv(r, 256) * m < INT32_MAX, "sketch_right: m too large for the direct path");
    dim3 grid((unsigned)(cdiv(r, 256) * m));
    sketch_right_direct_kernel<T><<<grid, 256, 0, st>>>(A, lda, m, colptr, entries, scale, r, out,
                                                        ldo);
    SKP_LAUNCHED(sketch_right_direct_kernel);
    if (fro2 || nonfinite) {
        sumsq_kernel<T><<<(unsigned)std::min<int64_t>(m, 148 * 8), 256, 0, st>>>(
            A, m, n, lda, fro2, reinterpret_cast<long long*>(nonfinite));
        SKP_LAUNCHED(sumsq_kernel);
    }
    return SKP_OK;
}

template <typename T>
int sketch_left_t(const T* X, int64_t ldx, int64_t n, int64_t c, const int32_t* colptr,
                  const int32_t* entries, int32_t s, int64_t r, T* out, int64_t ldo,
                  void* stream) {
    SKP_ARG(n >= 1 && c >= 1 && r >= 1 && s >= 1, "sketch_left_t: bad sizes");
    SKP_ARG(ldx >= c && ldo >= c, "sketch_left_t: bad leading dimension");
    SKP_ARG(r < 2147483647LL, "sketch_left_t: r too large");
    const T scale = T(1) / sqrt(T(s));
    int threads = c >= 256 ? 256 : (int)(cdiv(c, 32) * 32);
    int64_t ychunks = cdiv(c, threads);
    if (ychunks > 16) ychunks = 16;
    dim3 grid((unsigned)r, (unsigned)ychunks);
    sketch_left_t_kernel<T><<<grid, threads, 0, SKP_STREAM(stream)>>>(X, ldx, c, colptr, entries,
                                                                     scale, out, ldo);
    SKP_LAUNCHED(sketch_left_t_kernel);
    return SKP_OK;
}

template <typename T>
int sumsq(const T* X, int64_t rows, int64_t cols, int64_t ld, double* out, int64_t* nonfinite,
          void* stream) {
    SKP_ARG(rows >= 0 && cols >= 0 && ld >= cols, "sumsq: bad sizes");
    if (rows == 0 || cols == 0) return SKP_OK;
    const int64_t blocks = std::min<int64_t>(rows, 148 * 8);
    sumsq_kernel<T><<<(unsigned)blocks, 256, 0, SKP_STREAM(stream)>>>(
        X, rows, cols, ld, out, reinterpret_cast<long long*>(nonfinite));
    SKP_LAUNCHED(sumsq_kernel);
    return SKP_OK;
}

}  // namespace
}  // namespace skp

using namespace skp;

extern "C" int64_t skp_sketch_right_ws_bytes(int64_t n, int32_t s, int64_t r,
                                             int32_t elem_bytes) {
    return sketch_rows_ws_bytes(n, s, r, elem_bytes);
}
extern "C" int skp_sketch_right_f32(const float* A, int64_t lda, int64_t m, int64_t n,
                                    const int32_t* colptr, const int32_t* entries, int32_t s,
                                    int64_t r, float* out, int64_t ldo, double* fro2,
                                    int64_t* nonfinite, void* ws, int64_t ws_bytes,
                                    void* stream) {
    return sketch_right<float>(A, lda, m, n, colptr, entries, s, r, out, ldo, fro2, nonfinite,
                               ws, ws_bytes, stream);
}
extern "C" int skp_sketch_right_f64(const double* A, int64_t lda, int64_t m, int64_t n,
                                    const int32_t* colptr, const int32_t* entries, int32_t s,
                                    int64_t r, double* out, int64_t ldo, double* fro2,
                                    int64_t* nonfinite, void* ws, int64_t ws_bytes,
                                    void* stream) {
    return sketch_right<double>(A, lda, m, n, colptr, entries, s, r, out, ldo, fro2, nonfinite,
                                ws, ws_bytes, stream);
}
extern "C" int skp_sketch_left_t_f32(const float* X, int64_t ldx, int64_t n, int64_t c,
                                     const int32_t* colptr, const int32_t* entries, int32_t s,
                                     int64_t r, float* out, int64_t ldo, void* stream) {
    return sketch_left_t<float>(X, ldx, n, c, colptr, entries, s, r, out, ldo, stream);
}
extern "C" int skp_sketch_left_t_f64(const double* X, int64_t ldx, int64_t n, int64_t c,
                                     const int32_t* colptr, const int32_t* entries, int32_t s,
                                     int64_t r, double* out, int64_t ldo, void* stream) {
    return sketch_left_t<double>(X, ldx, n, c, colptr, entries, s, r, out, ldo, stream);
}
extern "C" int skp_sumsq_f32(const float* X, int64_t rows, int64_t cols, int64_t ld, double* out,
                             int64_t* nonfinite, void* stream) {
    return sumsq<float>(X, rows, cols, ld, out, nonfinite, stream);
}
extern "C" int skp_sumsq_f64(const double* X, int64_t rows, int64_t cols, int64_t ld,
                             double* out, int64_t* nonfinite, void* stream) {
    return sumsq<double>(X, rows, cols, ld, out, nonfinite, stream);
}
