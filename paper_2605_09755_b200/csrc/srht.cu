// K7: subsampled randomized Hadamard transform (reference sketching.py:65-90,
// :125-130, :167-171, :185-189), both directions in one strided kernel:
//
//   out[f, c] = scale * (H D pad(x_f))[subset[c]],   c < r
//
// for fibres f of the input: rows of A (apply_right: A S) or columns of X
// (apply_left_transpose: S^T X).  D = diag(signs) over the n_pad = 2^p
// padded coordinates, H the unnormalised Sylvester Hadamard matrix, scale =
// 1/sqrt(r).  The signs and the sorted subset are numpy's draw (host).
//
// One CTA per fibre at a time (persistent over fibres): the signed, padded
// fibre is loaded coalesced, its levels for index bits 0..4 are done across
// each warp with shuffles (lane = index % 32), it is staged in shared memory
// and the remaining levels run in passes of up to four in registers (radix
// 16 at strides >= 32, bank-conflict free), so 2^14 points take 3 passes /
// 3 block barriers instead of 14.  The Hadamard factors commute, so the
// level order does not change the result.
// Then the r subset coordinates are gathered (scaled) to the output.
// Bound: shared memory (2 x n_pad x elem bytes per pass) -- the FLOPs are
// n_pad log2 n_pad per fibre.
#include <algorithm>

#include "common.cuh"

namespace skp {
namespace {

constexpr int kSrhtThreads = 512;

template <typename T>
__global__ void __launch_bounds__(kSrhtThreads)
srht_kernel(const T* __restrict__ X, int64_t fibres, int64_t n, int64_t x_fs, int64_t x_es,
            const int8_t* __restrict__ signs, int logn, const int32_t* __restrict__ subset, int64_t r,
            T scale, T* __restrict__ out, int64_t o_fs, int64_t o_es) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    T* v = reinterpret_cast<T*>(sm_raw);
    const int npad = 1 << logn;
    const int lane = threadIdx.x & 31;
    const int lowbits = min(5, logn);  // levels done by warp shuffles
    for (int64_t f = blockIdx.x; f < fibres; f += gridDim.x) {
        const T* x = X + f * x_fs;
        // load + sign, then the levels of bits 0..4 in registers across the
        // warp (element j sits in lane j % 32: blockDim is a multiple of 32)
        // 16 loads of this thread in flight before any use (latency)
        for (int k0 = 0; k0 * kSrhtThreads < npad; k0 += 16) {
            T a[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const int j = threadIdx.x + (k0 + k) * kSrhtThreads;
                a[k] = (j < npad && j < n) ? x[(int64_t)j * x_es] * (T)signs[j] : (T)0;
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const int j = threadIdx.x + (k0 + k) * kSrhtThreads;
                if ((k0 + k) * kSrhtThreads < npad) {  // warp-uniform
#pragma unroll
                    for (int sb = 0; sb < 5; ++sb) {
                        if (sb < lowbits) {
                            const T b = __shfl_xor_sync(0xffffffffu, a[k], 1 << sb);
                            a[k] = (lane & (1 << sb)) ? b - a[k] : a[k] + b;
                        }
                    }
                    if (j < npad) v[j] = a[k];
                }
            }
        }
        __syncthreads();
        // bits 5.. in radix-16 register passes at strides h >= 32 (the 32
        // lanes of a warp touch 32 consecutive words: no bank conflicts)
        for (int lb = lowbits; lb < logn; lb += 4) {
            const int levels = min(4, logn - lb), w = 1 << levels, h = 1 << lb;
            const int groups = npad >> levels;
            for (int g = threadIdx.x; g < groups; g += blockDim.x) {
                const int base = ((g >> lb) << (lb + levels)) + (g & (h - 1));
                T e[16];
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    if (i < w) e[i] = v[base + i * h];
#pragma unroll
                for (int s = 1; s < 16; s <<= 1) {
                    if (s < w) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            if (i < w && !(i & s)) {
                                const T a = e[i], b = e[i + s];
                                e[i] = a + b;
                                e[i + s] = a - b;
                            }
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    if (i < w) v[base + i * h] = e[i];
            }
            __syncthreads();
        }
        T* o = out + f * o_fs;
        for (int64_t c = threadIdx.x; c < r; c += blockDim.x) o[c * o_es] = v[subset[c]] * scale;
        __syncthreads();
    }
}

template <typename T>
int srht_apply(const T* X, int64_t fibres, int64_t n, int64_t x_fs, int64_t x_es,
               const int8_t* signs, int64_t npad, const int32_t* subset, int64_t r, double scale,
               T* out, int64_t o_fs, int64_t o_es, cudaStream_t st) {
    SKP_ARG(fibres >= 0 && n >= 1 && r >= 1 && npad >= n && npad >= r, "srht: bad sizes");
    SKP_ARG((npad & (npad - 1)) == 0, "srht: padded length must be a power of two");
    SKP_ARG(X && signs && subset && out, "srht: null pointer");
    int logn = 0;
    while ((int64_t(1) << logn) < npad) ++logn;
    const size_t smem = (size_t)npad * sizeof(T);
    if (smem > 200 * 1024) {
        set_error("unsupported: srht needs the padded fibre (%lld x %d bytes) in shared memory",
                  (long long)npad, (int)sizeof(T));
        return SKP_ERR_UNSUPPORTED;
    }
    if (fibres == 0) return SKP_OK;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    SKP_CUDA(cudaFuncSetAttribute(srht_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    int per_sm = 1;
    SKP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, srht_kernel<T>, kSrhtThreads,
                                                           smem));
    const int64_t grid = std::min<int64_t>(fibres, (int64_t)sms * std::max(1, per_sm));
    srht_kernel<T><<<(unsigned)grid, kSrhtThreads, smem, st>>>(X, fibres, n, x_fs, x_es, signs, logn,
                                                              subset, r, (T)scale, out, o_fs, o_es);
    SKP_LAUNCHED(srht_kernel);
    return SKP_OK;
}

}  // namespace
}  // namespace skp

using namespace skp;

extern "C" int skp_srht_apply_f32(const float* X, int64_t fibres, int64_t n, int64_t x_fs,
                                  int64_t x_es, const int8_t* signs, int64_t n_pad,
                                  const int32_t* subset, int64_t r, double scale, float* out,
                                  int64_t o_fs, int64_t o_es, void* stream) {
    return srht_apply<float>(X, fibres, n, x_fs, x_es, signs, n_pad, subset, r, scale, out, o_fs,
                             o_es, SKP_STREAM(stream));
}
extern "C" int skp_srht_apply_f64(const double* X, int64_t fibres, int64_t n, int64_t x_fs,
                                  int64_t x_es, const int8_t* signs, int64_t n_pad,
                                  const int32_t* subset, int64_t r, double scale, double* out,
                                  int64_t o_fs, int64_t o_es, void* stream) {
    return srht_apply<double>(X, fibres, n, x_fs, x_es, signs, n_pad, subset, r, scale, out, o_fs,
                              o_es, SKP_STREAM(stream));
}
