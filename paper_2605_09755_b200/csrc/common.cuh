// Shared plumbing for the skp C-ABI: status codes, thread-local last error,
// launch checks, small device helpers.  sm_100a only.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>

#include "../../include/skp.h"

namespace skp {

void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);
void count_launch();

}  // namespace skp

#define SKP_ARG(cond, ...)                                   \
    do {                                                     \
        if (!(cond)) {                                       \
            skp::set_error(__VA_ARGS__);                     \
            return SKP_ERR_ARG;                              \
        }                                                    \
    } while (0)

#define SKP_CUDA(expr)                                                  \
    do {                                                                \
        cudaError_t e__ = (expr);                                       \
        if (e__ != cudaSuccess) return skp::cuda_fail(e__, #expr);      \
    } while (0)

#define SKP_LAUNCHED(name)          \
    do {                            \
        skp::count_launch();        \
        SKP_CUDA(cudaGetLastError()); \
    } while (0)

#define SKP_STREAM(s) (reinterpret_cast<cudaStream_t>(s))

namespace skp {

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sum into lane 0 of warp 0 (blockDim multiple of 32, <= 1024).
template <typename T>
__device__ T block_sum(T v, T* scratch /* >= 32 */) {
    v = warp_sum(v);
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) scratch[w] = v;
    __syncthreads();
    T r = T(0);
    if (w == 0) {
        r = (l < (int)(blockDim.x >> 5)) ? scratch[l] : T(0);
        r = warp_sum(r);
    }
    __syncthreads();
    return r;
}

}  // namespace skp
