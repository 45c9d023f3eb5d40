// On-chip ceiling of K2 v2's gather ("commit an SMEM-gather
// ceiling microbenchmark"): 28 warps per SM, each lane holding 44
// register-resident shared-memory byte offsets, stream the K2 step
//     LOP3 (address) -> LDS -> LOP3 (sign) -> FADD
// over a 96 KB row buffer with no HBM traffic at all.  Variants:
//   mode 0: conflict-free schedule (step t: 32 distinct banks), full K2 step
//   mode 1: conflict-free, LDS + FADD only (addresses pre-masked: the LDS issue limit)
//   mode 2: 2-way conflicts on every step (the 1.6 wavefronts/LDS regime)
// Output: LDS/s per SM, shared-memory wavefronts per clock per SM (peak 1 =
// 128 B/clk), and the K2 gather rate in "entries per second" -- the ceiling
// K2's achieved entries/s is compared with (bench.py "frac_onchip").
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 smem_gather.cu -o smem_gather
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kW = 28, kT = 44, kWords = 24576;

template <int MODE>
__global__ void __launch_bounds__(kW * 32, 1) gather(int rows, float* sink, long long* cycles) {
    extern __shared__ __align__(16) float buf[];
    for (int i = threadIdx.x; i < kWords; i += blockDim.x) buf[i] = (float)(i & 7) * 0.25f;
    if (threadIdx.x == 0) buf[kWords - 1] = 0.f;   // the per-row offset word (0)
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t e[kT];
#pragma unroll
    for (int t = 0; t < kT; ++t) {
        // word index: bank = lane (conflict-free) or lane / 2 (2-way) ; row of 32 words per step
        const int row = (warp * 131 + t * 37) % (kWords / 32 - 1);
        const int bank = MODE == 2 ? (lane >> 1) : lane;
        const int word = row * 32 + bank + (MODE == 2 ? (lane & 1) * 32 : 0);
        e[t] = (uint32_t)(word * 4) | ((t & 1) ? 0x80000000u : 0u);
        if (MODE == 1) e[t] &= 0x7fffffffu;
    }
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(buf);
    float acc = 0.f;
    long long t0 = clock64();
    for (int r = 0; r < rows; ++r) {
        // a per-row buffer offset the compiler cannot see (0 at run time), as
        // K2's double-buffered row base: the loads stay inside the row loop
        uint32_t off;
        asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(off) : "r"(base + 4u * (kWords - 1)) : "memory");
        const uint32_t rb = base + off;
#pragma unroll
        for (int t = 0; t < kT; ++t) {
            float x;
            if (MODE == 1) {
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(rb + e[t]));
                acc += x;
            } else {
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(rb + (e[t] & 0x7fffffffu)));
                acc += __int_as_float(__float_as_int(x) ^ (int)(e[t] & 0x80000000u));
            }
        }
    }
    long long t1 = clock64();
    if (acc == 12345.f) sink[threadIdx.x] = acc;
    if (threadIdx.x == 0) atomicMax(cycles, t1 - t0);
}

template <int MODE>
void run(const char* name, int sms) {
    const int rows = 4000;
    float* sink;
    long long* cyc;
    cudaMalloc(&sink, 4096 * 4);
    cudaMalloc(&cyc, 8);
    cudaFuncSetAttribute(gather<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWords * 4);
    gather<MODE><<<sms, kW * 32, kWords * 4>>>(10, sink, cyc);
    cudaMemset(cyc, 0, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    gather<MODE><<<sms, kW * 32, kWords * 4>>>(rows, sink, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double lds = (double)rows * kT * kW;            // warp-LDS per SM
    const double wf = lds * (MODE == 2 ? 2.0 : 1.0);      // wavefronts per SM
    const double entries = (double)sms * lds * 32 / (ms * 1e-3);
    printf("%-34s %8.3f ms  %.3f wavefronts/clk/SM  %.3f LDS/clk/SM  %.3e entries/s (chip)  "
           "clock %.0f MHz\n",
           name, ms, wf / c, lds / c, entries, c / (ms * 1e3));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>("conflict-free, full K2 step", sms);
    run<1>("conflict-free, LDS + FADD", sms);
    run<2>("2-way conflict every step", sms);
    return 0;
}
