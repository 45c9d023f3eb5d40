// tcgen05.mma cta_group::2 issue rate: SS vs TS (A in TMEM), tf32, back-to-back.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}
template <int N, bool TS, bool PAIR>
__global__ void bench(int iters, long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* s = (unsigned char*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    uint32_t rank = 0;
    if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tslot;
    if (warp == 0 && rank == 0) {
        constexpr uint32_t M = PAIR ? 256 : 128;
        constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((M >> 4) << 24);
        const uint32_t a = smem_u32(s), b = smem_u32(s + 65536);
        const uint64_t da = make_desc(a, 16, 512, 4);
        const uint64_t db = make_desc(b, 16, 512, 4);
        const uint32_t ta = tm + 256;
        long long t0 = clock64();
        for (int i = 0; i < iters; i += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint64_t o = (uint64_t)((j & 1) * 2);
                if (TS && PAIR)
                    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\t"
                                 "@p tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, 1;\n\t}"
                                 ::"r"(tm), "r"(ta + (j & 1) * 8), "l"(db + o), "r"(idesc) : "memory");
                else if (TS)
                    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\t"
                                 "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n\t}"
                                 ::"r"(tm), "r"(ta + (j & 1) * 8), "l"(db + o), "r"(idesc) : "memory");
                else if (PAIR)
                    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\t"
                                 "@p tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, 1;\n\t}"
                                 ::"r"(tm), "l"(da + o), "l"(db + o), "r"(idesc) : "memory");
                else
                    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\t"
                                 "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n\t}"
                                 ::"r"(tm), "l"(da + o), "l"(db + o), "r"(idesc) : "memory");
            }
        }
        if (PAIR)
            asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\t"
                         "@p tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
                         ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
        else
            asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\t"
                         "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
                         ::"r"(smem_u32(&bar)) : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
        long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    } else if (PAIR && warp == 0) {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
        if (threadIdx.x == 0) out[blockIdx.x] = 0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    }
}

template <int N, bool TS, bool PAIR>
void run(const char* name, long long* d) {
    auto k = bench<N, TS, PAIR>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
    const int iters = 8192;
    for (int grid : {2, 148}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 140 * 1024;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = PAIR ? 2 : 1; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr; cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k, iters, d);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s err %s\n", name, cudaGetErrorString(e)); return; }
        long long h[148]; cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
        long long mx = 0; for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
        double cyc = (double)mx / iters;
        double macs = (PAIR ? 256.0 : 128.0) * N * 8 / (PAIR ? 2 : 1);
        printf("%-28s grid=%3d: %6.1f cyc/mma  %6.0f MAC/cyc/SM\n", name, grid, cyc, macs / cyc);
    }
}

int main() {
    long long* d; cudaMalloc(&d, 148 * sizeof(long long));
    run<192, false, false>("1cta SS n192", d);
    run<192, true, false>("1cta TS n192", d);
    run<192, false, true>("pair SS n192", d);
    run<192, true, true>("pair TS n192", d);
    run<256, false, true>("pair SS n256", d);
    run<256, true, true>("pair TS n256", d);
    run<96, true, true>("pair TS n96", d);
    return 0;
}
