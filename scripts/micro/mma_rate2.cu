// Clean tcgen05.mma issue-rate probe: warp-uniform descriptors, elect.sync
// inside the asm, unrolled x8, fixed accumulator.
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
__device__ __forceinline__ void mma_tf32_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 r;\n\t"
                 "elect.sync r|p, 0xffffffff;\n\t"
                 "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n\t}"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc) : "memory");
}
__device__ __forceinline__ void mma_f16_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 r;\n\t"
                 "elect.sync r|p, 0xffffffff;\n\t"
                 "@p tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t}"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc) : "memory");
}

template <int KIND, int N, int AMN, int BMN, int LAYA, int LAYB>
__global__ void bench(int iters, long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* s = (unsigned char*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tslot;
    if (warp == 0) {
        constexpr uint32_t fmt = KIND == 0 ? 2u : 0u;
        constexpr uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)AMN << 15) |
                                   ((uint32_t)BMN << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint32_t a = smem_u32(s), b = smem_u32(s + 65536);
        const uint64_t da = make_desc(a, AMN ? 4096 : 16, 512, LAYA);
        const uint64_t db = make_desc(b, BMN ? 4096 : 16, 512, LAYB);
        long long t0 = clock64();
        for (int i = 0; i < iters; i += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint64_t o = (uint64_t)((j & 1) * 2);  // +32 B K-step
                if (KIND == 0) mma_tf32_elect(tm, da + o, db + o, idesc);
                else mma_f16_elect(tm, da + o, db + o, idesc);
            }
        }
        asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\t"
                     "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
                     ::"r"(smem_u32(&bar)) : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
        long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    }
}

template <int KIND, int N, int AMN, int BMN, int LAYA, int LAYB>
void run(const char* name, long long* d) {
    auto k = bench<KIND, N, AMN, BMN, LAYA, LAYB>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
    const int iters = 8192;
    for (int grid : {1, 148}) {
        k<<<grid, 128, 140 * 1024>>>(iters, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s err %s\n", name, cudaGetErrorString(e)); return; }
        long long h[148]; cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
        long long mx = 0; for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
        double cyc = (double)mx / iters;
        double macs = 128.0 * N * (KIND == 0 ? 8 : 16);
        printf("%-34s grid=%3d: %6.1f cyc/mma  %6.0f MAC/cyc/SM\n", name, grid, cyc, macs / cyc);
    }
}

int main() {
    long long* d; cudaMalloc(&d, 148 * sizeof(long long));
    run<0, 176, 0, 1, 4, 1>("tf32 n176 K-maj SW64 / MN SW128_32", d);
    run<0, 176, 0, 0, 4, 4>("tf32 n176 SW64 / SW64", d);
    run<0, 176, 0, 0, 2, 2>("tf32 n176 SW128 / SW128", d);
    run<0, 176, 1, 1, 1, 1>("tf32 n176 MN / MN", d);
    run<0, 256, 0, 0, 2, 2>("tf32 n256 SW128 / SW128", d);
    run<0, 128, 0, 0, 2, 2>("tf32 n128 SW128 / SW128", d);
    run<0, 64, 0, 0, 2, 2>("tf32 n64 SW128 / SW128", d);
    run<1, 256, 0, 0, 2, 2>("f16 n256 SW128 / SW128", d);
    run<1, 128, 0, 0, 2, 2>("f16 n128 SW128 / SW128", d);
    return 0;
}
