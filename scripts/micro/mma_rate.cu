// Microbenchmark: cycles per tcgen05.mma (SS operands, garbage smem) by kind /
// N / operand major-ness / swizzle, issued back-to-back by one thread, and the
// same with a commit+wait round trip after every k MMAs.
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

struct Cfg { int kind; int n; int amn; int bmn; int layA; int layB; int sync_every; int nacc; int m; };

__global__ void bench(Cfg c, int iters, long long* out) {
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
    if (threadIdx.x == 0) {
        // kind 0: tf32 (a/b fmt 2), kind 1: f16 (fmt 0), both f32 accum
        uint32_t fmt = c.kind == 0 ? 2u : 0u;
        uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)c.amn << 15) |
                         ((uint32_t)c.bmn << 16) | ((uint32_t)(c.n >> 3) << 17) | ((uint32_t)(c.m >> 4) << 24);
        uint32_t a = smem_u32(s), b = smem_u32(s + 65536);
        uint64_t da = make_desc(a, c.amn ? 4096 : 16, c.amn ? 512 : (c.layA == 2 ? 1024 : 512), c.layA);
        uint64_t db = make_desc(b, c.bmn ? 4096 : 16, c.bmn ? 512 : (c.layB == 2 ? 1024 : 512), c.layB);
        uint32_t ph = 0;
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t tmd = tm + (uint32_t)((i % c.nacc) * c.n);
            if (c.kind == 0)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(tmd), "l"(da), "l"(db), "r"(idesc), "r"(1) : "memory");
            else
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(tmd), "l"(da), "l"(db), "r"(idesc), "r"(1) : "memory");
            if (c.sync_every && (i + 1) % c.sync_every == 0) {
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
                uint32_t ok = 0;
                while (!ok)
                    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                                 : "=r"(ok) : "r"(smem_u32(&bar)), "r"(ph) : "memory");
                ph ^= 1;
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(&bar)), "r"(ph) : "memory");
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    }
}

int main() {
    long long* d; cudaMalloc(&d, 148 * sizeof(long long));
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
    // layout codes: 1 = SW128_BASE32B, 2 = SW128, 4 = SW64, 6 = SW32, 0 = none
    Cfg cfgs[] = {
        {0, 176, 0, 1, 4, 1, 0, 1, 128}, {0, 128, 0, 1, 4, 1, 0, 2, 128}, {0, 128, 0, 1, 4, 1, 0, 4, 128},
        {0, 64, 0, 1, 4, 1, 0, 1, 128}, {0, 64, 0, 1, 4, 1, 0, 4, 128}, {0, 32, 0, 1, 4, 1, 0, 1, 128},
        {0, 256, 0, 0, 4, 4, 0, 2, 128}, {0, 128, 0, 0, 4, 4, 0, 1, 64}, {1, 256, 0, 0, 2, 2, 0, 2, 128},
        {0, 16, 0, 0, 4, 4, 0, 1, 128}, {0, 16, 0, 0, 4, 4, 0, 8, 128},
    };
    const int iters = 4096;
    for (auto& c : cfgs) {
        for (int grid : {1, 148}) {
            bench<<<grid, 128, 140 * 1024>>>(c, iters, d);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            long long h[148]; cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
            long long mx = 0; for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
            printf("m=%d nacc=%d kind=%s n=%d amn=%d bmn=%d layA=%d layB=%d sync_every=%d grid=%d: %.1f cyc/mma\n",
                   c.m, c.nacc, c.kind ? "f16" : "tf32", c.n, c.amn, c.bmn, c.layA, c.layB, c.sync_every, grid,
                   (double)mx / iters);
        }
    }
    return 0;
}
