// Per-SM bulk-copy ingress: P CTAs per row group stream whole rows (n floats)
// into a double-buffered smem row exactly like K2 v2, without the gather.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 bulk_ingress.cu -o bulk_ingress
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void ingress(const float* A, int64_t m, int n, int P, int nbuf, int64_t* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    const uint32_t row_bytes = n * 4;
    const uint32_t buf = (row_bytes + 127) / 128 * 128;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + nbuf * buf);
    const int g = blockIdx.x / P, G = gridDim.x / P;
    if (threadIdx.x == 0) {
        for (int b = 0; b < nbuf; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[b])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    float acc = 0.f;
    if (threadIdx.x == 0) {
        for (int b = 0; b < nbuf; ++b) {
            int64_t row = g + (int64_t)b * G;
            if (row < m) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[b])), "r"(row_bytes) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(sa(sm + b * buf)), "l"(A + row * (int64_t)n), "r"(row_bytes), "r"(sa(&full[b])) : "memory");
            }
        }
    }
    int it = 0;
    for (int64_t i = g; i < m; i += G, ++it) {
        const int b = it % nbuf;
        const uint32_t ph = (it / nbuf) & 1;
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(sa(&full[b])), "r"(ph) : "memory");
        acc += reinterpret_cast<float*>(sm + b * buf)[threadIdx.x];
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t row = i + (int64_t)nbuf * G;
            if (row < m) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[b])), "r"(row_bytes) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(sa(sm + b * buf)), "l"(A + row * (int64_t)n), "r"(row_bytes), "r"(sa(&full[b])) : "memory");
            }
        }
    }
    if (acc == 12345.f) *sink = 1;
}

int main() {
    const int64_t m = 262144;
    const int n = 16384;
    float* A;
    int64_t* sink;
    cudaMalloc(&A, m * n * 4);
    cudaMemset(A, 0, m * n * 4);
    cudaMalloc(&sink, 8);
    for (int P : {1, 6}) {
        for (int nbuf : {2, 3}) {
            const int G = 144 / P;
            const size_t smem = nbuf * (size_t)(n * 4) + 64;
            cudaFuncSetAttribute(ingress, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            ingress<<<G * P, 768, smem>>>(A, m, n, P, nbuf, sink);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            for (int r = 0; r < 3; ++r) ingress<<<G * P, 768, smem>>>(A, m, n, P, nbuf, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            ms /= 3;
            const double bytes = (double)m * n * 4 * P;
            printf("P=%d nbuf=%d: %.3f ms  per-SM ingress %.1f GB/s  total %.2f TB/s  (%s)\n", P, nbuf, ms,
                   bytes / (G * P) / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e12,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
