// Row ingest at C5's K2 geometry (n = 16384 floats per column pass, 64 KB
// rows): P slice CTAs per row group each need every row in shared memory.
// Unicast (each CTA bulk-copies the row itself, as K2 v2 does) against cluster
// multicast (the C CTAs of a cluster each fetch 1/C of the row once and
// multicast it to all C; a buffer is refilled when every CTA of the cluster
// released it).  No gather: this is the L2 -> SM delivery ceiling alone.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 row_multicast.cu -o row_multicast
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void wait_par(uint64_t* bar, uint32_t ph) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(sa(bar)), "r"(ph) : "memory");
}

// C = 1: unicast.  C > 1: cluster of C CTAs = C slices of one row group.
template <int C>
__global__ void ingest(const float* A, int64_t m, int n, int P, int64_t* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    constexpr int NB = 2;
    const uint32_t row_bytes = n * 4;
    const uint32_t buf = (row_bytes + 127) / 128 * 128;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + NB * buf);
    uint64_t* empty = full + NB;
    const int g = blockIdx.x / P, G = gridDim.x / P;
    const uint32_t rank = C > 1 ? cta_rank() : 0;
    const uint32_t chunk = row_bytes / C;
    if (threadIdx.x == 0) {
        for (int b = 0; b < NB; ++b) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[b])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[b])), "r"(C));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (C > 1) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else __syncthreads();
    auto issue = [&](int b, int64_t row) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[b])), "r"(row_bytes) : "memory");
        if (C == 1) {
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(sa(sm + b * buf)), "l"(A + row * (int64_t)n), "r"(row_bytes), "r"(sa(&full[b])) : "memory");
        } else {
            const uint16_t mask = (uint16_t)((1u << C) - 1);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;"
                         ::"r"(sa(sm + b * buf) + rank * chunk), "l"(reinterpret_cast<const char*>(A + row * (int64_t)n) + rank * chunk),
                         "r"(chunk), "r"(sa(&full[b])), "h"(mask) : "memory");
        }
    };
    if (threadIdx.x == 0)
        for (int b = 0; b < NB; ++b)
            if (g + (int64_t)b * G < m) issue(b, g + (int64_t)b * G);
    float acc = 0.f;
    int it = 0;
    for (int64_t i = g; i < m; i += G, ++it) {
        const int b = it % NB;
        const uint32_t ph = (it / NB) & 1;
        wait_par(&full[b], ph);
        acc += reinterpret_cast<float*>(sm + b * buf)[threadIdx.x];
        __syncthreads();
        if (threadIdx.x == 0) {
            const int64_t row = i + (int64_t)NB * G;
            if (C > 1) {
                // release buffer b in every CTA of the cluster, then wait for all C releases
                for (uint32_t d = 0; d < C; ++d) {
                    uint32_t remote;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(sa(&empty[b])), "r"(d));
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
                }
                if (row < m) {
                    uint32_t ok = 0;
                    while (!ok)
                        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                                     : "=r"(ok) : "r"(sa(&empty[b])), "r"(ph) : "memory");
                    issue(b, row);
                }
            } else if (row < m) {
                issue(b, row);
            }
        }
    }
    if (C > 1) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (acc == 12345.f) *sink = 1;
}

template <int C>
void run(const float* A, int64_t m, int n, int P, int G, int64_t* sink) {
    const size_t smem = 2 * (size_t)(n * 4) + 64;
    cudaFuncSetAttribute(ingest<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (C > 8) cudaFuncSetAttribute(ingest<C>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G * P);
    cfg.blockDim = dim3(896);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, ingest<C>, &cfg);
    cudaLaunchKernelEx(&cfg, ingest<C>, A, m, n, P, sink);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) cudaLaunchKernelEx(&cfg, ingest<C>, A, m, n, P, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 3;
    const double bytes = (double)m * n * 4 * P;
    printf("C=%2d P=%2d G=%2d (%3d CTAs, max active clusters %3d): %8.3f ms  delivered %.2f TB/s  "
           "unique %.2f TB/s  C5-scaled pass %.1f ms  (%s)\n",
           C, P, G, G * P, ncl, ms, bytes / (ms * 1e-3) / 1e12, (double)m * n * 4 / (ms * 1e-3) / 1e12,
           ms * (1048576.0 / m), cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int64_t m = 131072;
    const int n = 16384;
    float* A;
    int64_t* sink;
    cudaMalloc(&A, m * n * 4);
    cudaMemset(A, 0, m * n * 4);
    cudaMalloc(&sink, 8);
    run<1>(A, m, n, 10, 14, sink);   // K2 v2 today at C5
    run<1>(A, m, n, 8, 18, sink);
    run<1>(A, m, n, 1, 144, sink);   // every row once: the unique-byte rate
    run<2>(A, m, n, 10, 14, sink);
    run<2>(A, m, n, 8, 18, sink);
    run<4>(A, m, n, 8, 18, sink);
    run<4>(A, m, n, 8, 16, sink);
    run<8>(A, m, n, 8, 18, sink);
    run<8>(A, m, n, 8, 16, sink);
    run<8>(A, m, n, 8, 14, sink);
    run<16>(A, m, n, 16, 8, sink);
    return 0;
}
