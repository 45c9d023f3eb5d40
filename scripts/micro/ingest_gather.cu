// Do K2's row ingest (bulk copies into shared memory) and its gather (LDS)
// share a bottleneck?  140 CTAs x 28 warps at C5's pass geometry (64 KB rows,
// P = 10 slice CTAs per row group): per row every warp runs S conflict-free
// LDS + FADD steps.  Modes: gather only (rows already resident), ingest only
// (S = 0), both.  If both ~ max(gather, ingest) the resources are separate.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 ingest_gather.cu -o ingest_gather
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int S, int NB = 2, int NCH = 1>
__global__ void __launch_bounds__(896, 1) kern(const float* A, int64_t m, int n, int P, int ingest, float* sink, int64_t mres) {
    extern __shared__ __align__(128) unsigned char sm[];
    const uint32_t row_bytes = n * 4;
    const uint32_t buf = (row_bytes + 127) / 128 * 128;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + NB * buf);
    uint32_t* done = reinterpret_cast<uint32_t*>(full + NB);
    const int g = blockIdx.x / P, G = gridDim.x / P;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int b = 0; b < NB; ++b) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[b])));
            done[b] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < NB * (int)buf / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1.f;
    __syncthreads();
    auto issue = [&](int b, int64_t row) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[b])), "r"(row_bytes) : "memory");
        for (int c = 0; c < NCH; ++c)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(sa(sm + b * buf) + c * (row_bytes / NCH)), "l"(reinterpret_cast<const char*>(A + (row % mres) * (int64_t)n) + c * (row_bytes / NCH)),
                         "r"(row_bytes / NCH), "r"(sa(&full[b])) : "memory");
    };
    if (ingest && threadIdx.x == 0)
        for (int b = 0; b < NB; ++b)
            if (g + (int64_t)b * G < m) issue(b, g + (int64_t)b * G);
    // conflict-free schedule: step t of lane L reads bank L
    uint32_t e[S > 0 ? S : 1];
#pragma unroll
    for (int t = 0; t < S; ++t) e[t] = sa(sm) + 4u * (uint32_t)(lane + 32 * ((t * 7 + lane * 3 + warp * 11) % 512));
    float acc = 0.f;
    int it = 0;
    for (int64_t i = g; i < m; i += G, ++it) {
        const int b = it % NB;
        const uint32_t ph = (it / NB) & 1;
        if (ingest) {
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(ok) : "r"(sa(&full[b])), "r"(ph) : "memory");
        }
#pragma unroll
        for (int t = 0; t < S; ++t) asm volatile("" : "+r"(e[t]));
#pragma unroll
        for (int t = 0; t < S; ++t) {
            float x;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(e[t] + (uint32_t)b * buf));
            acc += x;
        }
        __syncwarp();
        if (lane == 0 && atomicAdd(&done[b], 1u) == 27) {
            done[b] = 0;
            const int64_t row = i + (int64_t)NB * G;
            if (ingest && row < m) issue(b, row);
        }
    }
    if (acc == 12345.f) *sink = acc;
}

template <int S, int NB = 2, int NCH = 1>
void run(const float* A, int64_t m, int n, int ingest, float* sink, int P = 10, int G = 14, int64_t mres = 1 << 30) {
    const size_t smem = NB * (size_t)(n * 4) + 64;
    cudaFuncSetAttribute(kern<S, NB, NCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<S, NB, NCH><<<G * P, 896, smem>>>(A, m, n, P, ingest, sink, mres);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) kern<S, NB, NCH><<<G * P, 896, smem>>>(A, m, n, P, ingest, sink, mres);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 3;
    printf("NB=%d NCH=%d S=%2d ingest=%d P=%2d G=%3d mres=%lld: %8.3f ms  (C5 pass scaled %.1f ms)  per-SM ingest %.1f GB/s  total %.2f TB/s  %s\n",
           NB, NCH, S, ingest, P, G, (long long)(mres < m ? mres : m), ms, ms * 1048576.0 / m,
           (double)m * n * 4 * P / (G * P) / (ms * 1e-3) / 1e9, (double)m * n * 4 * P / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int64_t m = 131072;
    const int n = 16384;
    float* A;
    float* sink;
    cudaMalloc(&A, m * n * 4);
    cudaMemset(A, 0, m * n * 4);
    cudaMalloc(&sink, 8);
    run<0>(A, m, n, 1, sink);
    run<0, 3>(A, m, n, 1, sink);
    run<0, 2, 4>(A, m, n, 1, sink);
    run<0, 3, 4>(A, m, n, 1, sink);
    for (int G : {1, 14}) {
        run<0>(A, m / 4, n, 1, sink, 10, G, 1024);
        run<0, 3>(A, m / 4, n, 1, sink, 10, G, 1024);
        run<0, 3, 4>(A, m / 4, n, 1, sink, 10, G, 1024);
    }
    run<24>(A, m, n, 1, sink);
    run<24, 3>(A, m, n, 1, sink);
    run<24, 3, 4>(A, m, n, 1, sink);
    return 0;
}
