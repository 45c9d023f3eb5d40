// Per-SM row-ingest ceiling by path: one 64 KB TMA bulk copy per row vs
// 16-byte cp.async (LDGSTS) issued by all 896 threads, completing on the same
// mbarrier (.noinc arrivals).  Rows L2-resident (1024 rows re-read), two row
// buffers, a row buffer refilled when every warp has passed it.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 ingest_path.cu -o ingest_path
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>  // 0 TMA bulk, 1 cp.async by all threads
__global__ void __launch_bounds__(896, 1) kern(const float* A, int64_t m, int n, int P, int64_t mres, float* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    constexpr int NB = 2;
    const uint32_t row_bytes = n * 4;
    const uint32_t buf = (row_bytes + 127) / 128 * 128;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + NB * buf);
    uint64_t* empty = full + NB;
    const int g = blockIdx.x / P, G = gridDim.x / P;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int b = 0; b < NB; ++b) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&full[b])), "r"(MODE == 0 ? 1 : 896));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[b])), "r"(28));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int b, int64_t row) {
        const char* src = reinterpret_cast<const char*>(A + (row % mres) * (int64_t)n);
        if (MODE == 0) {
            if (threadIdx.x == 0) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[b])), "r"(row_bytes) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(sa(sm + b * buf)), "l"(src), "r"(row_bytes), "r"(sa(&full[b])) : "memory");
            }
        } else {
            for (uint32_t o = threadIdx.x * 16; o < row_bytes; o += 896 * 16)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(sm + b * buf) + o), "l"(src + o) : "memory");
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sa(&full[b])) : "memory");
        }
    };
    for (int b = 0; b < NB; ++b)
        if (g + (int64_t)b * G < m) issue(b, g + (int64_t)b * G);
    float acc = 0.f;
    int it = 0;
    for (int64_t i = g; i < m; i += G, ++it) {
        const int b = it % NB;
        const uint32_t ph = (it / NB) & 1;
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(sa(&full[b])), "r"(ph) : "memory");
        acc += reinterpret_cast<float*>(sm + b * buf)[threadIdx.x];
        const int64_t row = i + (int64_t)NB * G;
        if (MODE == 0) {
            __syncthreads();
            if (row < m) issue(b, row);
        } else {
            // every thread must see all warps done with buffer b before it refills its part
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[b])) : "memory");
            ok = 0;
            while (!ok)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(ok) : "r"(sa(&empty[b])), "r"(ph) : "memory");
            if (row < m) issue(b, row);
        }
    }
    if (acc == 12345.f) *sink = acc;
}

template <int MODE>
void run(const float* A, int64_t m, int n, int P, int G, int64_t mres, float* sink) {
    const size_t smem = 2 * (size_t)(n * 4) + 64;
    cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<MODE><<<G * P, 896, smem>>>(A, m, n, P, mres, sink);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) kern<MODE><<<G * P, 896, smem>>>(A, m, n, P, mres, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 3;
    printf("%s P=%2d G=%2d mres=%6lld: %8.3f ms  per-SM ingest %.1f GB/s  total %.2f TB/s  %s\n",
           MODE == 0 ? "TMA bulk " : "cp.async ", P, G, (long long)(mres < m ? mres : m), ms,
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
    for (int G : {1, 14}) {
        run<0>(A, m / 4, n, 10, G, 1024, sink);
        run<1>(A, m / 4, n, 10, G, 1024, sink);
    }
    run<0>(A, m, n, 10, 14, 1 << 30, sink);
    run<1>(A, m, n, 10, 14, 1 << 30, sink);
    return 0;
}
