// TMA load throughput per SM by box geometry (L2-resident source), all SMs.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int DIMS>
__global__ void bench(const __grid_constant__ CUtensorMap map, int iters, uint32_t box_bytes, int nstage,
                      int rows_span, long long* out, int prefetch) {
    if (prefetch) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* s = (unsigned char*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t bars[16];
    (void)0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < nstage; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    long long t0 = clock64();
    constexpr int NS = 8;
    nstage = NS;
    int c1 = blockIdx.x % rows_span;
    for (int it = 0; it < iters; ++it) {
        const int st = it & (NS - 1);
        const uint32_t ph = (it >> 3) & 1;
        if (it >= nstage) {
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(ok) : "r"(smem_u32(&bars[st])), "r"(ph ^ 1) : "memory");
        }
        asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\t"
                     "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t}" ::"r"(smem_u32(&bars[st])), "r"(box_bytes) : "memory");
        if (++c1 >= rows_span) c1 = 0;
        if (DIMS == 2)
            asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\t"
                         "@p cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n\t}"
                         ::"r"(smem_u32(s + st * 24576)), "l"(&map), "r"(smem_u32(&bars[st])), "r"(0), "r"(c1 * 16) : "memory");
        else
            asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\t"
                         "@p cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n\t}"
                         ::"r"(smem_u32(s + st * 24576)), "l"(&map), "r"(smem_u32(&bars[st])), "r"(0), "r"(c1 * 16), "r"(0) : "memory");
    }
    for (int i = 0; i < NS; ++i) {
        const int it = iters - NS + i;
        const int st = it & (NS - 1);
        const uint32_t ph = (it >> 3) & 1;
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(&bars[st])), "r"(ph) : "memory");
    }
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

PFN_cuTensorMapEncodeTiled_v12000 enc;

void run2d(const char* name, float* base, uint64_t cols, uint64_t rows, uint32_t bc, uint32_t br,
           CUtensorMapSwizzle sw, long long* d) {
    CUtensorMap m;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 4};
    cuuint32_t box[2] = {bc, br};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("%s encode failed %d\n", name, r); return; }
    uint32_t bytes = bc * br * 4;
    int iters = 4000, nst = bytes <= 8192 ? 12 : 6;
    cudaFuncSetAttribute(bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int pf = 0; pf < 2; ++pf) {
    bench<2><<<148, 32, 200 * 1024>>>(m, iters, bytes, nst, (int)(rows / 16 - br / 16), d, pf);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s err %s\n", name, cudaGetErrorString(e)); exit(1); }
    long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    double cyc = (double)mx / iters;
    printf("%-36s pf=%d box %5u B: %7.1f cyc/box  %5.1f B/clk/SM  %5.2f cyc/row\n", name, pf, bytes, cyc, bytes / cyc, cyc / br);
  }
}

int main() {
    cudaDriverEntryPointQueryResult q; void* fn;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    long long* d; cudaMalloc(&d, 148 * sizeof(long long));
    // L2-resident: 4096 rows x 128 cols fp32 = 2 MB (row = 512 B) / wide rows 4096 x 512
    float* a; cudaMalloc(&a, 64 << 20); cudaMemset(a, 0, 64 << 20);
    run2d("K-major SW64  {16 x 128}", a, 128, 4096, 16, 128, CU_TENSOR_MAP_SWIZZLE_64B, d);
    run2d("K-major SW128 {32 x 128}", a, 128, 4096, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B, d);
    run2d("K-major SW128 {32 x 192}", a, 128, 4096, 32, 192, CU_TENSOR_MAP_SWIZZLE_128B, d);
    run2d("K-major SW32  {8 x 128}", a, 128, 4096, 8, 128, CU_TENSOR_MAP_SWIZZLE_32B, d);
    run2d("MN 128B-atom32 {32 x 16}", a, 128, 4096, 32, 16, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, d);
    run2d("MN none {32 x 16}", a, 128, 4096, 32, 16, CU_TENSOR_MAP_SWIZZLE_NONE, d);
    run2d("none {64 x 64} 256B rows", a, 128, 4096, 64, 64, CU_TENSOR_MAP_SWIZZLE_NONE, d);
    run2d("none {128 x 32} 512B rows", a, 128, 4096, 128, 32, CU_TENSOR_MAP_SWIZZLE_NONE, d);


    return 0;
}
