// Cycles per call of K5 32x32 tile factor + inverse (tile_chol_inv), one CTA.
// Measured: the block version (one barrier per step) 22.8k cycles; a one-warp
// register version (row per lane, shuffles; fully unrolled) 21.1k -- and 48.9k
// with a shuffle-based inverse: the unrolled straight-line code (~50 KB) is
// instruction-fetch bound, so the block version stays.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tc scripts/micro/tile_chol.cu -lcuda -Lpaper_2605_09755_b200 -lskp
#include "../../paper_2605_09755_b200/csrc/cholinv.cu"
#include <cstdio>
namespace skp { namespace {
__global__ void __launch_bounds__(256, 1) bench_tile(const double* g, double* out, long long* cyc) {
    __shared__ CIShared sh;
    for (int q = threadIdx.x; q < CB * CB; q += blockDim.x) sh.c[q / CB][q % CB] = g[q];
    __syncthreads();
    double mn, mx;
    long long t0 = 0;
    for (int it = 0; it < 101; ++it) {
        if (it == 1) t0 = clock64();
        for (int q = threadIdx.x; q < CB * CB; q += blockDim.x) sh.a[q / CB][q % CB] = sh.c[q / CB][q % CB];
        __syncthreads();
        tile_chol_inv(sh.a, sh.b, sh.e, sh.invd, &mn, &mx);
        __syncthreads();
    }
    if (threadIdx.x == 0) *cyc = (clock64() - t0) / 100;
    for (int q = threadIdx.x; q < CB * CB; q += blockDim.x) out[q] = sh.b[q / CB][q % CB];
}
}}
int main() {
    double h[1024];
    for (int i = 0; i < 32; ++i) for (int j = 0; j < 32; ++j) h[i * 32 + j] = (i == j ? 40.0 : 0.0) + 1.0 / (1 + i + j);
    double *g, *o; long long* c;
    cudaMalloc(&g, 8192); cudaMalloc(&o, 8192); cudaMalloc(&c, 8);
    cudaMemcpy(g, h, 8192, cudaMemcpyHostToDevice);
    skp::bench_tile<<<1, 256>>>(g, o, c);
    long long cyc; cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("tile_chol_inv: %lld cycles per call (%s)\n", cyc, cudaGetErrorString(cudaGetLastError()));
}
