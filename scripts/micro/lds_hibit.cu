#include <cstdio>
#include <cstdint>
__global__ void k(float* out, uint32_t hib) {
    __shared__ float buf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (float)i;
    __syncthreads();
    uint32_t a = (uint32_t)__cvta_generic_to_shared(buf) + 4u * threadIdx.x;
    float x;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(a | hib));
    out[threadIdx.x] = x;
}
int main() {
    float* o; cudaMalloc(&o, 128);
    for (uint32_t hib : {0u, 0x01000000u, 0x80000000u}) {
        k<<<1, 32>>>(o, hib);
        cudaError_t e = cudaDeviceSynchronize();
        float h[32] = {};
        if (e == cudaSuccess) cudaMemcpy(h, o, 128, cudaMemcpyDeviceToHost);
        printf("hibit %08x -> %s, out[5] = %g\n", hib, cudaGetErrorString(e), h[5]);
        if (e != cudaSuccess) break;
    }
    return 0;
}
