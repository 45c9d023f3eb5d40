// Dependent-chain latencies on one warp (DFMA, 64-bit SHFL, rsqrtf, f64<->f32):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat scripts/micro/lat.cu
// B200 (this pool): DFMA 9, SHFL.f64 + DADD 39, rsqrtf + FADD 44, F2F + DADD 14 cycles.
#include <cstdio>
__global__ void k(double* o, long long* c, int n) {
    double a = o[threadIdx.x], b = 1.0000001, x = 0.5;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = fma(a, b, x);
    long long t1 = clock64();
    double s = a;
    for (int i = 0; i < n; ++i) s = __shfl_sync(0xffffffffu, s, (threadIdx.x + 1) & 31) + 1e-9;
    long long t2 = clock64();
    float f = (float)s;
    for (int i = 0; i < n; ++i) f = rsqrtf(f) + 0.5f;
    long long t3 = clock64();
    double d = s;
    for (int i = 0; i < n; ++i) d = (double)(float)d + 0.25;
    long long t4 = clock64();
    o[threadIdx.x] = a + s + f + d;
    if (threadIdx.x == 0) { c[0] = (t1 - t0) / n; c[1] = (t2 - t1) / n; c[2] = (t3 - t2) / n; c[3] = (t4 - t3) / n; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8 * 32); cudaMalloc(&c, 32); cudaMemset(o, 0, 256);
    k<<<1, 32>>>(o, c, 1000);
    long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("cycles: DFMA dep %lld, SHFL.f64+DADD dep %lld, rsqrtf+FADD dep %lld, F2F d->f->d + DADD %lld\n", h[0], h[1], h[2], h[3]);
}
