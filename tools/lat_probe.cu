// FP64 / shuffle / shared-memory / barrier latency probe (one warp or one CTA, dependent chains).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_probe tools/lat_probe.cu
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b) {
    double x = a + threadIdx.x;
    __shared__ double sm[64];
    sm[threadIdx.x] = x;
    __syncwarp();
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1000; ++i) { x = fma(x, b, a); }
    long long t1 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1000; ++i) { x = x + b; }
    long long t2 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1000; ++i) { x = __shfl_xor_sync(0xffffffffu, x, 1) + 0.0; }
    long long t3 = clock64();
    int idx = threadIdx.x;
#pragma unroll 1
    for (int i = 0; i < 1000; ++i) { double v = sm[idx]; idx = (int)v & 31; x += v; }
    long long t4 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1000; ++i) { __syncthreads(); }
    long long t5 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8 * 256); cudaMalloc(&c, 64);
    for (int nt : {32, 256}) {
        k<<<1, nt>>>(o, c, 1e-3, 0.999); long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
        printf("threads %d: DFMA %.1f DADD %.1f SHFL64+DADD %.1f LDS+DADD(dep) %.1f BAR %.1f cycles\n", nt, h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0, h[4] / 1000.0);
    }
}
