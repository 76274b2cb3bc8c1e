// FP64 peak probe for the B200 roofline denominator (DMMA tensor pipe and DFMA).
// Register-only loops with 4 independent accumulator chains per warp; best of 10
// CUDA-event timings. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
    double c[4][2] = {};
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int q = 0; q < 4; ++q) s += c[q][0] + c[q][1];
    if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dfma_loop(double* out, int iters) {
    double c[8];
    for (int q = 0; q < 8; ++q) c[q] = q;
    double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q) c[q] = fma(c[q], a, b);
    }
    double s = 0;
    for (int q = 0; q < 8; ++q) s += c[q];
    if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out;
    cudaMalloc(&out, 1 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int threads : {128, 256, 512, 1024}) {
        for (int blocks_per_sm : {1, 2}) {
            int grid = sms * blocks_per_sm;
            float best = 1e30f;
            for (int r = 0; r < 11; ++r) {
                cudaEventRecord(e0);
                dmma_loop<<<grid, threads>>>(out, iters);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (r > 0 && ms < best) best = ms;
            }
            double flops = 2.0 * 256 * 4 * (double)iters * (grid * threads / 32);
            printf("{\"probe\":\"dmma_m8n8k4\",\"threads\":%d,\"grid\":%d,\"tflops\":%.3f}\n", threads, grid,
                   flops / best / 1e9);
            best = 1e30f;
            for (int r = 0; r < 11; ++r) {
                cudaEventRecord(e0);
                dfma_loop<<<grid, threads>>>(out, iters);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (r > 0 && ms < best) best = ms;
            }
            flops = 2.0 * 8 * (double)iters * grid * threads;
            printf("{\"probe\":\"dfma\",\"threads\":%d,\"grid\":%d,\"tflops\":%.3f}\n", threads, grid,
                   flops / best / 1e9);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
