// Micro-benchmark: latency of one all-to-all exchange round among G persistent CTAs through
// level-tagged values in global memory (the HODLR sweep's per-level hop).  Each round, every CTA
// publishes NV tagged doubles (st.relaxed.gpu), then its 256 threads poll the values of all other
// CTAs (spinning ld.relaxed.gpu) until every tag is current, then a block barrier.  Prints ns/round.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/xchg_latency tools/xchg_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void st_tagged(double* p, double v, unsigned tag) {
    const unsigned long long bits = ((unsigned long long)__double_as_longlong(v) & ~1ull) | tag;
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;\n" ::"l"(p), "l"(bits) : "memory");
}
__device__ __forceinline__ unsigned long long ld_bits(const double* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}

template <int NV>
__global__ void __launch_bounds__(256, 1) xchg(double* buf, int rounds, int per_thread, unsigned long long* out) {
    const int G = gridDim.x, c = blockIdx.x, t = threadIdx.x;
    unsigned long long t0 = 0;
    for (int lv = 0; lv < rounds; ++lv) {
        if (lv == 2 && t == 0) t0 = clock64();
        const int par = lv & 1;
        const unsigned tag = (unsigned)(lv >> 1) & 1u;
        double* b = buf + (long long)par * G * NV;
        if (t < NV) st_tagged(b + c * NV + t, 1.0 + lv, tag);
        // thread t polls per_thread values spread over all CTAs
        // (every CTA polls every other CTA, so none can run two rounds ahead and reuse a buffer)
        if (per_thread > 0) {
            for (int u = 0; u < per_thread; ++u) {
                const int e = (t % G) * NV + (t / G + u) % NV;
                unsigned n = 0;
                while ((unsigned)(ld_bits(b + e) & 1ull) != tag)
                    if (++n == (1u << 26)) __trap();
            }
        } else {  // 16 polls per thread in flight together, failed ones re-issued
            if (per_thread < 0) {  // first spin on one value alone
                unsigned n = 0;
                while ((unsigned)(ld_bits(b + (t % G) * NV + (t / G) % NV) & 1ull) != tag)
                    if (++n == (1u << 26)) __trap();
            }
            // coalesced like the sweep: warp w reads whole vectors (w * 16 + u) mod G, lane = element
            unsigned long long v[16];
            const int w = t >> 5, l = t & 31;
#define SRC(u) (b + (((w * 16 + (u)) % G) * NV) + l)
#pragma unroll
            for (int u = 0; u < 16; ++u) v[u] = ld_bits(SRC(u));
            for (unsigned n = 0;; ++n) {
                bool ok = true;
#pragma unroll
                for (int u = 0; u < 16; ++u) ok = ok && (unsigned)(v[u] & 1ull) == tag;
                if (ok) break;
                if (n == (1u << 26)) __trap();
#pragma unroll
                for (int u = 0; u < 16; ++u)
                    if ((unsigned)(v[u] & 1ull) != tag) v[u] = ld_bits(SRC(u));
            }
        }
        __syncthreads();
    }
    if (t == 0 && c == 0) *out = clock64() - t0;
}

int main() {
    int G = 128;
    const int rounds = 2000;
    double* buf;
    unsigned long long* out;
    cudaMalloc(&buf, 2 * 148 * 32 * sizeof(double));
    cudaMalloc(&out, 8);
    for (int g : {16, 64, 128, 148}) {
        G = g;
        for (int pt : {1, 0, -1}) {
            cudaMemset(buf, 0xff, 2 * 148 * 32 * sizeof(double));
            void* args[] = {&buf, (void*)&rounds, &pt, &out};
            int r = rounds;
            args[1] = &r;
            cudaLaunchCooperativeKernel((const void*)xchg<32>, dim3(G), dim3(256), args, 0, 0);
            cudaDeviceSynchronize();
            unsigned long long cyc;
            cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
            printf("G=%d polls/thread=%d: %.0f cycles/round\n", G, pt, (double)cyc / (rounds - 2));
        }
    }
    return 0;
}
