// Shared-memory Stockham FFTs of length 2^LG (<= 1024) for groups of threads: the transforms of the
// tau-PCG block solve (K5, precond_iter.cu) and of the FFT operator apply (K1f, toeplitz_fft.cu).
#pragma once

#include <cuda_runtime.h>


namespace fib {
namespace {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 mul_i(double2 a, bool inv) {  // -i a (forward), +i a (inverse)
    return inv ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}
// shared-memory index with one pad element per 8 (the radix-8 scatter of the first pass is conflict-free)
__device__ __forceinline__ int pad8(int i) { return i + (i >> 3); }


// Stockham FFT of length L = 2^LG by the L/8 threads (index t) of one group, between the group's two padded
// shared buffers (index pad8(i)): radix-8 passes, one radix-2 or radix-4 pass first when LG % 3 != 0, one
// butterfly per thread.  Input in src (natural order); the output lands in src when the number of passes is
// even, else in dst (natural order).  LG and the direction are template parameters so the index arithmetic
// folds to constants.  tw: the STAGE twiddle table (fft_stage_twiddles): per radix-8 pass of span p > 1 the
// seven factors exp(-2 pi i m k / (8p)) as [m - 1][k], so that the lanes of a warp (consecutive k) read
// consecutive entries — a table indexed m k L / (8p) put up to 8 lanes of a warp on one bank (measured:
// 8x the ideal shared-memory wavefronts on those loads).  Every thread of the CTA must call it (it contains
// __syncthreads); groups without a unit pass active = false.  Not inlined: one copy per length and direction
// serves every pass (instruction cache).
__device__ __forceinline__ void dft8(double2 (&v)[8], bool inv) {
    constexpr double r = 0.70710678118654752440;
    double2 b[8];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        b[m] = cadd(v[m], v[m + 4]);
        b[m + 4] = csub(v[m], v[m + 4]);
    }
    if (!inv) {
        b[5] = make_double2(r * (b[5].x + b[5].y), r * (b[5].y - b[5].x));
        b[7] = make_double2(r * (b[7].y - b[7].x), -r * (b[7].x + b[7].y));
    } else {
        b[5] = make_double2(r * (b[5].x - b[5].y), r * (b[5].x + b[5].y));
        b[7] = make_double2(-r * (b[7].x + b[7].y), r * (b[7].x - b[7].y));
    }
    b[6] = mul_i(b[6], inv);
    const double2 c0 = cadd(b[0], b[2]), c2 = csub(b[0], b[2]), c1 = cadd(b[1], b[3]), c3 = mul_i(csub(b[1], b[3]), inv);
    const double2 c4 = cadd(b[4], b[6]), c6 = csub(b[4], b[6]), c5 = cadd(b[5], b[7]), c7 = mul_i(csub(b[5], b[7]), inv);
    v[0] = cadd(c0, c1);
    v[4] = csub(c0, c1);
    v[2] = cadd(c2, c3);
    v[6] = csub(c2, c3);
    v[1] = cadd(c4, c5);
    v[5] = csub(c4, c5);
    v[3] = cadd(c6, c7);
    v[7] = csub(c6, c7);
}

// The stage twiddle table of length L = 2^lg (it needs fewer than L entries) from exp(-2 pi i k / L):
// full(k) for k < L.  All threads of the CTA cooperate; the caller synchronises.
template <class Full>
__device__ __forceinline__ void fft_stage_twiddles(double2* dst, int lg, Full full) {
    const int L = 1 << lg, rem = lg % 3;
    int off = 0;
    for (int s = rem; s < lg; s += 3) {
        const int p = 1 << s;
        if (p > 1) {
            for (int q = threadIdx.x; q < 7 * p; q += blockDim.x) {
                const int m = q / p + 1, k = q % p;
                dst[off + q] = full((m * k * (L / (8 * p))) & (L - 1));
            }
            off += 7 * p;
        }
    }
}

template <int LG, bool INV>
__device__ __noinline__ void fft_group(double2* src, double2* dst, const double2* tw, int t, bool active) {
    constexpr int L = 1 << LG, NT = (L >> 3) > 0 ? (L >> 3) : 1, REM = LG % 3;
    if constexpr (REM == 1) {
        if (active)
            for (int j = t; j < (L >> 1); j += NT) {
                const double2 x0 = src[pad8(j)], x1 = src[pad8(j + (L >> 1))];
                dst[pad8(2 * j)] = cadd(x0, x1);
                dst[pad8(2 * j + 1)] = csub(x0, x1);
            }
        __syncthreads();
        double2* tt = src;
        src = dst;
        dst = tt;
    } else if constexpr (REM == 2) {
        constexpr int Q = L >> 2;
        if (active)
            for (int j = t; j < Q; j += NT) {
                const double2 a0 = src[pad8(j)], a1 = src[pad8(j + Q)], a2 = src[pad8(j + 2 * Q)], a3 = src[pad8(j + 3 * Q)];
                const double2 s02 = cadd(a0, a2), d02 = csub(a0, a2), s13 = cadd(a1, a3), d13 = mul_i(csub(a1, a3), INV);
                dst[pad8(4 * j)] = cadd(s02, s13);
                dst[pad8(4 * j + 1)] = cadd(d02, d13);
                dst[pad8(4 * j + 2)] = csub(s02, s13);
                dst[pad8(4 * j + 3)] = csub(d02, d13);
            }
        __syncthreads();
        double2* tt = src;
        src = dst;
        dst = tt;
    }
    constexpr int Q8 = L >> 3;
    int off = 0;
#pragma unroll
    for (int s = REM; s < LG; s += 3) {
        const int p = 1 << s;
        if (active && Q8 > 0) {
            const int j = t, k = j & (p - 1);
            double2 v[8];
#pragma unroll
            for (int m = 0; m < 8; ++m) v[m] = src[pad8(j + m * Q8)];
            if (p > 1) {
#pragma unroll
                for (int m = 1; m < 8; ++m) {
                    double2 w = tw[off + (m - 1) * p + k];
                    if (INV) w.y = -w.y;
                    v[m] = make_double2(v[m].x * w.x - v[m].y * w.y, v[m].x * w.y + v[m].y * w.x);
                }
            }
            dft8(v, INV);
            const int o = 8 * (j - k) + k;
#pragma unroll
            for (int m = 0; m < 8; ++m) dst[pad8(o + m * p)] = v[m];
        }
        if (p > 1) off += 7 * p;
        __syncthreads();
        double2* tt = src;
        src = dst;
        dst = tt;
    }
}
constexpr int kFftRadix = 8;
// runtime dispatch on the transform length; returns the buffer index (0 = src) holding the output
__device__ __forceinline__ int fft_dispatch(double2* src, double2* dst, int lg, const double2* tw, bool inv, int t,
                                            bool active) {
#define FI_FFT_CASE(n)                                        \
    case n:                                                   \
        if (inv) fft_group<n, true>(src, dst, tw, t, active); \
        else fft_group<n, false>(src, dst, tw, t, active);    \
        break;
    switch (lg) {
        FI_FFT_CASE(2)
        FI_FFT_CASE(3)
        FI_FFT_CASE(4)
        FI_FFT_CASE(5)
        FI_FFT_CASE(6)
        FI_FFT_CASE(7)
        FI_FFT_CASE(8)
        FI_FFT_CASE(9)
        FI_FFT_CASE(10)
        default: __trap();
    }
#undef FI_FFT_CASE
    return ((lg / 3) + (lg % 3 ? 1 : 0)) & 1;
}


}  // namespace
}  // namespace fib
