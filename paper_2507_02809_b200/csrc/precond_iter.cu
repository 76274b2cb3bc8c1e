// K5 — the substituted per-block solve for 2D blocks too large to invert densely (configs 2-4).
//
// The reference factorises every diagonal block densely (krylov.cpp:24-46) and refuses blocks
// above its cap of 4096 (ResourceLimitError).  For the 2D BASELINE configurations (N = 127^2,
// 255^2) each block is solved instead by tau-preconditioned CG on the SPD form (
// the oracle's TauPCG runs the identical recurrence):
//   G_s y = r  <=>  M y = r / D2,   M = c B + diag(delta),  delta = e0 D1/D2 (f-block: c = cr, 0)
//   tau^{-1} = S diag(1/(c g(theta) + mean(delta))) S,   S = orthonormal 2D DST-I
// B x is a 2D circulant-embedded convolution (forward/inverse 2D FFT of size L1 x L2 with
// L_i = 2(n_i + 1) a power of two); the DST-I is an odd-extended FFT of the same size.  The FFTs are
// hand-written Stockham transforms in shared memory.
//
// Control flow never returns to the host inside an apply: the whole forward substitution (level
// loop, CG loop, scalars) is ONE cooperative kernel, tau_pcg_fused, with grid barriers between the
// row and column passes of each CG step.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "precond.cuh"

namespace fib {
namespace {

constexpr int CB = 4;   // columns per CTA of the setup column FFT (spectrum of B)

// warm start: extrapolation order (previous levels used) and the coefficients
// (-1)^(j+1) C(k, j) of the degree-(k-1) polynomial through them
constexpr int kWarmOrder = 6;
__constant__ double kWarmCoef[kWarmOrder + 1][kWarmOrder + 1] = {
    {0, 0, 0, 0, 0, 0, 0},          {0, 1, 0, 0, 0, 0, 0},           {0, 2, -1, 0, 0, 0, 0},
    {0, 3, -3, 1, 0, 0, 0},         {0, 4, -6, 4, -1, 0, 0},         {0, 5, -10, 10, -5, 1, 0},
    {0, 6, -15, 20, -15, 6, -1}};

struct ItArgs {
    int n1, n2, ld2, L1, L2, lg1, lg2, S, levels, maxit;
    long long Np;
    double tol, cs, cr, e0, inv_LL;
    const double2* tw1;  // exp(-2 pi i k / L1), k < L1/2
    const double2* tw2;
    const double* lamB;  // L1 x L2 real spectrum of the embedded B
    const double* lamT;  // n1 x n2 tau eigenvalues g(theta)
    const double* dmean; // per level mean(delta)
    const int* direct;   // per level: D2 == 0 (G = e0 D1)
    const double* z_in;  // right-hand side of P (padded layout)
    double* y;           // output of P (padded layout); x of the level is y's slice
    const double* D1;
    const double* d2inv;
    const double* e;
    double* r;
    double* zz;  // PCG z
    double* p;
    double* Ap;
    double2* X;   // L1 x L2 complex work
    double* hb;   // 8 x Np: old part of the L1 history of the current 8-level block's targets
    double* Rr;   // n1 x n2 real DST work
    const int* skip;
    int warm;    // extrapolated initial guesses for the time levels (FI_TAU_WARM, default 1)
};

__device__ __forceinline__ bool skipped(const ItArgs& a) { return a.skip && *a.skip; }
__device__ __forceinline__ double level_c(const ItArgs& a, int lv) { return lv < a.S ? a.cs : a.cr; }
__device__ __forceinline__ double level_dmean(const ItArgs& a, int lv) { return lv < a.S ? a.dmean[lv] : 0.0; }

// ------------------------------------------------------------------ Stockham radix-2 FFT in smem
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// `cnt` independent length-L transforms stored back to back in src (ping-pong with dst);
// returns the buffer holding the result.  tw: L/2 forward twiddles (conjugated for inverse).
__device__ double2* fft_smem(double2* src, double2* dst, int cnt, int L, int lg, const double2* tw, bool inverse,
                             int tid, int nthr) {
    const int half = L >> 1;
    for (int s = 0, p = 1; s < lg; ++s, p <<= 1) {
        for (int q = tid; q < cnt * half; q += nthr) {
            const int c = q / half, j = q - c * half;
            const int k = j & (p - 1);
            double2 w = __ldg(tw + k * (half / p));
            if (inverse) w.y = -w.y;
            const double2* sc = src + c * L;
            double2* dc = dst + c * L;
            const double2 x0 = sc[j];
            const double2 x1 = cmul(sc[j + half], w);
            dc[2 * j - k] = make_double2(x0.x + x1.x, x0.y + x1.y);
            dc[2 * j - k + p] = make_double2(x0.x - x1.x, x0.y - x1.y);
        }
        __syncthreads();
        double2* t = src;
        src = dst;
        dst = t;
    }
    return src;
}

// Radix-4 Stockham variant for the fused kernel: half the passes (and __syncthreads) of fft_smem,
// power-of-two index arithmetic, twiddles from a shared-memory copy of the half table
// (tw[t] = exp(-2 pi i t / L), t < L/2; t >= L/2 uses -tw[t - L/2]).  Same transform as fft_smem.
__device__ __forceinline__ double2 tw_at(const double2* tw, int t, int half) {
    if (t < half) return tw[t];
    const double2 w = tw[t - half];
    return make_double2(-w.x, -w.y);
}
__device__ double2* fft4_smem(double2* src, double2* dst, int cnt, int L, int lg, const double2* tw, bool inverse,
                              int tid, int nthr) {
    const int half = L >> 1;
    int s = 0, p = 1;
    if (lg & 1) {  // one radix-2 pass first (p = 1: no twiddles)
        for (int q = tid; q < cnt * half; q += nthr) {
            const int c = q >> (lg - 1), j = q & (half - 1);
            const double2* sc = src + c * L;
            double2* dc = dst + c * L;
            const double2 x0 = sc[j], x1 = sc[j + half];
            dc[2 * j] = make_double2(x0.x + x1.x, x0.y + x1.y);
            dc[2 * j + 1] = make_double2(x0.x - x1.x, x0.y - x1.y);
        }
        __syncthreads();
        double2* t = src;
        src = dst;
        dst = t;
        s = 1;
        p = 2;
    }
    const int quarter = L >> 2;
    for (; s < lg; s += 2, p <<= 2) {
        const int lgp = s;  // p = 2^s
        const int tstep = L >> (lgp + 2);  // L / (4p)
        for (int q = tid; q < cnt * quarter; q += nthr) {
            const int c = q >> (lg - 2), j = q & (quarter - 1);
            const int k = j & (p - 1);
            const double2* sc = src + c * L;
            double2* dc = dst + c * L;
            double2 a0 = sc[j], a1 = sc[j + quarter], a2 = sc[j + 2 * quarter], a3 = sc[j + 3 * quarter];
            if (k) {
                double2 w1 = tw_at(tw, k * tstep, half), w2 = tw_at(tw, 2 * k * tstep, half),
                        w3 = tw_at(tw, 3 * k * tstep, half);
                if (inverse) {
                    w1.y = -w1.y;
                    w2.y = -w2.y;
                    w3.y = -w3.y;
                }
                a1 = cmul(a1, w1);
                a2 = cmul(a2, w2);
                a3 = cmul(a3, w3);
            }
            const double2 s02 = make_double2(a0.x + a2.x, a0.y + a2.y), d02 = make_double2(a0.x - a2.x, a0.y - a2.y);
            const double2 s13 = make_double2(a1.x + a3.x, a1.y + a3.y), d13 = make_double2(a1.x - a3.x, a1.y - a3.y);
            // forward: y1 = d02 - i d13, y3 = d02 + i d13 (inverse: signs of i swapped)
            const double2 id13 = inverse ? make_double2(-d13.y, d13.x) : make_double2(d13.y, -d13.x);  // -/+ i d13
            const int o = 4 * (j - k) + k;
            dc[o] = make_double2(s02.x + s13.x, s02.y + s13.y);
            dc[o + p] = make_double2(d02.x + id13.x, d02.y + id13.y);
            dc[o + 2 * p] = make_double2(s02.x - s13.x, s02.y - s13.y);
            dc[o + 3 * p] = make_double2(d02.x - id13.x, d02.y - id13.y);
        }
        __syncthreads();
        double2* t = src;
        src = dst;
        dst = t;
    }
    return src;
}

// circulant spectrum of the embedded B: lamB = Re FFT2(c), c[k1][k2] = a[l1][l2]
__global__ void spec_embed(ItArgs a, const double* gen, int gen_stride) {
    const long long tot = (long long)a.L1 * a.L2;
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < tot; q += (long long)gridDim.x * blockDim.x) {
        const int k1 = (int)(q / a.L2), k2 = (int)(q % a.L2);
        const int l1 = k1 < a.n1 ? k1 : (k1 > a.L1 - a.n1 ? k1 - a.L1 : 1 << 30);
        const int l2 = k2 < a.n2 ? k2 : (k2 > a.L2 - a.n2 ? k2 - a.L2 : 1 << 30);
        double val = 0.0;
        if (l1 != (1 << 30) && l2 != (1 << 30)) val = gen[(long long)(l1 + a.n1 - 1) * gen_stride + l2 + a.ld2];
        a.X[q] = make_double2(val, 0.0);
    }
}
__global__ void fft_rows_plain(ItArgs a) {
    extern __shared__ double2 sm[];
    double2* u = sm;
    double2* v = sm + a.L2;
    double2* row = a.X + (long long)blockIdx.x * a.L2;
    for (int j = threadIdx.x; j < a.L2; j += blockDim.x) u[j] = row[j];
    __syncthreads();
    const double2* U = fft_smem(u, v, 1, a.L2, a.lg2, a.tw2, false, threadIdx.x, blockDim.x);
    for (int j = threadIdx.x; j < a.L2; j += blockDim.x) row[j] = U[j];
}
__global__ void fft_cols_to_spec(ItArgs a, double* lamB) {
    extern __shared__ double2 sm[];
    double2* u = sm;
    double2* v = sm + CB * a.L1;
    const int k0 = blockIdx.x * CB;
    for (int q = threadIdx.x; q < CB * a.L1; q += blockDim.x) {
        const int c = q / a.L1, j = q - c * a.L1;
        u[q] = a.X[(long long)j * a.L2 + k0 + c];
    }
    __syncthreads();
    const double2* U = fft_smem(u, v, CB, a.L1, a.lg1, a.tw1, false, threadIdx.x, blockDim.x);
    for (int q = threadIdx.x; q < CB * a.L1; q += blockDim.x) {
        const int c = q / a.L1, j = q - c * a.L1;
        lamB[(long long)j * a.L2 + k0 + c] = U[q].x;
    }
}

// ------------------------------------------------------------------ fused persistent solve
// The whole forward substitution of a tau-PCG preconditioner apply in ONE cooperative kernel: the
// level loop and the CG loop run on the device, the FFT passes of a CG step are phases separated
// by grid barriers (6 per step instead of 7 dependent kernel launches), the scalars of the
// recurrence (alpha, beta, rz, ...) live in every CTA's registers, and the global dot products are
// summed in a fixed order (every CTA obtains the identical, bit-reproducible value).
struct FusedCtl {
    unsigned* bar;    // monotone grid-barrier counter (zeroed before the launch)
    double* parts;    // 2 x G block partials (ping-pong by reduction index)
    unsigned long long* trace;  // optional [10] per-phase time sums of CTA 0 (FI_ITER_TRACE=1)
    int rpc;    // rows per CTA in the row passes (G * rpc >= n1)
    int cbf;    // columns per CTA in the column passes (power of two, cbf * L1 <= 8 * 256)
    int lgcbf;
    int cbt, lgcbt;  // the same for the tau column pass (n2 columns instead of L2)
};
__device__ __forceinline__ unsigned long long gtime_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(256, 2) tau_pcg_fused(ItArgs a, FusedCtl ctl) {
    if (skipped(a)) return;
    extern __shared__ double2 sm[];
    __shared__ double wred[8];
    __shared__ double bcast;
    const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x, nthr = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nwarp = nthr >> 5;
    const long long Np = a.Np;
    const int rpc = ctl.rpc, cbf = ctl.cbf, lgc = ctl.lgcbf, cbt = ctl.cbt, lgt = ctl.lgcbt;
    unsigned target = 0;
    int rk = 0;
    unsigned long long tlast = 0;
    auto stamp = [&](int ph) {
        if (ctl.trace && cta == 0 && tid == 0) {
            const unsigned long long now = gtime_ns();
            if (tlast) ctl.trace[ph] += now - tlast;
            tlast = now;
        }
    };
    auto gsync = [&]() {
        __syncthreads();
        if (tid == 0) {
            const unsigned long long t0 = ctl.trace && cta == 0 ? gtime_ns() : 0;
            target += (unsigned)G;
            __threadfence();
            atomicAdd(ctl.bar, 1u);
            unsigned n = 0;
            // relaxed polls (an acquire load invalidates the SM's L1 on every iteration), one acquire
            while (ld_relaxed_u32(ctl.bar) < target) {
                __nanosleep(32);
                if (++n == (1u << 26)) __trap();
            }
            (void)ld_acquire_u32(ctl.bar);
            if (ctl.trace && cta == 0) {
                ctl.trace[8] += gtime_ns() - t0;
                ctl.trace[9] += 1;
            }
        }
        __syncthreads();
    };
    // deterministic grid sum: block partials in fixed order, every CTA gets the same total
    auto greduce = [&](double v) -> double {
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) wred[warp] = v;
        __syncthreads();
        double* pp = ctl.parts + (rk & 1) * G;
        if (tid == 0) {
            double b = 0.0;
            for (int w = 0; w < nwarp; ++w) b += wred[w];
            __stcg(pp + cta, b);
        }
        gsync();
        if (warp == 0) {
            // all of a lane's partials in flight at once (G <= 320), then a fixed-order sum
            double pv[10];
#pragma unroll
            for (int u2 = 0; u2 < 10; ++u2) {
                const int k = lane + 32 * u2;
                pv[u2] = k < G ? __ldcg(pp + k) : 0.0;
            }
            double t = 0.0;
#pragma unroll
            for (int u2 = 0; u2 < 10; ++u2) t += pv[u2];
            for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
            if (lane == 0) bcast = t;
        }
        __syncthreads();
        ++rk;
        return bcast;
    };
    const double sc1 = sqrt(2.0 / (a.n1 + 1)) * -0.5, sc2 = sqrt(2.0 / (a.n2 + 1)) * -0.5;
    const int hs = max(rpc * a.L2, cbf * a.L1);
    double2* u = sm;
    double2* v = sm + hs;           // ping-pong halves
    double2* tws1 = sm + 2 * hs;    // twiddle half tables in shared memory
    double2* tws2 = tws1 + a.L1 / 2;
    for (int t = tid; t < a.L1 / 2; t += nthr) tws1[t] = a.tw1[t];
    for (int t = tid; t < a.L2 / 2; t += nthr) tws2[t] = a.tw2[t];
    __syncthreads();
    // this CTA's rows for every row pass (G * rpc >= n1): r0 .. r0 + nr - 1, transformed together
    const int r0 = cta * rpc, nr = max(0, min(rpc, a.n1 - r0));

    // rows n1..L1-1 of the embedded B input stay zero for the whole apply
    for (long long q = (long long)cta * nthr + tid; q < (long long)(a.L1 - a.n1) * a.L2; q += (long long)G * nthr)
        a.X[(long long)a.n1 * a.L2 + q] = make_double2(0.0, 0.0);

    // DST-I along this CTA's rows of `src` (row stride sstride, n2 values) into the same rows of Rr
    auto dst_rows = [&](const double* src, long long sstride) {
        if (nr == 0) return;
        for (int q = tid; q < nr * a.L2; q += nthr) {
            const int i = q >> a.lg2, j = q & (a.L2 - 1);
            const double* row = src + (long long)(r0 + i) * sstride;
            double val = 0.0;
            if (j >= 1 && j <= a.n2) val = row[j - 1];
            else if (j >= a.n2 + 2) val = -row[a.L2 - j - 1];
            u[q] = make_double2(val, 0.0);
        }
        __syncthreads();
        const double2* U = fft4_smem(u, v, nr, a.L2, a.lg2, tws2, false, tid, nthr);
        for (int q = tid; q < nr * a.n2; q += nthr) {
            const int i = q / a.n2, k = q - i * a.n2;
            a.Rr[(long long)(r0 + i) * a.n2 + k] = sc2 * U[i * a.L2 + k + 1].y;
        }
        __syncthreads();
    };
    // column pass of the tau solve: DST along columns, divide by the tau eigenvalues, DST back
    auto tau_cols_phase = [&](int lv) {
        const double c = level_c(a, lv), dmean = level_dmean(a, lv);
        const int ngroups = (a.n2 + cbt - 1) / cbt;
        for (int g = cta; g < ngroups; g += G) {
            const int k0 = g * cbt, nc = min(cbt, a.n2 - k0);
            // the tau eigenvalues of the element each thread divides later are loaded with the data
            double ilam[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const int q = tid + t * nthr;
                const int cc = q & (cbt - 1), j = q >> lgt;  // column fastest: adjacent loads
                ilam[t] = 0.0;
                if (q < cbt * a.L1) {
                    double val = 0.0;
                    if (cc < nc) {
                        int k = -1;
                        if (j >= 1 && j <= a.n1) {
                            val = a.Rr[(long long)(j - 1) * a.n2 + k0 + cc];
                            k = j;
                        } else if (j >= a.n1 + 2) {
                            val = -a.Rr[(long long)(a.L1 - j - 1) * a.n2 + k0 + cc];
                            k = a.L1 - j;
                        }
                        if (k > 0) ilam[t] = a.lamT[(long long)(k - 1) * a.n2 + k0 + cc];
                    }
                    u[cc * a.L1 + j] = make_double2(val, 0.0);
                }
            }
            __syncthreads();
            double2* U = fft4_smem(u, v, cbt, a.L1, a.lg1, tws1, false, tid, nthr);
            double2* W = U == u ? v : u;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const int q = tid + t * nthr;
                if (q < cbt * a.L1) {
                    const int cc = q & (cbt - 1), j = q >> lgt;
                    double val = 0.0;
                    if (cc < nc) {
                        int k = -1;
                        double sgn = 1.0;
                        if (j >= 1 && j <= a.n1) k = j;
                        else if (j >= a.n1 + 2) {
                            k = a.L1 - j;
                            sgn = -1.0;
                        }
                        if (k > 0) val = sgn * (sc1 * U[cc * a.L1 + k].y) / (c * ilam[t] + dmean);
                    }
                    W[cc * a.L1 + j] = make_double2(val, 0.0);
                }
            }
            __syncthreads();
            double2* V = W == u ? v : u;
            const double2* R = fft4_smem(W, V, cbt, a.L1, a.lg1, tws1, false, tid, nthr);
            for (int q = tid; q < nc * a.n1; q += nthr) {
                const int cc = q % nc, k = q / nc;
                a.Rr[(long long)k * a.n2 + k0 + cc] = sc1 * R[cc * a.L1 + k + 1].y;
            }
            __syncthreads();
        }
    };
    // final row pass of the tau solve: zz = DST rows of Rr, returns the partial r.zz; init: p = zz
    auto tau_out_phase = [&](bool init) -> double {
        double part = 0.0;
        if (nr == 0) return part;
        for (int q = tid; q < nr * a.L2; q += nthr) {
            const int i = q >> a.lg2, j = q & (a.L2 - 1);
            const double* src = a.Rr + (long long)(r0 + i) * a.n2;
            double val = 0.0;
            if (j >= 1 && j <= a.n2) val = src[j - 1];
            else if (j >= a.n2 + 2) val = -src[a.L2 - j - 1];
            u[q] = make_double2(val, 0.0);
        }
        __syncthreads();
        const double2* U = fft4_smem(u, v, nr, a.L2, a.lg2, tws2, false, tid, nthr);
        for (int q = tid; q < nr * a.n2; q += nthr) {
            const int i = q / a.n2, k = q - i * a.n2;
            const long long o = (long long)(r0 + i) * a.ld2 + k;
            const double zv = sc2 * U[i * a.L2 + k + 1].y;
            a.zz[o] = zv;
            if (init) a.p[o] = zv;
            part += a.r[o] * zv;
        }
        __syncthreads();
        return part;
    };

    // the three passes of a CG step (B1 rows, B2 columns, B3 rows; grid barriers between them are the
    // caller's).  B1 returns the partial p.delta.p, B2 the partial p.Bp (Parseval), B3 the partial ||r||^2.
    auto passB1 = [&](int lv, int it, double beta) -> double {
        const long long lo_lv = (long long)min(lv, a.S - 1) * Np;
        // B1: p = zz + beta p (after the first step), row FFT of the embedded p; partial delta p.p
        double pdp = 0.0;
        if (nr > 0) {
            for (int q = tid; q < nr * a.L2; q += nthr) {
                const int i = q >> a.lg2, j = q & (a.L2 - 1);
                double val = 0.0;
                if (j < a.n2) {
                    const long long o = (long long)(r0 + i) * a.ld2 + j;
                    val = a.p[o];
                    if (it > 0) {
                        val = a.zz[o] + beta * val;
                        a.p[o] = val;
                    }
                    if (lv < a.S) pdp += a.e0 * a.D1[lo_lv + o] * a.d2inv[lo_lv + o] * val * val;
                }
                u[q] = make_double2(val, 0.0);
            }
            __syncthreads();
            const double2* U = fft4_smem(u, v, nr, a.L2, a.lg2, tws2, false, tid, nthr);
            double2* Xr = a.X + (long long)r0 * a.L2;
            for (int q = tid; q < nr * a.L2; q += nthr) Xr[q] = U[q];
            __syncthreads();
        }
        return pdp;
    };
    auto passB2 = [&]() -> double {
        // B2: column FFT, times the circulant spectrum, inverse column FFT.  By Parseval the
        // spectrum also gives p.Bp = sum lam |P^|^2 / (L1 L2), so p.Ap = c p.Bp + p.delta.p is
        // known here and the inverse row pass can update x and r at once.
        double pbp = 0.0;
        for (int g = cta; g < a.L2 / cbf; g += G) {
            const int k0 = g * cbf;
            // element q = (row j, column cc) with the column fastest: cbf adjacent values per row
            double lamv[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const int q = tid + t * nthr;
                const int cc = q & (cbf - 1), j = q >> lgc;
                if (q < cbf * a.L1) {
                    u[cc * a.L1 + j] = a.X[(long long)j * a.L2 + k0 + cc];
                    lamv[t] = a.lamB[(long long)j * a.L2 + k0 + cc];
                }
            }
            __syncthreads();
            double2* U = fft4_smem(u, v, cbf, a.L1, a.lg1, tws1, false, tid, nthr);
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const int q = tid + t * nthr;
                const int cc = q & (cbf - 1), j = q >> lgc;
                if (q < cbf * a.L1) {
                    const double2 w = U[cc * a.L1 + j];
                    pbp += lamv[t] * (w.x * w.x + w.y * w.y);
                    U[cc * a.L1 + j] = make_double2(w.x * lamv[t], w.y * lamv[t]);
                }
            }
            __syncthreads();
            double2* W = U == u ? v : u;
            const double2* Y = fft4_smem(U, W, cbf, a.L1, a.lg1, tws1, true, tid, nthr);
            for (int q = tid; q < cbf * a.n1; q += nthr) {
                const int cc = q & (cbf - 1), j = q >> lgc;
                a.X[(long long)j * a.L2 + k0 + cc] = Y[cc * a.L1 + j];
            }
            __syncthreads();
        }
        return pbp;
    };
    auto passB3 = [&](int lv, double c, double alpha, double* x) -> double {
        const long long lo_lv = (long long)min(lv, a.S - 1) * Np;
        double part;
        // B3: inverse row FFT, Ap = c B p + delta o p; x += alpha p, r -= alpha Ap, ||r||^2, and
        // the DST rows of the new r (first pass of the next tau solve)
        part = 0.0;
        if (nr > 0) {
            const double2* Xr = a.X + (long long)r0 * a.L2;
            for (int q = tid; q < nr * a.L2; q += nthr) u[q] = Xr[q];
            __syncthreads();
            const double2* Y = fft4_smem(u, v, nr, a.L2, a.lg2, tws2, true, tid, nthr);
            for (int q = tid; q < nr * a.n2; q += nthr) {
                const int i = q / a.n2, j = q - i * a.n2;
                const long long o = (long long)(r0 + i) * a.ld2 + j;
                const double pv = a.p[o];
                const double delta = lv < a.S ? a.e0 * a.D1[lo_lv + o] * a.d2inv[lo_lv + o] : 0.0;
                const double ap = c * (Y[i * a.L2 + j].x * a.inv_LL) + delta * pv;
                x[o] += alpha * pv;
                const double rv = a.r[o] - alpha * ap;
                a.r[o] = rv;
                part += rv * rv;
            }
            __syncthreads();
            dst_rows(a.r, a.ld2);
        }
        return part;
    };

    // a guess worse than zero (||b - M x0|| > ||b||: the input is not smooth in time) switches the
    // warm start off for the rest of the apply (the decision is grid-uniform: it uses reduced values)
    bool warm_ok = true;
    for (int lv = 0; lv < a.levels; ++lv) {
        // ---- level setup: rhs (forward substitution, krylov.cpp:55-68), b = rhs / D2, x = 0
        const bool direct = lv < a.S && a.direct[lv];
        // warm start: time levels after the first whose predecessors were solved by CG
        const int kx = min(lv, kWarmOrder);  // previous levels in the extrapolation
        bool warm = a.warm && warm_ok && lv >= 1 && lv < a.S && !direct;
        for (int j = 1; j <= kx; ++j) warm = warm && !a.direct[lv - j];
        double* x = a.y + (long long)lv * Np;
        double part = 0.0;
        for (long long i = (long long)cta * nthr + tid; i < Np; i += (long long)G * nthr) {
            const int i2 = (int)(i % a.ld2);
            double b = 0.0, xv = 0.0;
            if (i2 < a.n2) {
                if (lv < a.S) {
                    // L1 history sum_{m < lv} e_{lv-m} y_m, blocked over 8 levels: at a block start
                    // B0 the old part sum_{m < B0} e_{L-m} y_m of the block's 8 targets L is formed
                    // reading each y_m once (8x less traffic than per level; this thread owns element
                    // i at every level, so hb needs no synchronisation); per level the <= 7 recent
                    // terms m in [B0, lv) are added
                    const int B0 = lv & ~7, jt = lv & 7;
                    if (jt == 0 && B0 > 0) {
                        double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                        const int nt = min(8, a.S - B0);
                        for (int m = 0; m < B0; ++m) {
                            const double ym = a.y[(long long)m * Np + i];
#pragma unroll
                            for (int t = 0; t < 8; ++t)
                                if (t < nt) acc[t] += a.e[B0 + t - m] * ym;
                        }
#pragma unroll
                        for (int t = 0; t < 8; ++t) a.hb[(long long)t * Np + i] = acc[t];
                    }
                    double hist = B0 > 0 ? a.hb[(long long)jt * Np + i] : 0.0;
                    for (int m = B0; m < lv; ++m) hist += a.e[lv - m] * a.y[(long long)m * Np + i];
                    const long long o = (long long)lv * Np + i;
                    const double rhs = a.z_in[o] - a.D1[o] * hist;
                    if (direct) xv = rhs / (a.e0 * a.D1[o]);
                    else b = rhs * a.d2inv[o];
                } else {
                    const double rhs = a.z_in[(long long)a.S * Np + i] - a.y[(long long)(a.S - 1) * Np + i];
                    b = rhs * a.d2inv[(long long)(a.S - 1) * Np + i];
                }
            }
            // initial guess of the time levels (not the f-block): the polynomial extrapolation through
            // the previous kx levels' solutions, x0 = sum_j (-1)^(j+1) C(kx, j) y_(lv-j), passed
            // through p to the pre-step
            double x0 = 0.0;
            if (warm && i2 < a.n2)
                for (int j = 1; j <= kx; ++j) x0 += kWarmCoef[kx][j] * a.y[(long long)(lv - j) * Np + i];
            a.r[i] = b;
            a.zz[i] = b;
            a.p[i] = x0;
            x[i] = xv;
            part += b * b;
        }
        stamp(7);
        const double bn2 = greduce(part);
        stamp(0);
        const bool conv = bn2 == 0.0 || direct;
        if (conv) continue;
        const double c = level_c(a, lv);
        const long long lo_lv = (long long)min(lv, a.S - 1) * Np;  // D1, 1/D2 rows of the level
        bool from_zero = true;
        if (warm) {
            // pre-step with alpha = 1 along p = x0: x = x0, r = b - M x0 (and the DST rows of r)
            passB1(lv, 0, 0.0);
            gsync();
            passB2();
            gsync();
            const double rn0 = greduce(passB3(lv, c, 1.0, x));
            if (sqrt(rn0) <= a.tol * sqrt(bn2)) continue;  // the guess already solves the level
            from_zero = rn0 > bn2;  // a guess worse than 0: restart from x = 0, r = b
            if (from_zero) {
                warm_ok = false;
                for (long long i = (long long)cta * nthr + tid; i < Np; i += (long long)G * nthr) {
                    a.r[i] = a.zz[i];
                    x[i] = 0.0;
                }
                gsync();
            }
        }
        // ---- initial tau solve: zz = tau^{-1} r, p = zz, rz = r.zz
        if (from_zero) dst_rows(a.r, a.ld2);
        gsync();
        tau_cols_phase(lv);
        gsync();
        double rz = greduce(tau_out_phase(true));
        stamp(1);
        double beta = 0.0;
        int it = 0;
        while (true) {
            const double pdp = passB1(lv, it, beta);
            gsync();
            stamp(2);
            const double pbp = passB2();
            const double alpha = rz / greduce(c * a.inv_LL * pbp + pdp);
            stamp(3);
            part = passB3(lv, c, alpha, x);
            stamp(4);
            const double rn2 = greduce(part);
            stamp(5);
            ++it;
            if (sqrt(rn2) <= a.tol * sqrt(bn2) || it >= a.maxit) break;
            tau_cols_phase(lv);
            gsync();
            stamp(6);
            const double rz_new = greduce(tau_out_phase(false));
            stamp(7);
            beta = rz_new / rz;
            rz = rz_new;
        }
    }
}

int ilog2(int v) {
    int l = 0;
    while ((1 << l) < v) ++l;
    return l;
}

// column kernels stage 2 x CB x L1 complex values (64 KiB at L1 = 512): above the 48 KiB default
void allow_column_smem() {
    static bool done = false;
    if (done) return;
    const int bytes = 2 * CB * 1024 * (int)sizeof(double2);
    FI_CUDA(cudaFuncSetAttribute(fft_cols_to_spec, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done = true;
}

ItArgs make_args(fi_precond* P) {
    const fi_system* sys = P->sys;
    const Layout& L = sys->L;
    const long long Np = L.Np;
    ItArgs a{};
    a.n1 = L.n1;
    a.n2 = L.n2;
    a.ld2 = L.ld2;
    a.L1 = P->it_L1;
    a.L2 = P->it_L2;
    a.lg1 = ilog2(a.L1);
    a.lg2 = ilog2(a.L2);
    a.S = L.S;
    a.maxit = P->it_maxit;
    a.Np = Np;
    a.tol = P->it_tol;
    a.cs = sys->cs;
    a.cr = sys->cr;
    a.e0 = sys->e_h[0];
    a.inv_LL = 1.0 / ((double)a.L1 * a.L2);
    a.tw1 = P->it_tw1.p;
    a.tw2 = P->it_tw2.p;
    a.lamB = P->it_lamB.p;
    a.lamT = P->it_lamT.p;
    a.dmean = P->it_dmean_d.p;
    a.direct = P->it_direct_d.p;
    a.D1 = sys->D1.p;
    a.d2inv = P->d2inv.p;
    a.e = sys->e.p;
    a.r = P->it_vec.p;
    a.zz = P->it_vec.p + Np;
    a.p = P->it_vec.p + 2 * Np;
    a.Ap = P->it_vec.p + 3 * Np;
    a.X = P->it_X.p;
    a.hb = P->it_hb.p;
    static const int warm = std::getenv("FI_TAU_WARM") ? std::atoi(std::getenv("FI_TAU_WARM")) : 1;
    a.warm = warm;
    a.Rr = P->it_Rr.p;
    return a;
}

}  // namespace

bool iterative_supported(const Layout& L) {
    if (L.d != 2) return false;
    const int a = L.n1 + 1, b = L.n2 + 1;
    return (a & (a - 1)) == 0 && (b & (b - 1)) == 0 && 2 * a <= 1024 && 2 * b <= 1024;
}

void precond_build_iterative(fi_precond* P, double tol, int maxit) {
    fi_system* sys = P->sys;
    fi_ctx* ctx = sys->ctx;
    const Layout& L = sys->L;
    const int S = L.S;
    const long long N = L.N, Np = L.Np;
    if (!iterative_supported(L))
        throw Error(FI_E_RESOURCE, "precond_build: 2D block of " + std::to_string(N) +
                                       " unknowns needs n_i + 1 a power of two (<= 512) for the tau-PCG solve");
    const double e0 = sys->e_h[0];
    // admissibility (as the dense path) and per-level mean(delta)
    std::vector<double> d2inv((size_t)S * Np, 0.0), dmean((size_t)S + 1, 0.0);
    std::vector<int> direct((size_t)S + 1, 0);
    for (int s = 1; s <= S; ++s) {
        bool all_zero = true;
        for (long long j = 0; j < N; ++j) all_zero = all_zero && sys->D2_h[(size_t)(s - 1) * N + j] == 0.0;
        double acc = 0.0;
        for (long long j = 0; j < N; ++j) {
            const double d1 = sys->D1_h[(size_t)(s - 1) * N + j], d2 = sys->D2_h[(size_t)(s - 1) * N + j];
            const long long pidx = (long long)(s - 1) * Np + (j / L.n2) * L.ld2 + j % L.n2;
            if (all_zero) {
                if (d1 == 0.0 || e0 == 0.0)
                    throw Error(FI_E_SINGULAR, "precond_build: singular block at time level " + std::to_string(s), s);
                continue;
            }
            if (d2 == 0.0) {
                if (d1 == 0.0 || e0 == 0.0)
                    throw Error(FI_E_SINGULAR, "precond_build: singular block at time level " + std::to_string(s), s);
                throw Error(FI_E_DOMAIN, "precond_build: gamma2 vanishes at part of level " + std::to_string(s));
            }
            if (d1 / d2 < 0.0)
                throw Error(FI_E_DOMAIN, "precond_build: gamma1/gamma2 < 0 at level " + std::to_string(s));
            d2inv[(size_t)pidx] = 1.0 / d2;
            acc += e0 * d1 / d2;
        }
        direct[(size_t)s - 1] = all_zero ? 1 : 0;
        dmean[(size_t)s - 1] = acc / (double)N;
    }
    for (long long j = 0; j < N; ++j)
        if (sys->D2_h[(size_t)(S - 1) * N + j] == 0.0)
            throw Error(FI_E_SINGULAR, "precond_build: singular block at time level " + std::to_string(S + 1), S + 1);
    P->it_direct = direct;
    P->it_dmean = dmean;
    P->it_tol = tol;
    P->it_maxit = maxit;
    P->mode = 1;
    P->refine = 0;
    P->levels = S + 1;
    P->it_L1 = 2 * (L.n1 + 1);
    P->it_L2 = 2 * (L.n2 + 1);
    const int L1 = P->it_L1, L2 = P->it_L2;
    P->d2inv.alloc((size_t)S * Np);
    FI_CUDA(cudaMemcpy(P->d2inv.p, d2inv.data(), d2inv.size() * sizeof(double), cudaMemcpyHostToDevice));
    P->it_dmean_d.alloc(dmean.size());
    FI_CUDA(cudaMemcpy(P->it_dmean_d.p, dmean.data(), dmean.size() * sizeof(double), cudaMemcpyHostToDevice));
    P->it_direct_d.alloc(direct.size());
    FI_CUDA(cudaMemcpy(P->it_direct_d.p, direct.data(), direct.size() * sizeof(int), cudaMemcpyHostToDevice));
    // twiddles exp(-2 pi i k / L)
    std::vector<double2> t1((size_t)L1 / 2), t2((size_t)L2 / 2);
    for (int k = 0; k < L1 / 2; ++k)
        t1[(size_t)k] = make_double2(std::cos(2.0 * M_PI * k / L1), -std::sin(2.0 * M_PI * k / L1));
    for (int k = 0; k < L2 / 2; ++k)
        t2[(size_t)k] = make_double2(std::cos(2.0 * M_PI * k / L2), -std::sin(2.0 * M_PI * k / L2));
    P->it_tw1.alloc(t1.size());
    P->it_tw2.alloc(t2.size());
    FI_CUDA(cudaMemcpy(P->it_tw1.p, t1.data(), t1.size() * sizeof(double2), cudaMemcpyHostToDevice));
    FI_CUDA(cudaMemcpy(P->it_tw2.p, t2.data(), t2.size() * sizeof(double2), cudaMemcpyHostToDevice));
    // tau eigenvalues g(theta_j1, theta_j2) = (4 sin^2(theta_1/2) + 4 sin^2(theta_2/2))^{omega/2}
    const double omega_half = sys->omega / 2.0;
    std::vector<double> lamT((size_t)N);
    for (int j1 = 1; j1 <= L.n1; ++j1)
        for (int j2 = 1; j2 <= L.n2; ++j2) {
            const double s1 = std::sin(j1 * M_PI / (L.n1 + 1) / 2.0), s2 = std::sin(j2 * M_PI / (L.n2 + 1) / 2.0);
            lamT[(size_t)(j1 - 1) * L.n2 + (j2 - 1)] = std::pow(4.0 * s1 * s1 + 4.0 * s2 * s2, omega_half);
        }
    P->it_lamT.alloc(lamT.size());
    FI_CUDA(cudaMemcpy(P->it_lamT.p, lamT.data(), lamT.size() * sizeof(double), cudaMemcpyHostToDevice));
    P->it_X.alloc((size_t)L1 * L2);
    P->it_Rr.alloc((size_t)N);
    P->it_lamB.alloc((size_t)L1 * L2);
    P->it_vec.alloc((size_t)4 * Np);  // r, z, p, Ap
    P->it_hb.alloc((size_t)8 * Np);   // blocked L1 history
    FI_CUDA(cudaMemset(P->it_vec.p, 0, P->it_vec.bytes()));
    // circulant spectrum of B with the same FFT kernels
    allow_column_smem();
    ItArgs a = make_args(P);
    spec_embed<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(a, sys->gen.p, 2 * L.ld2 + 8);
    FI_LAUNCHED(ctx);
    fft_rows_plain<<<L1, std::min(L2 / 2, 256), 2 * L2 * sizeof(double2), ctx->stream>>>(a);
    FI_LAUNCHED(ctx);
    fft_cols_to_spec<<<L2 / CB, 256, 2 * CB * L1 * sizeof(double2), ctx->stream>>>(a, P->it_lamB.p);
    FI_LAUNCHED(ctx);
    FI_CUDA(cudaStreamSynchronize(ctx->stream));
}

void precond_apply_iterative(fi_ctx* ctx, fi_precond* P, const double* z, double* y, int levels, const int* skip) {
    {
        // one cooperative kernel for the whole substitution (tau_pcg_fused)
        ItArgs a = make_args(P);
        a.z_in = z;
        a.y = y;
        a.levels = levels;
        a.skip = skip;
        // grid: one row (pair of columns) per CTA when the GPU holds that many CTAs (two per SM),
        // otherwise each CTA transforms rpc rows / cbf columns at once; every pass is one round
        if (P->it_fgrid == 0) {
            const size_t smem_max = (2 * (size_t)std::max(4 * a.L2, 4 * a.L1) + a.L1 / 2 + a.L2 / 2) * sizeof(double2);
            FI_CUDA(cudaFuncSetAttribute(tau_pcg_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::min<size_t>(smem_max, 227 * 1024)));
            const size_t smem1 = (2 * (size_t)std::max(a.L2, 2 * a.L1) + a.L1 / 2 + a.L2 / 2) * sizeof(double2);
            int per_sm = 0;
            FI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tau_pcg_fused, 256, smem1));
            if (per_sm < 1) throw Error(FI_E_CUDA, "tau_pcg_fused cannot be resident");
            P->it_fgrid = std::min(ctx->sm_count * std::min(per_sm, 2), std::max(a.n1, (a.L2 + 1) / 2));
            P->it_fparts.alloc((size_t)2 * P->it_fgrid);
            P->it_fbar.alloc(1);
        }
        const int G = P->it_fgrid;
        const int rpc = (a.n1 + G - 1) / G;
        int cbf = 1;
        while (cbf * G < a.L2 && cbf * 2 * a.L1 <= 8 * 256) cbf *= 2;
        const size_t hs = (size_t)std::max(rpc * a.L2, cbf * a.L1);
        const size_t smem = (2 * hs + a.L1 / 2 + a.L2 / 2) * sizeof(double2);
        if (smem > 227 * 1024) throw Error(FI_E_RESOURCE, "tau_pcg_fused: shared memory");
        static const bool tracing = std::getenv("FI_ITER_TRACE") != nullptr;
        DevBuf<unsigned long long> trace;
        if (tracing) {
            trace.alloc(10);
            FI_CUDA(cudaMemsetAsync(trace.p, 0, trace.bytes(), ctx->stream));
        }
        int lgc = 0;
        while ((1 << lgc) < cbf) ++lgc;
        int cbt = 1, lgt = 0;  // tau column pass: n2 columns over the grid
        while (cbt * G < a.n2 && cbt < cbf) {
            cbt *= 2;
            ++lgt;
        }
        FusedCtl ctl{P->it_fbar.p, P->it_fparts.p, tracing ? trace.p : nullptr, rpc, cbf, lgc, cbt, lgt};
        FI_CUDA(cudaMemsetAsync(P->it_fbar.p, 0, sizeof(unsigned), ctx->stream));
        void* args[] = {&a, &ctl};
        FI_CUDA(cudaLaunchCooperativeKernel((const void*)tau_pcg_fused, dim3(P->it_fgrid), dim3(256), args, smem,
                                            ctx->stream));
        FI_LAUNCHED(ctx);
        if (tracing) {
            unsigned long long h[10];
            FI_CUDA(cudaMemcpyAsync(h, trace.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
            FI_CUDA(cudaStreamSynchronize(ctx->stream));
            std::fprintf(stderr,
                         "[tau_pcg_fused] ms: setup %.3f | tau0 %.3f | B1 %.3f | B2 %.3f | B3+red %.3f | U+T1+red %.3f | "
                         "T2 %.3f | T3+red %.3f | barrier wait (CTA 0) %.3f over %llu barriers\n",
                         h[0] * 1e-6, h[1] * 1e-6, h[2] * 1e-6, h[3] * 1e-6, h[4] * 1e-6, h[5] * 1e-6, h[6] * 1e-6,
                         h[7] * 1e-6, h[8] * 1e-6, h[9]);
        }
    }
}

}  // namespace fib

fi_precond::~fi_precond() { fib::hodlr_destroy(hodlr); }
