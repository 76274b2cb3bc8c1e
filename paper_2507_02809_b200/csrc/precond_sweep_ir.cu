// K2 — P^{-1} z: forward block substitution AND its iterative refinement in ONE persistent kernel.
//
// P^{-1} z with LU-grade accuracy needs one refinement step on top of the explicit-inverse sweep
// (DESIGN §6):  y1 = P~^{-1} z (FP64 inverses),  r = z - P y1 (exact FP64 residual),
// d = P~^{-1} r (FP32 inverses),  y = y1 + d.  Run as separate kernels that is two sequential
// S-level dependency chains plus an operator launch.  Here they are interleaved with a lag:
//   step t:  tiles of H64_t x1_t          (chain 1: sweep 1, level t)
//            tiles of B y1_{t-1}          (chain 2: residual of level t-1, B generated from its symbol)
//            tiles of H32_{t-2} x2_{t-2}  (chain 2: sweep 2, level t-2)
// and the chains are decoupled: each has its own owner phase and its own per-row-block release
// counter, run by dedicated warps, so the ring warps never sit in an owner phase — while chain 1's
// owners publish x1_{t+1}, the ring streams the FP32 tiles of step t, and while chain 2's owners
// publish x2_{t-1}, it streams the FP64 tiles of step t+1.
// Warps (12, 168 registers): a producer (cp.async.bulk / TMA into an mbarrier ring of half-tile
// slots, evict-first in L2), 6 ring warps (FP64 and FP32 tile products), 3 owner warps (both
// chains' reductions, the x vectors, the L1 history sums) and 2 B-tile warps.  Dataflow: warp-uniform
// relaxed polls on per-row-block counters, one release fence per warp and phase, fixed-order
// (bit-reproducible) reductions, bounded spins.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "precond.cuh"

namespace fib {
namespace {

constexpr int TB = 64;
constexpr int TILE = TB * TB;
constexpr int NW = 11;                  // worker warps; + 1 producer = 12 warps (3 per SMSP)
constexpr int THREADS = NW * 32 + 32;
constexpr int NST = 6;                  // ring warps (tile item k -> warp k % NST)
constexpr int NHS = 2 * NST;            // ring half-slots of 16 KiB: a tile streams as two row halves
constexpr int HSLOT = TILE / 2;         // doubles per half-slot
constexpr int RCAP = 32;   // owned rows per CTA: one per lane
constexpr int CSTR = kCounterStride;
constexpr int TCAP = 64;   // tiles per CTA and level (coordinate table)

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// streaming variant: the tiles are read once, so they are marked evict-first in L2 and do not push
// out the sweep's small, re-read working set (x, partial products, history rows)
__device__ __forceinline__ void tma_bulk_g2s_stream(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                                    uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_relaxed(unsigned* p, unsigned v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// warp-uniform poll (all 32 lanes): the warp never diverges, so later shfl.sync stay cheap
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Poll relaxed (an acquire load invalidates the SM's L1 on every iteration, evicting the symbol and
// weight lines other warps read through L1), then one acquire load once the counter has moved.
// Spin bound: a dataflow wait that exceeds ~seconds is a bug; trap instead of hanging the GPU.
constexpr unsigned kSpinLimit = 1u << 25;
__device__ __forceinline__ void warp_spin_until(const unsigned* p, unsigned target) {
    for (unsigned n = 0; !__all_sync(0xffffffffu, ld_relaxed(p) >= target); ++n) {
        __nanosleep(64);
        if (n == kSpinLimit) __trap();
    }
    (void)ld_acquire(p);
}
__device__ __forceinline__ void tile_coords(long long t, int& bi, int& bj) {
    int r = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while ((long long)(r + 1) * (r + 2) / 2 <= t) ++r;
    while ((long long)r * (r + 1) / 2 > t) --r;
    bi = r;
    bj = (int)(t - (long long)r * (r + 1) / 2);
}
__device__ __forceinline__ int owners_of_block(int rb, long long R, unsigned G) {
    const long long first = (long long)rb * TB / R;
    const long long last = min((long long)G - 1, ((long long)rb * TB + TB - 1) / R);
    return (int)(last - first + 1);
}

struct IrArgs {
    const double* H64;
    const float* H32;
    long long T;
    int nb, nlev, S, n1, n2, ld2, gen_stride;
    long long Np;
    const double* z;
    double* y;    // output y1 + d
    double* Y1;   // sweep-1 result, all levels
    float* DLf;   // sweep-2 correction, all levels (FP32 copy: only its history sums read it)
    const double* D1;
    const double* D2;
    const double* d2inv;
    const double* e;
    const double* gen;
    const double* epad;  // e with zero padding: epad[k] = e_k for 0 <= k < S
    double cs, cr;
    double* xb;   // [3 kinds][2 parities][Np]
    double* pb;   // [3 kinds][2 parities][nb][nb][TB]
    unsigned* xready;  // [nb] (stride CSTR); version 2: chain-1 counters
    unsigned* xready2;  // version 2: chain-2 counters [nb]
    unsigned* pdone;   // [3][nb] (stride CSTR); kind 1 (B tiles) counts the even steps only
    unsigned* pdone1b;  // [nb]: B tiles of the odd steps.  The B tiles run up to one step ahead of
                        // their consumer (owner2), so one cumulative counter could reach step t-1's
                        // target with step-t bumps; split by step parity, a counter cannot run ahead
    const int* skip;
    int evict_first;
    unsigned long long* trace;  // optional [G][nsteps+1][8] phase timestamps (FI_SWEEP_TRACE=1)
};

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Symmetric tile product for one warp: rowsums (H x_j) -> prow[0..63], colsums (H^T x_i) -> pcol.
// hrow(half, q) fetches row 32 half + q as the lane's two columns (2 lane, 2 lane + 1); begin(half) /
// end(half) bracket the rows of a half (ring-slot wait / release: a half-slot is freed as soon as its
// rows are read, before the reduction).
template <class Begin, class RowFn, class End>
__device__ __forceinline__ void tile_product(Begin begin, RowFn hrow, End end, double2 xj, const double* xi,
                                             double* prow, double* pcol, bool diag, int lane) {
    double c0 = 0.0, c1 = 0.0;
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {  // not unrolled: keeps the kernel inside the instruction cache
        double pr[32];
        begin(half);
#pragma unroll
        for (int q = 0; q < 32; ++q) {
            const double2 hv = hrow(half, q);
            pr[q] = hv.x * xj.x + hv.y * xj.y;
            const double xr = xi[half * 32 + q];
            c0 += hv.x * xr;
            c1 += hv.y * xr;
        }
        end(half);
#pragma unroll
        for (int w = 16; w >= 1; w >>= 1) {
            const bool upper = (lane & w) != 0;
#pragma unroll
            for (int i = 0; i < w; ++i) {
                const double send = upper ? pr[i] : pr[i + w];
                const double keep = upper ? pr[i + w] : pr[i];
                pr[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
            }
        }
        prow[half * 32 + lane] = pr[0];
    }
    if (!diag) reinterpret_cast<double2*>(pcol)[lane] = make_double2(c0, c1);
}

// FP32 variant for the refinement sweep (H32 tiles): the correction d ~ 1e-12 |y| needs only a few
// significant digits, so the products and sums run in FP32 (no F64<->F32 conversions per element,
// 32-bit shuffles); the partial products are stored in FP64 for the owner's reduction.
template <class Begin, class RowFn, class End>
__device__ __forceinline__ void tile_product_f32(Begin begin, RowFn hrow, End end, float2 xj, const float* xi,
                                                 double* prow, double* pcol, bool diag, int lane) {
    float c0 = 0.f, c1 = 0.f;
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
        float pr[32];
        begin(half);
#pragma unroll
        for (int q = 0; q < 32; ++q) {
            const float2 hv = hrow(half, q);
            pr[q] = fmaf(hv.x, xj.x, hv.y * xj.y);
            const float xr = xi[half * 32 + q];
            c0 = fmaf(hv.x, xr, c0);
            c1 = fmaf(hv.y, xr, c1);
        }
        end(half);
#pragma unroll
        for (int w = 16; w >= 1; w >>= 1) {
            const bool upper = (lane & w) != 0;
#pragma unroll
            for (int i = 0; i < w; ++i) {
                const float send = upper ? pr[i] : pr[i + w];
                const float keep = upper ? pr[i + w] : pr[i];
                pr[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
            }
        }
        prow[half * 32 + lane] = (double)pr[0];
    }
    if (!diag) reinterpret_cast<double2*>(pcol)[lane] = make_double2((double)c0, (double)c1);
}

// Per step, ring warps in FIFO order: FP64 tiles of level t (gate: chain-1 counter, partials kind 0,
// one release fence), FP32 tiles of level t-2 (gate: chain-2 counter, kind 2).  B-tile warps: B tiles
// of level t-1 (gate: chain-1 counter, kind 1).  Owner warps: owner1(t) (y1_{t-1}, x1_t), history of
// chain 1, owner2(t) (d_{t-3}, y = y1 + d, x2_{t-2}), history of chain 2.  The residual
// r_l = z_l - P y1 reuses the numerator w_l = z_l - D1_l o hist1_l of x1_l (kept in shared memory),
// so chain 2 needs no history of y1.
constexpr int NR = NST;        // ring warps
constexpr int NS = NW - NST;   // spare warps: NSO owner warps (owners + history), NS - NSO B-tile warps
constexpr int NSO = 3;
constexpr int KPS = 24;        // partials per owner warp and kind: nb <= KPS * NSO
__device__ __forceinline__ void spare_bar() { asm volatile("bar.sync 2, %0;\n" ::"n"(NSO * 32) : "memory"); }
__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__global__ void __maxnreg__(168) sweep_ir_kernel(IrArgs a) {
    if (a.skip && *a.skip) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* ring = reinterpret_cast<double*>(smem_raw);  // NHS x HSLOT
    double* red = ring + NHS * HSLOT;                     // 2 x NSO x 32 owner partial sums
    double* hred = red + 2 * NSO * 32;                    // NSO x 64 history partials
    double* h1p = hred + NSO * 64;                        // 32: chain-1 history of the next owner1
    double* h2p = h1p + 32;                               // 32: chain-2 history of the next owner2
    double* wbuf = h2p + 32;                              // 4 x 32: w_l = z_l - D1_l o hist1_l
    double* ybuf = wbuf + 4 * 32;                         // 4 x 32: y1_l of the owned rows
    double* xis = ybuf + 4 * 32;                          // NW x TB staging of x_i
    double* segs = xis + NW * TB;                         // NS x 128 symbol segments (B tiles)
    int* tcs = reinterpret_cast<int*>(segs + NS * 128);   // TCAP packed (bi << 16 | bj)
    uint64_t* full = reinterpret_cast<uint64_t*>(tcs + TCAP);
    uint64_t* empty = full + NHS;

    const unsigned G = gridDim.x;
    const long long t0 = (long long)blockIdx.x * a.T / G;
    const long long t1 = (long long)(blockIdx.x + 1) * a.T / G;
    const long long ntiles = t1 - t0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nlev = a.nlev, S = a.S, nbb = a.nb;
    const long long Np = a.Np;
    const int nsteps = nlev + 2;  // tile steps 0..nlev+1
    const long long kstride = (long long)nbb * nbb * TB;

    for (long long k = threadIdx.x; k < ntiles; k += blockDim.x) {
        int bi, bj;
        tile_coords(t0 + k, bi, bj);
        tcs[k] = (bi << 16) | bj;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < NHS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    auto h64_valid = [&](int t) { return t < nlev; };
    auto b_valid = [&](int t) { return t >= 1 && t - 1 < nlev; };
    auto h32_valid = [&](int t) { return t >= 2 && t - 2 < nlev; };

    if (warp == NW) {
        // ---------------- producer: per step, the FP64 tiles of level t then the FP32 tiles of level t-2
        if (lane == 0) {
            uint64_t policy;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(policy));
            long long it = 0;
            for (int t = 0; t < nsteps; ++t) {
                for (int kind = 0; kind < 2; ++kind) {
                    if (!(kind == 0 ? h64_valid(t) : h32_valid(t))) continue;
                    const int lv = kind == 0 ? t : t - 2;
                    const unsigned hbytes = kind == 0 ? TILE / 2 * sizeof(double) : TILE / 2 * sizeof(float);
                    for (long long k = 0; k < ntiles; ++k, ++it) {
                        const long long tix = (long long)lv * a.T + t0 + k;
                        const char* src = kind == 0 ? (const char*)(a.H64 + tix * TILE) : (const char*)(a.H32 + tix * TILE);
                        for (int h = 0; h < 2; ++h) {
                            const long long j = 2 * it + h;
                            const int slot = (int)(j % NHS);
                            if (j >= NHS) {
                                const unsigned long long tw0 = a.trace ? gtime() : 0;
                                mbar_wait(&empty[slot], (unsigned)((j / NHS - 1) & 1));
                                if (a.trace) a.trace[((long long)blockIdx.x * (nsteps + 1) + t) * 12 + 8] += gtime() - tw0;
                            }
                            mbar_expect_tx(&full[slot], hbytes);
                            if (a.evict_first)
                                tma_bulk_g2s_stream(ring + slot * HSLOT, src + h * hbytes, hbytes, &full[slot], policy);
                            else
                                tma_bulk_g2s(ring + slot * HSLOT, src + h * hbytes, hbytes, &full[slot]);
                        }
                    }
                }
            }
        }
        return;
    }

    const long long R = ((Np + G - 1) / G + 3) / 4 * 4;  // multiple of 4: vector history loads
    const long long r0 = min(Np, (long long)blockIdx.x * R);
    const long long r1 = min(Np, r0 + R);
    const int rb0 = (int)(r0 / TB), rb1 = r1 > r0 ? (int)((r1 - 1) / TB) : rb0 - 1;
    unsigned* xr1 = a.xready;   // chain 1: x1_t and y1_{t-1} published
    unsigned* xr2 = a.xready2;  // chain 2: x2_{t-2} published

    auto trp = [&](int t) -> unsigned long long* {
        return a.trace ? a.trace + ((long long)blockIdx.x * (nsteps + 1) + t) * 12 : nullptr;
    };
    // poll all x blocks a list of items reads (lanes 2c: bi, 2c+1: bj), relaxed, one acquire
    auto poll_items = [&](int nitems, auto coords_of, const unsigned* xr, unsigned tmul) {
        for (int c0 = 0; c0 < nitems; c0 += 16) {
            const int c = c0 + (lane >> 1);
            const unsigned* ctr = nullptr;
            unsigned tgt = 0;
            if (c < nitems) {
                int bi, bj;
                coords_of(c, bi, bj);
                const int blk = (lane & 1) ? bj : bi;
                ctr = xr + blk * CSTR;
                tgt = (unsigned)owners_of_block(blk, R, G) * tmul;
            }
            for (unsigned n = 0; !__all_sync(0xffffffffu, ctr == nullptr || ld_relaxed(ctr) >= tgt); ++n) {
                __nanosleep(64);
                if (n == kSpinLimit) __trap();
            }
            if (ctr) (void)ld_acquire(ctr);
        }
    };
    if (warp < NR) {
        // ================================================= ring warps
        long long it = 0;
        double* xi = xis + warp * TB;
        float* xif = reinterpret_cast<float*>(xi);
        // streamed tiles (FP64: kind 0 / FP32: kind 2) of one step, in ring order
        auto ring_items = [&](int kind, long long base, int t, const unsigned* xr, unsigned tmul) -> int {
            const long long kk0 = ((long long)warp - base % NR + NR) % NR;
            const int nitems = kk0 < ntiles ? (int)((ntiles - kk0 + NR - 1) / NR) : 0;
            auto coords_of = [&](int c, int& bi, int& bj) {
                const int v = tcs[kk0 + (long long)c * NR];
                bi = v >> 16;
                bj = v & 0xffff;
            };
            poll_items(nitems, coords_of, xr, tmul);
            const double* xb = a.xb + (long long)(kind * 2 + (t & 1)) * Np;
            double* pbk = a.pb + (long long)(kind * 2 + (t & 1)) * kstride;
            double2 nxj = make_double2(0.0, 0.0), nxi = nxj;
            auto load_x = [&](int c) {
                int bi, bj;
                coords_of(c, bi, bj);
                nxj = __ldcg(reinterpret_cast<const double2*>(xb + (long long)bj * TB) + lane);
                nxi = __ldcg(reinterpret_cast<const double2*>(xb + (long long)bi * TB) + lane);
            };
            if (nitems > 0) load_x(0);
            for (int c = 0; c < nitems; ++c) {
                const double2 xj = nxj;
                if (kind == 0)
                    reinterpret_cast<double2*>(xi)[lane] = nxi;
                else
                    reinterpret_cast<float2*>(xif)[lane] = make_float2((float)nxi.x, (float)nxi.y);
                if (c + 1 < nitems) load_x(c + 1);
                __syncwarp();
                int bi, bj;
                coords_of(c, bi, bj);
                const long long item = base + kk0 + (long long)c * NR;
                double* prow = pbk + ((long long)bi * nbb + bj) * TB;
                double* pcol = pbk + ((long long)bj * nbb + bi) * TB;
                const int hs0 = (int)((2 * item) % NHS);
                auto begin = [&](int h) {
                    const long long j = 2 * item + h;
                    mbar_wait(&full[j % NHS], (unsigned)((j / NHS) & 1));
                };
                auto end = [&](int h) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[(2 * item + h) % NHS]);
                };
                if (kind == 0) {
                    tile_product(
                        begin,
                        [&](int h, int q) {
                            return reinterpret_cast<const double2*>(ring + (hs0 + h) * HSLOT + q * TB)[lane];
                        },
                        end, xj, xi, prow, pcol, bi == bj, lane);
                } else {
                    const float* ringf = reinterpret_cast<const float*>(ring);
                    tile_product_f32(
                        begin,
                        [&](int h, int q) {
                            return reinterpret_cast<const float2*>(ringf + (hs0 + h) * (2 * HSLOT) + q * TB)[lane];
                        },
                        end, make_float2((float)xj.x, (float)xj.y), xif, prow, pcol, bi == bj, lane);
                }
                __syncwarp();
            }
            return nitems;
        };
        auto bump = [&](int kind, long long kk0, int nitems) {
            for (int c = 0; c < nitems; ++c) {
                const int v = tcs[kk0 + (long long)c * NR];
                const int bi = v >> 16, bj = v & 0xffff;
                red_relaxed(a.pdone + (kind * nbb + bi) * CSTR, 1u);
                if (bi != bj) red_relaxed(a.pdone + (kind * nbb + bj) * CSTR, 1u);
            }
        };
        for (int t = 0; t < nsteps; ++t) {
            const long long base0 = it, base1 = it + (h64_valid(t) ? ntiles : 0);
            unsigned long long* tr = trp(t);
            if (tr && warp == 0 && lane == 0) tr[7] = gtime();
            // (a) FP64 tiles of level t
            if (h64_valid(t)) {
                const int n0 = ring_items(0, base0, t, xr1, (unsigned)(t + 1));
                __syncwarp();
                if (lane == 0 && n0 > 0) {
                    asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
                    bump(0, ((long long)warp - base0 % NR + NR) % NR, n0);
                }
                if (tr && lane == 0) atomicMax(tr + 2, gtime());
            }
            // (c) FP32 tiles of level t-2
            int n2 = 0;
            if (h32_valid(t)) n2 = ring_items(2, base1, t, xr2, (unsigned)(t - 1));
            __syncwarp();
            if (lane == 0 && n2 > 0) {
                asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
                bump(2, ((long long)warp - base1 % NR + NR) % NR, n2);
            }
            if (tr && lane == 0) atomicMax(tr + 4, gtime());
            it += (h64_valid(t) ? ntiles : 0) + (h32_valid(t) ? ntiles : 0);
        }
        return;
    }

    // ================================================= spare warps: owners of both chains + history
    const int sw = warp - NR;
    if (sw >= NSO) {
        // ================================================= B-tile warps
        constexpr int NB2 = NS - NSO;
        const int bw = sw - NSO;
        for (int t = 1; t < nsteps; ++t) {
            // B tiles of the residual of level t-1, generated from the symbol (no HBM traffic): B warp
            // bw takes tiles bw, bw + NB2, ...
            if (b_valid(t)) {
                unsigned long long* tr = trp(t);
                double* xi = xis + warp * TB;
                double* seg = segs + bw * 128;
                const int nbt = bw < ntiles ? (int)((ntiles - bw + NB2 - 1) / NB2) : 0;
                auto coords_of = [&](int c, int& bi, int& bj) {
                    const int v = tcs[bw + (long long)c * NB2];
                    bi = v >> 16;
                    bj = v & 0xffff;
                };
                poll_items(nbt, coords_of, xr1, (unsigned)(t + 1));
                const double* xb = a.xb + (long long)(1 * 2 + (t & 1)) * Np;
                double* pbk = a.pb + (long long)(1 * 2 + (t & 1)) * kstride;
                double2 nxj = make_double2(0.0, 0.0), nxi = nxj;
                double ng[4];
                auto load_b = [&](int c) {
                    int bi, bj;
                    coords_of(c, bi, bj);
                    const long long i0 = (long long)bi * TB, j0 = (long long)bj * TB;
                    const int i1 = (int)(i0 / a.ld2), i2 = (int)(i0 % a.ld2);
                    const int j1 = (int)(j0 / a.ld2), j2 = (int)(j0 % a.ld2);
                    const double* g = a.gen + (long long)(i1 - j1 + a.n1 - 1) * a.gen_stride + a.ld2 + i2 - j2 - 63;
#pragma unroll
                    for (int u = 0; u < 4; ++u) ng[u] = (lane + 32 * u < 127) ? __ldg(g + lane + 32 * u) : 0.0;
                    nxj = __ldcg(reinterpret_cast<const double2*>(xb + j0) + lane);
                    nxi = __ldcg(reinterpret_cast<const double2*>(xb + i0) + lane);
                };
                if (nbt > 0) load_b(0);
                for (int c = 0; c < nbt; ++c) {
                    const double2 xj = nxj;
                    reinterpret_cast<double2*>(xi)[lane] = nxi;
#pragma unroll
                    for (int u = 0; u < 4; ++u) seg[lane + 32 * u] = ng[u];
                    if (c + 1 < nbt) load_b(c + 1);
                    __syncwarp();
                    int bi, bj;
                    coords_of(c, bi, bj);
                    // pad columns meet zero entries of x; pad rows are zeroed by the owner
                    tile_product([](int) {},
                                 [&](int h, int q) {
                                     const int rr2 = h * 32 + q;
                                     return make_double2(seg[rr2 - 2 * lane + 63], seg[rr2 - 2 * lane + 62]);
                                 },
                                 [](int) {}, xj, xi, pbk + ((long long)bi * nbb + bj) * TB,
                                 pbk + ((long long)bj * nbb + bi) * TB, bi == bj, lane);
                    __syncwarp();
                }
                if (lane == 0 && nbt > 0) {
                    asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
                    unsigned* pc = (t & 1) ? a.pdone1b : a.pdone + nbb * CSTR;
                    for (int c = 0; c < nbt; ++c) {
                        int bi, bj;
                        coords_of(c, bi, bj);
                        red_relaxed(pc + bi * CSTR, 1u);
                        if (bi != bj) red_relaxed(pc + bj * CSTR, 1u);
                    }
                }
                if (tr && lane == 0) atomicMax(tr + 3, gtime());
            }
        }
        return;
    }
    const long long r = r0 + lane;
    const bool rvalid = r < r1;
    const long long rr = rvalid ? r : (r1 > r0 ? r0 : 0);  // clamped in-range row for inactive lanes
    const bool pad = (int)(rr % a.ld2) >= a.n2;
    const long long rb_own = rr / TB, ro_own = rr % TB;
    const int nrb = rb1 - rb0 + 1;
    const double e1 = a.epad[1];
    // polls of the partial-product counters of this CTA's row blocks, spread over the spare warps
    auto poll_pdone = [&](int kind, unsigned target) {
        for (int q = sw; q < nrb; q += NSO) warp_spin_until(a.pdone + (kind * nbb + rb0 + q) * CSTR, target);
    };
    // B tiles of step s (1 <= s) done for the CTA's row blocks: the parity counter of s has seen all
    // (s + 1) / 2 of its steps up to s
    auto poll_bstep = [&](int s) {
        const unsigned* pc = (s & 1) ? a.pdone1b : a.pdone + nbb * CSTR;
        for (int q = sw; q < nrb; q += NSO) warp_spin_until(pc + (rb0 + q) * CSTR, (unsigned)(nbb * ((s + 1) / 2)));
    };
    // fixed-order sum of the nb partials of `kind` (parity par) for the owned rows -> red[slot]
    auto load_partials = [&](int kind, int par, int slot) {
        const double* pbk = a.pb + (long long)(kind * 2 + par) * kstride + rb_own * nbb * TB + ro_own;
        double pv[KPS];
#pragma unroll
        for (int u = 0; u < KPS; ++u) {
            const int k = sw + u * NSO;
            pv[u] = k < nbb ? __ldcg(pbk + (long long)k * TB) : 0.0;
        }
        double s0 = 0.0;
#pragma unroll
        for (int u = 0; u < KPS; ++u) s0 += pv[u];
        red[(slot * NSO + sw) * 32 + lane] = s0;
    };
    auto sum_partials = [&](int slot) {
        double v = 0.0;
        for (int w = 0; w < NSO; ++w) v += red[(slot * NSO + w) * 32 + lane];
        return pad ? 0.0 : v;
    };
    auto release_rows = [&](unsigned* xr) {
        __syncwarp();
        if (lane == 0)
            for (int rb = rb0; rb <= rb1; ++rb) red_release(xr + rb * CSTR, 1u);
    };

    for (int t = 0; t <= nlev + 2; ++t) {
        // ---------------- owner1(t): y1_{t-1}, x1_t (and the B-tile input y1_{t-1})
        if (t <= nlev) {
            double c_z = 0, c_d1 = 0, c_di = 0, c_h = 0;
            if (sw == 0 && t < nlev) {
                if (t < S) {
                    const long long o = (long long)t * Np + rr;
                    c_z = a.z[o];
                    c_d1 = a.D1[o];
                    c_di = a.d2inv[o];
                } else {
                    c_z = a.z[(long long)S * Np + rr];
                    c_di = a.d2inv[(long long)(S - 1) * Np + rr];
                }
            }
            double v0 = 0.0;
            if (t >= 1) {
                poll_pdone(0, (unsigned)(nbb * min(t, nlev)));
                // xb1[t & 1] is rewritten below: the B tiles of step t-2 that read it are done
                if (t >= 3) poll_bstep(t - 2);
                spare_bar();
                if (sw == 0) c_h = h1p[lane];
                load_partials(0, (t - 1) & 1, 0);
                spare_bar();
                if (sw == 0) {
                    v0 = sum_partials(0);
                    if (rvalid) {
                        a.Y1[(long long)(t - 1) * Np + r] = v0;
                        a.xb[(long long)(1 * 2 + (t & 1)) * Np + r] = v0;
                    }
                    ybuf[((t - 1) & 3) * 32 + lane] = v0;
                }
            }
            if (sw == 0) {
                if (t < nlev && rvalid) {
                    double w;
                    if (t < S) {
                        const double hist = (t >= 2 ? c_h : 0.0) + (t >= 1 ? e1 * v0 : 0.0);
                        w = c_z - c_d1 * hist;
                    } else {
                        w = c_z - v0;  // f-level: z_f - y1_{S-1}
                    }
                    wbuf[(t & 3) * 32 + lane] = w;
                    a.xb[(long long)(0 * 2 + (t & 1)) * Np + r] = pad ? 0.0 : w * c_di;
                }
                release_rows(xr1);
                if (trp(t) && lane == 0) trp(t)[0] = gtime();
            }
            spare_bar();
            // chain-1 history of owner1(t+1): h1p = sum_{m<=t-1} e_{t+1-m} y1_m
            if (t >= 1 && t + 1 < S && t + 1 < nlev) {
                const double* ep = a.epad;
                const int py = lane & 15, gy = lane >> 4;
                const long long ry = r0 + 2 * py;
                const bool vy = ry < r1;
                double2 a1 = make_double2(0.0, 0.0);
                for (int i0 = 0; i0 <= t - 1; i0 += 2 * NSO * 8) {
                    double2 yv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int m = i0 + 2 * sw + gy + u * 2 * NSO;
                        yv[u] = vy && m <= t - 1
                                    ? __ldcg(reinterpret_cast<const double2*>(a.Y1 + (long long)m * Np + ry))
                                    : make_double2(0.0, 0.0);
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const double ev = __ldg(ep + t + 1 - (i0 + 2 * sw + gy + u * 2 * NSO));
                        a1.x += ev * yv[u].x;
                        a1.y += ev * yv[u].y;
                    }
                }
                a1.x += __shfl_down_sync(0xffffffffu, a1.x, 16);
                a1.y += __shfl_down_sync(0xffffffffu, a1.y, 16);
                if (lane < 16) {
                    hred[sw * 64 + 2 * lane] = a1.x;
                    hred[sw * 64 + 2 * lane + 1] = a1.y;
                }
                spare_bar();
                if (sw == 0) {
                    double s1 = 0.0;
                    for (int w2 = 0; w2 < NSO; ++w2) s1 += hred[w2 * 64 + lane];
                    h1p[lane] = s1;
                }
                spare_bar();
                if (trp(t) && sw == 0 && lane == 0) trp(t)[5] = gtime();
            }
        }
        // ---------------- owner2(t): d_{t-3} (y = y1 + d), x2_{t-2}
        if (t >= 2) {
            const int l = t - 2;
            const bool k1 = b_valid(t - 1), k2 = h32_valid(t - 1), do_x2 = l < nlev;
            double c_d1 = 0, c_d2 = 0, c_di = 0, c_h2 = 0;
            if (sw == 0 && do_x2) {
                const long long o = (long long)min(l, S - 1) * Np + rr;
                c_d1 = l < S ? a.D1[o] : 0.0;
                c_d2 = a.D2[o];
                c_di = a.d2inv[o];
            }
            if (k1) poll_bstep(t - 1);
            if (k2) poll_pdone(2, (unsigned)(nbb * clampi(t - 2, 0, nlev)));
            spare_bar();
            if (sw == 0) c_h2 = h2p[lane];
            if (k1) load_partials(1, (t - 1) & 1, 0);
            if (k2) load_partials(2, (t - 1) & 1, 1);
            spare_bar();
            if (sw == 0) {
                const double v1 = k1 ? sum_partials(0) : 0.0;
                const double v2 = k2 ? sum_partials(1) : 0.0;
                if (k2 && rvalid) {
                    const long long o = (long long)(t - 3) * Np + r;
                    a.DLf[o] = (float)v2;
                    a.y[o] = ybuf[((t - 3) & 3) * 32 + lane] + v2;
                }
                if (do_x2) {
                    if (rvalid) {
                        const double w = wbuf[(l & 3) * 32 + lane];
                        double x;
                        if (l < S) {
                            // r_l = w_l - e0 D1 o y1_l - cs D2 o B y1_l;  hist2 + e1 d_{l-1} (= v2)
                            const double res = w - c_d1 * a.epad[0] * ybuf[(l & 3) * 32 + lane] - a.cs * c_d2 * v1;
                            const double hist = (l >= 2 ? c_h2 : 0.0) + (l >= 1 ? e1 * v2 : 0.0);
                            x = (res - c_d1 * hist) * c_di;
                        } else {
                            // f-level: r_f = w_f - cr D2_{S-1} o B y1_S;  x2 = (r_f - d_{S-1}) / D2
                            x = (w - a.cr * c_d2 * v1 - v2) * c_di;
                        }
                        a.xb[(long long)(2 * 2 + (t & 1)) * Np + r] = pad ? 0.0 : x;
                    }
                    release_rows(xr2);
                }
                if (trp(t) && lane == 0) trp(t)[1] = gtime();
            }
            spare_bar();
            // chain-2 history of owner2(t+1) (l' = t-1): h2p = sum_{m<=t-3} e_{t-1-m} d_m
            if (t >= 3 && t - 1 < S && t - 1 < nlev) {
                const double* ep = a.epad;
                const int pd = lane & 7, gd = lane >> 3;
                const long long rdr = r0 + 4 * pd;
                const bool vd = rdr < r1;
                double a2[4] = {0.0, 0.0, 0.0, 0.0};
                for (int i0 = 0; i0 <= t - 3; i0 += 4 * NSO * 4) {
                    float4 dv[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int m = i0 + 4 * sw + gd + u * 4 * NSO;
                        dv[u] = vd && m <= t - 3
                                    ? __ldcg(reinterpret_cast<const float4*>(a.DLf + (long long)m * Np + rdr))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const double em = __ldg(ep + t - 1 - (i0 + 4 * sw + gd + u * 4 * NSO));
                        a2[0] += em * dv[u].x;
                        a2[1] += em * dv[u].y;
                        a2[2] += em * dv[u].z;
                        a2[3] += em * dv[u].w;
                    }
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    a2[i] += __shfl_down_sync(0xffffffffu, a2[i], 16);
                    a2[i] += __shfl_down_sync(0xffffffffu, a2[i], 8);
                }
                if (lane < 8)
#pragma unroll
                    for (int i = 0; i < 4; ++i) hred[sw * 64 + 32 + 4 * lane + i] = a2[i];
                spare_bar();
                if (sw == 0) {
                    double s2 = 0.0;
                    for (int w2 = 0; w2 < NSO; ++w2) s2 += hred[w2 * 64 + 32 + lane];
                    h2p[lane] = s2;
                }
                spare_bar();
                if (trp(t) && sw == 0 && lane == 0) trp(t)[6] = gtime();
            }
        }
    }
}

int sweep_ir_smem_bytes() {
    return NHS * HSLOT * (int)sizeof(double) +
           (2 * NSO * 32 + NSO * 64 + 32 + 32 + 4 * 32 + 4 * 32 + NW * TB + NS * 128) * (int)sizeof(double) +
           TCAP * (int)sizeof(int) + 2 * NHS * (int)sizeof(uint64_t);
}


}  // namespace

bool sweep_ir_available(const fi_precond* P) {
    static const int env = [] {
        const char* v = getenv("FI_SWEEP_IR");
        return v ? atoi(v) : 1;
    }();
    return env != 0 && P->mode == 0 && P->Hf.p != nullptr && ((P->sys->L.Np + P->G - 1) / P->G + 3) / 4 * 4 <= RCAP &&
           P->nb <= KPS * NSO && (P->T + P->G - 1) / P->G <= TCAP;
}

void launch_sweep_ir(fi_ctx* ctx, fi_precond* P, const double* z, double* y, int levels, const int* skip) {
    const int smem = sweep_ir_smem_bytes();
    const void* kern = (const void*)sweep_ir_kernel;
    ensure_smem_attr(kern, (size_t)smem);
    {
        int per_sm = 0;
        FI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem));
        if (per_sm < 1) throw Error(FI_E_CUDA, "sweep_ir_kernel cannot be resident");
    }
    const fi_system* sys = P->sys;
    const Layout& L = sys->L;
    if (((L.Np + P->G - 1) / P->G + 3) / 4 * 4 > RCAP) throw Error(FI_E_RESOURCE, "sweep_ir: too many rows per CTA");
    if (!P->ir_xb.p) {
        P->ir_xb.alloc((size_t)6 * L.Np);
        P->ir_pb.alloc((size_t)6 * P->nb * P->nb * TB);
        P->ir_counters.alloc((size_t)6 * P->nb * CSTR);
    }
    IrArgs a;
    a.H64 = P->H.p;
    a.H32 = P->Hf.p;
    a.T = P->T;
    a.nb = P->nb;
    a.nlev = levels;
    a.S = L.S;
    a.n1 = L.n1;
    a.n2 = L.n2;
    a.ld2 = L.ld2;
    a.gen_stride = 2 * L.ld2 + 8;
    a.Np = L.Np;
    a.z = z;
    a.y = y;
    a.Y1 = P->rbuf.p;
    a.DLf = reinterpret_cast<float*>(P->dbuf.p);
    a.D1 = sys->D1.p;
    a.D2 = sys->D2.p;
    a.d2inv = P->d2inv.p;
    a.e = sys->e.p;
    a.epad = sys->epad.p + kEOFF;
    a.gen = sys->gen.p;
    a.cs = sys->cs;
    a.cr = sys->cr;
    a.xb = P->ir_xb.p;
    a.pb = P->ir_pb.p;
    a.xready = P->ir_counters.p;
    a.pdone = P->ir_counters.p + (size_t)P->nb * CSTR;
    a.xready2 = P->ir_counters.p + (size_t)4 * P->nb * CSTR;
    a.pdone1b = P->ir_counters.p + (size_t)5 * P->nb * CSTR;
    a.skip = skip;
    static const int evict = [] {
        const char* v = std::getenv("FI_IR_EVICT");
        return v ? std::atoi(v) : 1;
    }();
    a.evict_first = evict;
    a.trace = nullptr;
    static const bool tracing = std::getenv("FI_SWEEP_TRACE") != nullptr;
    const int nst1 = levels + 3;
    DevBuf<unsigned long long> trace;
    if (tracing) {
        trace.alloc((size_t)P->G * nst1 * 12);
        FI_CUDA(cudaMemsetAsync(trace.p, 0, trace.bytes(), ctx->stream));
        a.trace = trace.p;
    }
    FI_CUDA(cudaMemsetAsync(P->ir_counters.p, 0, P->ir_counters.bytes(), ctx->stream));
    void* args[] = {&a};
    FI_CUDA(cudaLaunchCooperativeKernel(kern, dim3(P->G), dim3(THREADS), args, (size_t)smem, ctx->stream));
    FI_LAUNCHED(ctx);
    if (tracing) {
        std::vector<unsigned long long> h(trace.n);
        FI_CUDA(cudaMemcpyAsync(h.data(), trace.p, trace.bytes(), cudaMemcpyDeviceToHost, ctx->stream));
        FI_CUDA(cudaStreamSynchronize(ctx->stream));
        auto ph = [&](int c, int t, int i) { return (double)h[((size_t)c * nst1 + t) * 12 + i]; };
        // relative to the ring's step start (CTA c, step t): owner1 publish, owner2 publish, FP64 done,
        // B done, FP32 done, hist1 done, hist2 done
        for (int lo : {4, nst1 / 2, nst1 - 40}) {
            double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
            int cnt = 0;
            for (int c = 0; c < P->G; ++c)
                for (int t = lo; t < lo + 32 && t < nst1 - 4; ++t) {
                    const double s0 = ph(c, t, 7);
                    for (int i = 0; i < 7; ++i) acc[i] += ph(c, t, i) - s0;
                    acc[7] += ph(c, t + 1, 7) - s0;
                    acc[8] += ph(c, t, 8);
                    ++cnt;
                }
            std::fprintf(stderr,
                         "[sweep_ir] steps %3d+: step %6.2f us | own1 pub %6.2f | own2 pub %6.2f | FP64 done %6.2f | "
                         "B done %6.2f | FP32 done %6.2f | hist1 %6.2f | hist2 %6.2f | producer blocked %6.2f\n",
                         lo, acc[7] / cnt * 1e-3, acc[0] / cnt * 1e-3, acc[1] / cnt * 1e-3, acc[2] / cnt * 1e-3,
                         acc[3] / cnt * 1e-3, acc[4] / cnt * 1e-3, acc[5] / cnt * 1e-3, acc[6] / cnt * 1e-3,
                         acc[8] / cnt * 1e-3);
        }
    }
}

}  // namespace fib
