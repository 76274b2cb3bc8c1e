// K2 — block lower-triangular preconditioner apply (forward block substitution), B200.
//
// Reference: BlockTriangularPreconditioner::apply (krylov.cpp:48-70):
//   y_s = G_s^{-1} (z_s - D1_s o sum_{m<s} e_{s-m} y_m)  (s = 1..S),   y_f = G_f^{-1} (z_f - y_S).
// Each block is G = D2 M with M symmetric positive definite; precond_build.cu stores
// H = M^{-1} as the packed lower triangle of 64x64 tiles, so a level is
//   x_s = D2_s^{-1} (z_s - D1_s o hist_s),   y_s = H_s x_s   (symmetric tile products).
//
// One persistent cooperative kernel per sweep, with no grid-wide barrier on the level path:
//  * warp 16 (producer) streams this CTA's tiles of every level from HBM with
//    cp.async.bulk (TMA bulk copy) into an mbarrier ring, and keeps about one level of
//    tiles ahead in L2 with cp.async.bulk.prefetch.L2 — the HBM stream never waits for the
//    sequential substitution;
//  * warps 0-15 each take whole tiles: tile (bi,bj) waits only for the two 64-row blocks of
//    x it reads (per-row-block release/acquire counters `xready`), computes H x_bj (row sums,
//    warp butterfly transpose-reduction) and H^T x_bi (column sums, per lane), writes the two
//    partial products and bumps `pdone` of both row blocks;
//  * the owner of a row range waits for `pdone` of its row blocks, sums the nb partials
//    (fixed order: bit-reproducible), and publishes the next level's x.  The L1 history
//    sum of the next level is accumulated from the CTA's own rows while tiles stream.
// The only grid-wide barrier is before the f-block refinement residual (once per sweep).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "precond.cuh"

namespace fib {
namespace {

constexpr int TB = 64;
constexpr int TILE = TB * TB;
constexpr int NW = 11;                  // worker warps (>= ring stages); 12 warps = 3 per SMSP at 168 regs
constexpr int NWT = NW * 32;            // worker threads
constexpr int THREADS = NWT + 32;       // + producer warp
constexpr int RING_BYTES = 196608;      // 6 x 32 KB (double) / 12 x 16 KB (float)
constexpr int RCAP = 128;               // max owned rows per CTA (checked on the host)
constexpr int CSTR = kCounterStride;    // counters one 128-byte line apart (no polling hot spot)
constexpr int CH = 4;                   // tiles per warp chunk (batched x waits / loads)

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
__device__ __forceinline__ void prefetch_l2(const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void history_bar(int nthreads) {
    asm volatile("bar.sync 2, %0;\n" ::"r"(nthreads) : "memory");
}
__device__ __forceinline__ void worker_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(NWT) : "memory"); }
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// release-ordered increment: this thread's earlier writes (and, cumulatively, writes it observed
// through bar.sync / __syncwarp) are visible before the counter moves
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// Warp-uniform wait (call with all 32 lanes): every lane polls the same word (one request per
// warp) and the exit test is a warp vote, so the warp never splits.  A lane-0-only spin leaves
// the warp diverged and every later shfl.sync pays a reconvergence (measured: 15 us per tile).
__device__ __forceinline__ void red_relaxed(unsigned* p, unsigned v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void warp_spin_until(const unsigned* p, unsigned target) {
    while (!__all_sync(0xffffffffu, ld_acquire(p) >= target)) __nanosleep(64);
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

__device__ __forceinline__ void tile_coords(long long t, int& bi, int& bj) {
    int r = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while ((long long)(r + 1) * (r + 2) / 2 <= t) ++r;
    while ((long long)r * (r + 1) / 2 > t) --r;
    bi = r;
    bj = (int)(t - (long long)r * (r + 1) / 2);
}

template <typename T>
struct Vec2;
template <>
struct Vec2<double> {
    using type = double2;
};
template <>
struct Vec2<float> {
    using type = float2;
};

struct SweepArgs {
    const void* H;  // [level][tile][TILE] of T
    long long T;    // tiles per level
    int nb, levels, S, n1, n2, ld2, gen_stride, refine_f, pf_tiles;
    long long Np;
    const double* z;
    double* y;
    const double* D1;
    const double* d2inv;
    const double* e;
    const double* gen;
    double cr;
    double* xbuf;            // 2 x Np (pass parity)
    double* pbuf;            // 2 x nb x nb x TB (pass parity)
    unsigned* xready;        // nb
    unsigned* pdone;         // nb
    unsigned* bar;           // grid barrier (refinement only)
    const int* skip;
    unsigned long long* trace;  // optional phase timestamps [G][npass][5] (FI_SWEEP_TRACE=1)
};

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ int owners_of_block(int rb, long long R, unsigned G) {
    const long long first = (long long)rb * TB / R;
    const long long last = min((long long)G - 1, ((long long)rb * TB + TB - 1) / R);
    return (int)(last - first + 1);
}

template <typename T>
// 168 registers x 384 threads (3 warps per SM sub-partition) fit one CTA per SM; without the cap
// ptxas stops at 128 and spills the butterfly row partials to local memory (L1 misses after every level)
__global__ void __maxnreg__(168) sweep_kernel(SweepArgs a) {
    if (a.skip && *a.skip) return;
    constexpr int NST = sizeof(T) == 8 ? 6 : 11;  // ring stages inside the RING_BYTES region
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* ring = reinterpret_cast<T*>(smem_raw);
    double* red = reinterpret_cast<double*>(smem_raw + RING_BYTES);  // NW x 32
    double* histp = red + NW * 32;                                     // RCAP
    double* xis = histp + RCAP;                                        // NST x CH x TB (x_bi staging)
    uint64_t* full = reinterpret_cast<uint64_t*>(xis + NST * CH * TB);
    uint64_t* empty = full + NST;

    const unsigned G = gridDim.x;
    const long long t0 = (long long)blockIdx.x * a.T / G;
    const long long t1 = (long long)(blockIdx.x + 1) * a.T / G;
    const long long ntiles = t1 - t0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int npass = a.levels + a.refine_f;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    if (warp == NW) {
        // ---------------- producer: every pass's tiles, in (pass, tile) order; L2 prefetch ahead
        if (lane == 0) {
            const T* Hb = reinterpret_cast<const T*>(a.H);
            const long long total = (long long)npass * ntiles;
            auto src_of = [&](long long it) {
                const long long p = it / ntiles, k = it % ntiles;
                return Hb + ((long long)min((int)p, a.S) * a.T + t0 + k) * TILE;
            };
            const long long npf = (long long)a.pf_tiles < total ? (long long)a.pf_tiles : total;
            for (long long it = 0; it < npf; ++it)
                prefetch_l2(src_of(it), TILE * sizeof(T));
            for (long long it = 0; it < total; ++it) {
                if (it + a.pf_tiles < total) prefetch_l2(src_of(it + a.pf_tiles), TILE * sizeof(T));
                const int slot = (int)(it % NST);
                if (it >= NST) mbar_wait(&empty[slot], (unsigned)((it / NST - 1) & 1));
                mbar_expect_tx(&full[slot], TILE * sizeof(T));
                tma_bulk_g2s(ring + slot * TILE, src_of(it), TILE * sizeof(T), &full[slot]);
            }
        }
        return;
    }

    // ---------------- workers
    const long long Np = a.Np;
    const long long R = (Np + G - 1) / G;
    const long long r0 = min(Np, (long long)blockIdx.x * R);
    const long long r1 = min(Np, r0 + R);
    const int rb0 = (int)(r0 / TB), rb1 = r1 > r0 ? (int)((r1 - 1) / TB) : rb0 - 1;  // owned row blocks
    const int nbb = a.nb;
    unsigned bar_target = 0;

    // owner: y of pass q on owned rows = sum of nb partials (fixed order)
    auto owner_reduce = [&](int q, bool accumulate) {
        if (warp == 0)
            for (int rb = rb0; rb <= rb1; ++rb) warp_spin_until(a.pdone + rb * CSTR, (unsigned)nbb * (q + 1));
        worker_bar();
        const double* pb = a.pbuf + (long long)(q & 1) * nbb * nbb * TB;
        const int lvl = min(q, a.S);
        for (long long rc = r0; rc < r1; rc += 32) {
            const long long r = rc + lane;
            const bool valid = r < r1;
            double part = 0.0;
            if (valid) {
                const long long rb = r / TB, ro = r % TB;
                double acc[4] = {0, 0, 0, 0};
                int k = warp;
                for (; k + 3 * NW < nbb; k += 4 * NW) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) acc[u] += __ldcg(pb + (rb * nbb + k + u * NW) * TB + ro);
                }
                for (; k < nbb; k += NW) acc[0] += __ldcg(pb + (rb * nbb + k) * TB + ro);
                part = (acc[0] + acc[1]) + (acc[2] + acc[3]);
            }
            red[warp * 32 + lane] = part;
            worker_bar();
            if (warp == 0 && valid) {
                double s = 0.0;
                for (int w = 0; w < NW; ++w) s += red[w * 32 + lane];
                double* yp = a.y + (long long)lvl * Np + r;
                if (accumulate) s += *yp;
                *yp = s;
            }
            worker_bar();
        }
    };
    // owner: publish x of pass p on owned rows (hist = precomputed part + e_1 y_{p-1})
    auto owner_x = [&](int p) {
        double* xb = a.xbuf + (long long)(p & 1) * Np;
        if (warp == 0) {
            for (long long rc = r0; rc < r1; rc += 32) {
                const long long r = rc + lane;
                if (r >= r1) continue;
                double x;
                if (p < a.S) {
                    double hist = p > 0 ? histp[r - r0] + a.e[1] * __ldcg(a.y + (long long)(p - 1) * Np + r) : 0.0;
                    if (p == 1) hist = a.e[1] * __ldcg(a.y + r);
                    const long long o = (long long)p * Np + r;
                    x = (a.z[o] - a.D1[o] * hist) * a.d2inv[o];
                } else {
                    const long long o = (long long)a.S * Np + r;
                    x = (a.z[o] - __ldcg(a.y + (long long)(a.S - 1) * Np + r)) *
                        a.d2inv[(long long)(a.S - 1) * Np + r];
                }
                xb[r] = x;
            }
        }
        worker_bar();
        if (threadIdx.x == 0) {
            for (int rb = rb0; rb <= rb1; ++rb) red_release(a.xready + rb * CSTR, 1u);
        }
    };

    long long it = 0;
    for (int p = 0; p < npass; ++p) {
        const bool refine = p == a.levels;
        // ---- owner step: finish y of pass p-1, publish x of pass p
        unsigned long long* tr = a.trace ? a.trace + ((long long)blockIdx.x * npass + p) * 5 : nullptr;
        if (tr && threadIdx.x == 0) tr[0] = gtime();
        if (p > 0) owner_reduce(p - 1, false);
        if (tr && threadIdx.x == 0) tr[1] = gtime();
        if (refine) {
            // residual of the f-block solve needs every row of y_f: the sweep's only grid barrier
            worker_bar();
            bar_target += G;
            if (threadIdx.x == 0) red_release(a.bar, 1u);
            if (warp == 0) warp_spin_until(a.bar, bar_target);
            worker_bar();
            const double* yf = a.y + (long long)a.S * Np;
            const double* xf = a.xbuf + (long long)((p - 1) & 1) * Np;
            double* xb = a.xbuf + (long long)(p & 1) * Np;
            for (long long r = r0 + warp; r < r1; r += NW) {
                const int i1 = (int)(r / a.ld2), i2 = (int)(r % a.ld2);
                double acc = 0.0;
                if (i2 < a.n2) {
                    for (int j1 = 0; j1 < a.n1; ++j1) {
                        const double* grow = a.gen + (long long)(i1 - j1 + a.n1 - 1) * a.gen_stride + i2 + a.ld2;
                        const double* yrow = yf + (long long)j1 * a.ld2;
                        for (int j2 = lane; j2 < a.n2; j2 += 32) acc += grow[-j2] * __ldcg(yrow + j2);
                    }
                }
                acc = warp_sum(acc);
                if (lane == 0) xb[r] = i2 < a.n2 ? __ldcg(xf + r) - a.cr * acc : 0.0;
            }
            worker_bar();
            if (threadIdx.x == 0) {
                for (int rb = rb0; rb <= rb1; ++rb) red_release(a.xready + rb * CSTR, 1u);
            }
        } else {
            owner_x(p);
        }
        if (tr && threadIdx.x == 0) tr[2] = gtime();

        // ---- tiles of pass p: warp w < NST takes tiles k = w, w + NST, ...  (items k and k + NST
        //      share a ring slot, so the same warp consumes them in order: mbarrier parity safe).
        //      Per chunk of CH tiles the warp waits for all their x blocks in one poll round and
        //      stages them with one round of loads, so later tiles add no global round trips.
        const double* xb = a.xbuf + (long long)(p & 1) * Np;
        double* pb = a.pbuf + (long long)(p & 1) * nbb * nbb * TB;
        for (long long kc = warp; warp < NST && kc < ntiles; kc += (long long)CH * NST) {
            int cbi[CH], cbj[CH];
            int nch = 0;
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const long long k = kc + (long long)c * NST;
                cbi[c] = cbj[c] = 0;
                if (k < ntiles) {
                    tile_coords(t0 + k, cbi[c], cbj[c]);
                    nch = c + 1;
                }
            }
            // poll the 2*nch x-ready counters at once: lane 2c polls x_bi, lane 2c+1 polls x_bj
            {
                int rbs = 0;
#pragma unroll
                for (int c = 0; c < CH; ++c)
                    if ((lane >> 1) == c) rbs = (lane & 1) ? cbj[c] : cbi[c];
                const bool mine = lane < 2 * nch;
                const unsigned* cp = a.xready + rbs * CSTR;
                const unsigned tgt = (unsigned)owners_of_block(rbs, R, G) * (p + 1);
                while (!__all_sync(0xffffffffu, !mine || ld_acquire(cp) >= tgt)) __nanosleep(64);
            }
            // stage x_bi (all 64 values, smem) and x_bj (this lane's 2 columns, registers)
            double2 xj[CH];
            double* xs = xis + warp * (CH * TB);
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                if (c < nch) {
                    xj[c] = __ldcg(reinterpret_cast<const double2*>(xb + (long long)cbj[c] * TB) + lane);
                    reinterpret_cast<double2*>(xs + c * TB)[lane] =
                        __ldcg(reinterpret_cast<const double2*>(xb + (long long)cbi[c] * TB) + lane);
                } else {
                    xj[c] = make_double2(0.0, 0.0);
                }
            }
            __syncwarp();
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                if (c >= nch) break;
                const int bi = cbi[c], bj = cbj[c];
                const long long item = it + kc + (long long)c * NST;
                const int slot = (int)(item % NST);
                const double* xi = xs + c * TB;
                mbar_wait(&full[slot], (unsigned)((item / NST) & 1));
                const T* tile = ring + slot * TILE;
                double c0 = 0.0, c1 = 0.0;
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    double pr[32];
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        const int r = half * 32 + q;
                        const auto hv = reinterpret_cast<const typename Vec2<T>::type*>(tile + r * TB)[lane];
                        const double hx = (double)hv.x, hy = (double)hv.y;
                        pr[q] = hx * xj[c].x + hy * xj[c].y;
                        const double xr = xi[r];
                        c0 += hx * xr;
                        c1 += hy * xr;
                    }
                    // butterfly transpose-reduction: lane l ends with sum over lanes of pr[l]
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
                    pb[((long long)bi * nbb + bj) * TB + half * 32 + lane] = pr[0];
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[slot]);
                if (bi != bj)
                    reinterpret_cast<double2*>(pb + ((long long)bj * nbb + bi) * TB)[lane] = make_double2(c0, c1);
            }
            __syncwarp();
        }
        // one release fence per warp and pass, then relaxed counter bumps for all its tiles
        // (a red.release per tile cost ~2 us each on the warp's critical path)
        if (warp < NST && warp < ntiles) {
            __syncwarp();
            if (lane == 0) {
                asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
                for (long long k = warp; k < ntiles; k += NST) {
                    int bi, bj;
                    tile_coords(t0 + k, bi, bj);
                    red_relaxed(a.pdone + bi * CSTR, 1u);
                    if (bi != bj) red_relaxed(a.pdone + bj * CSTR, 1u);
                }
            }
        }
        it += ntiles;
        if (tr) {
            worker_bar();
            if (threadIdx.x == 0) tr[3] = gtime();
        }

        // ---- L1 history of the next time level from this CTA's own rows (m <= p-1), while
        //      other CTAs' tiles are still streaming: hist_{p+1} = sum_{m<p} e_{p+1-m} y_m.
        //      With spare warps (NW > NST) they run it concurrently with the tile warps.
        if (!refine && p + 1 < a.S && p >= 1 && (NW == NST || warp >= NST)) {
            const int hw0 = NW == NST ? 0 : NST;       // first history warp
            const int nhw = NW - hw0;                   // history warps
            const int hwarp = warp - hw0;
            for (long long rc = r0; rc < r1; rc += 32) {
                const long long r = rc + lane;
                const bool valid = r < r1;
                double part = 0.0;
                if (valid) {
                    // 8 independent accumulators keep 8 L2 loads in flight per lane
                    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                    int m = hwarp;
                    for (; m + 7 * nhw < p; m += 8 * nhw) {
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int mm = m + u * nhw;
                            acc[u] += __ldg(a.e + p + 1 - mm) * __ldcg(a.y + (long long)mm * Np + r);
                        }
                    }
                    for (; m < p; m += nhw) acc[0] += __ldg(a.e + p + 1 - m) * __ldcg(a.y + (long long)m * Np + r);
                    part = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
                }
                red[hwarp * 32 + lane] = part;
                history_bar(nhw * 32);
                if (hwarp == 0 && valid) {
                    double sum = 0.0;
                    for (int w = 0; w < nhw; ++w) sum += red[w * 32 + lane];
                    histp[r - r0] = sum;
                }
                history_bar(nhw * 32);
            }
        }
        if (tr && threadIdx.x == 0) tr[4] = gtime();
    }
    // y of the last pass
    owner_reduce(npass - 1, a.refine_f != 0);
    (void)0;
}

template <typename T>
int sweep_smem_bytes() {
    constexpr int NST = sizeof(T) == 8 ? 6 : 11;  // ring stages inside the RING_BYTES region
    return RING_BYTES + (NW * 32 + RCAP + NST * CH * TB) * (int)sizeof(double) + 2 * NST * (int)sizeof(uint64_t);
}

__global__ void axpy_kernel(double* y, const double* d, long long n, const int* skip) {
    if (skip && *skip) return;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] += d[i];
}

// (A - P) v: the only block where the operator and its block lower-triangular preconditioner differ
// is the f column of the time rows, -eta q_s I (spectra.cpp:34-36); u_s = -eta q_s f_v, u_f = 0.
__global__ void coupling_kernel(const double* __restrict__ v, double* __restrict__ u, const double* __restrict__ q,
                                double eta, int S, long long Np, const int* skip) {
    if (skip && *skip) return;
    const long long n = (long long)(S + 1) * Np;
    const double* f = v + (long long)S * Np;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long s = i / Np, j = i - s * Np;
        u[i] = s < S ? -eta * q[s] * f[j] : 0.0;
    }
}
__global__ void add_kernel(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out,
                           long long n, const int* skip) {
    if (skip && *skip) return;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = a[i] + b[i];
}

template <typename T>
void launch_sweep(fi_ctx* ctx, fi_precond* P, const T* H, const double* z, double* y, int levels, int refine_f,
                  const int* skip) {
    const int smem = sweep_smem_bytes<T>();
    ensure_smem_attr((const void*)sweep_kernel<T>, (size_t)smem);
    const fi_system* sys = P->sys;
    SweepArgs a;
    a.H = H;
    a.T = P->T;
    a.nb = P->nb;
    a.levels = levels;
    a.S = sys->L.S;
    a.n1 = sys->L.n1;
    a.n2 = sys->L.n2;
    a.ld2 = sys->L.ld2;
    a.gen_stride = 2 * sys->L.ld2 + 8;
    a.refine_f = refine_f;
    // L2 prefetch distance (tiles ahead of the TMA issue point; FI_PF_TILES overrides), capped
    // so the grid keeps at most FI_PF_MB (default 80) MB of prefetched tiles in the 126 MB L2
    static const long long pf_env = [] {
        const char* s = std::getenv("FI_PF_TILES");
        return s ? std::atoll(s) : -1ll;
    }();
    static const long long pf_mb = [] {
        const char* s = std::getenv("FI_PF_MB");
        return s ? std::atoll(s) : 80ll;
    }();
    const long long per_cta = (P->T + P->G - 1) / P->G;
    const long long cap = (pf_mb << 20) / ((long long)P->G * TILE * (long long)sizeof(T));
    // measured on config 1: every prefetch distance > 0 slowed the sweep (L2 thrash) -> default 0
    const long long want = pf_env >= 0 ? pf_env : 0;
    (void)per_cta;
    a.pf_tiles = (int)std::max<long long>(0, std::min(want, cap));
    a.Np = sys->L.Np;
    a.z = z;
    a.y = y;
    a.D1 = sys->D1.p;
    a.d2inv = P->d2inv.p;
    a.e = sys->e.p;
    a.gen = sys->gen.p;
    a.cr = sys->cr;
    a.xbuf = P->xbuf.p;
    a.pbuf = P->pbuf.p;
    a.xready = P->counters.p;
    a.pdone = P->counters.p + (size_t)P->nb * CSTR;
    a.bar = P->counters.p + (size_t)2 * P->nb * CSTR;
    a.skip = skip;
    a.trace = nullptr;

    static const bool tracing = std::getenv("FI_SWEEP_TRACE") != nullptr;
    DevBuf<unsigned long long> trace;
    const int npass = levels + refine_f;
    if (tracing) {
        trace.alloc((size_t)P->G * npass * 5);
        FI_CUDA(cudaMemsetAsync(trace.p, 0, trace.bytes(), ctx->stream));
        a.trace = trace.p;

    }
    FI_CUDA(cudaMemsetAsync(P->counters.p, 0, P->counters.bytes(), ctx->stream));
    void* args[] = {&a};
    FI_CUDA(cudaLaunchCooperativeKernel((const void*)sweep_kernel<T>, dim3(P->G), dim3(THREADS), args, (size_t)smem,
                                        ctx->stream));
    FI_LAUNCHED(ctx);
    if (tracing) {
        std::vector<unsigned long long> h(trace.n);
        FI_CUDA(cudaMemcpyAsync(h.data(), trace.p, trace.bytes(), cudaMemcpyDeviceToHost, ctx->stream));
        FI_CUDA(cudaStreamSynchronize(ctx->stream));
        const unsigned long long base = h[0];
        for (int c : {0, P->G / 2, P->G - 1})
            for (int p : {1, 2, npass / 2, npass - 2})
                if (p >= 0 && p < npass) {
                    const unsigned long long* t = h.data() + ((size_t)c * npass + p) * 5;
                    std::fprintf(stderr,
                                 "[sweep<%s>] cta %3d pass %3d: start %8.2f us | reduce %6.2f | x %6.2f | tiles %6.2f | "
                                 "hist %6.2f\n",
                                 sizeof(T) == 8 ? "f64" : "f32", c, p, (t[0] - base) * 1e-3, (t[1] - t[0]) * 1e-3,
                                 (t[2] - t[1]) * 1e-3, (t[3] - t[2]) * 1e-3, t[4] > t[3] ? (t[4] - t[3]) * 1e-3 : 0.0);
                }
    }
}

}  // namespace

int precond_apply_grid(fi_ctx* ctx, long long T, long long Np) {
    int per_sm = 0;
    ensure_smem_attr((const void*)sweep_kernel<double>, (size_t)sweep_smem_bytes<double>());
    FI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_kernel<double>, THREADS,
                                                          sweep_smem_bytes<double>()));
    if (per_sm < 1) throw Error(FI_E_CUDA, "precond sweep kernel cannot be resident");
    long long G = std::min<long long>(ctx->sm_count, std::max<long long>(T, (Np + 31) / 32));
    G = std::max<long long>(G, (Np + RCAP - 1) / RCAP);
    if (G > (long long)ctx->sm_count * per_sm)
        throw Error(FI_E_RESOURCE, "precond sweep: block of " + std::to_string(Np) + " rows needs " +
                                       std::to_string(G) + " resident CTAs");
    return (int)G;
}

// w = P^{-1} A v computed as v + P^{-1} ((A - P) v): one sweep and no operator apply (the identity is
// exact; the rounding differs from P^{-1}(A v) at the level of the sweep's own accuracy).  u, t: scratch.
void precond_times_operator(fi_ctx* ctx, fi_precond* P, const double* v, double* w, double* u, double* t,
                            const int* skip) {
    const fi_system* sys = P->sys;
    const long long n = sys->L.nI();
    coupling_kernel<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(v, u, sys->q.p, sys->eta, sys->L.S, sys->L.Np, skip);
    FI_LAUNCHED(ctx);
    precond_apply(ctx, P, u, t, sys->L.S + 1, skip);
    add_kernel<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(v, t, w, n, skip);
    FI_LAUNCHED(ctx);
}

void precond_apply(fi_ctx* ctx, fi_precond* P, const double* z, double* y, int levels, const int* skip) {
    if (P->mode == 1) {
        precond_apply_iterative(ctx, P, z, y, levels, skip);
        return;
    }
    const fi_system* sys = P->sys;
    const bool full = levels == sys->L.S + 1;
    if (P->hodlr) {
        // HODLR blocks: sweep, residual r = z - P y through K1, correction sweep, y += d
        hodlr_sweep(ctx, P->hodlr, sys, P->d2inv.p, z, y, levels, skip);
        if (!P->refine) return;
        if (!full)
            FI_CUDA(cudaMemsetAsync(y + (long long)sys->L.S * sys->L.Np, 0, sys->L.Np * sizeof(double), ctx->stream));
        toeplitz_apply(ctx, sys->view(), y, P->rbuf.p, skip, z, true);
        hodlr_sweep(ctx, P->hodlr, sys, P->d2inv.p, P->rbuf.p, P->dbuf.p, levels, skip);
        axpy_kernel<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(y, P->dbuf.p, (long long)levels * sys->L.Np, skip);
        FI_LAUNCHED(ctx);
        return;
    }
    if (P->refine && sweep_ir_available(P)) {
        // sweep + residual + refinement sweep interleaved in one persistent kernel
        launch_sweep_ir(ctx, P, z, y, levels, skip);
        return;
    }
    // sweep 1: forward block substitution with the FP64 inverses (+ in-kernel f-block refinement)
    launch_sweep<double>(ctx, P, P->H.p, z, y, levels, full ? 1 : 0, skip);
    if (!P->refine) return;
    // one step of iterative refinement: r = z - P y for all levels at once with
    // K1, d = P^{-1} r with the FP32 copy of the inverses (|d| ~ 1e-12 |y|), y += d
    if (!full)
        FI_CUDA(cudaMemsetAsync(y + (long long)sys->L.S * sys->L.Np, 0, sys->L.Np * sizeof(double), ctx->stream));
    toeplitz_apply(ctx, sys->view(), y, P->rbuf.p, skip, z, true);
    launch_sweep<float>(ctx, P, P->Hf.p, P->rbuf.p, P->dbuf.p, levels, 0, skip);
    const long long n = (long long)levels * sys->L.Np;
    axpy_kernel<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(y, P->dbuf.p, n, skip);
    FI_LAUNCHED(ctx);
}

}  // namespace fib
