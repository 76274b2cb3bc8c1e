// K2 — block lower-triangular preconditioner: setup and apply on the B200.
//
// Reference: BlockTriangularPreconditioner (krylov.cpp:24-70).  Each diagonal block is
//   G_s = cs D2_s B + e0 D1_s   (s = 1..S),      G_f = cr D2_S B   (f-block),
// which the reference LU-factorises and solves per level.  Here every block is written
// as G = D2 M with M = cs B + e0 diag(D1/D2) (resp. cr B) symmetric positive definite, and
// the library stores the explicit symmetric inverse H = M^{-1} once, packed as the lower
// triangle of 64x64 tiles.  The apply is the reference's forward block substitution
//   x_s = D2_s^{-1} (z_s - D1_s o sum_{m<s} e_{s-m} y_m),   y_s = H_s x_s,
//   x_f = D2_S^{-1} (z_f - y_S),                            y_f = H_f x_f,
// executed by ONE persistent cooperative kernel: a producer warp streams each CTA's tiles
// of all levels from HBM with cp.async.bulk (TMA bulk copies) into a 6-stage mbarrier
// ring, running ahead across level boundaries, while 16 compute warps do the symmetric
// tile products; two grid barriers per level order the sequential substitution.  HBM
// traffic per apply is half of an LU-factor stream (symmetric storage).
//
// Setup: batched blocked Gauss-Jordan inversion (no pivoting — M is SPD) on the device,
// FP64 DMMA for the rank-64 updates.  Pivot check as krylov.cpp:14-20 on the Gauss-Jordan
// pivots (the LDL^T diagonal of M).
#include <cmath>

#include "precond.cuh"

namespace fib {
namespace {

constexpr int TB = 64;            // tile edge
constexpr int TILE = TB * TB;     // doubles per tile
constexpr int NST = 6;            // TMA ring stages (32 KB each)
constexpr int NCW = 16;           // compute warps
constexpr int NCT = NCW * 32;     // compute threads
constexpr int APPLY_THREADS = NCT + 32;  // + producer warp

// ------------------------------------------------------------------ PTX helpers
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
__device__ __forceinline__ void compute_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(NCT) : "memory"); }

__device__ __forceinline__ void grid_sync(unsigned* ctr, unsigned& target, unsigned G) {
    compute_bar();
    if (threadIdx.x == 0) {
        target += G;
        __threadfence();
        atomicAdd(ctr, 1u);
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ctr) : "memory");
        } while (v < target);
        __threadfence();
    }
    compute_bar();
}

__device__ __forceinline__ void tile_coords(long long t, int& bi, int& bj) {
    // lower-triangular row-major order: t = bi (bi + 1) / 2 + bj, bj <= bi
    int r = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while ((long long)(r + 1) * (r + 2) / 2 <= t) ++r;
    while ((long long)r * (r + 1) / 2 > t) --r;
    bi = r;
    bj = (int)(t - (long long)r * (r + 1) / 2);
}

// ------------------------------------------------------------------ apply kernel
struct ApplyArgs {
    const void* H;  // [level][tile][64*64] of T (double: main pass, float: refinement pass)
    long long T;
    int nb, levels, S, n2, ld2;
    long long Np;
    const double* z;
    double* y;
    const double* D1;
    const double* d2inv;
    const double* e;
    double* xbuf;
    double* pbuf;
    unsigned* bar;
    const int* skip;
    // f-block refinement (levels == S+1): generating tensor of B for the residual x_f - cr B y_f
    int refine_f, n1, gen_stride;
    const double* gen;
    double cr;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
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

template <typename T>
__global__ void __launch_bounds__(APPLY_THREADS, 1) precond_apply_kernel(ApplyArgs a) {
    if (a.skip && *a.skip) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* ring = reinterpret_cast<T*>(smem_raw);                           // NST x TILE
    double* csum = reinterpret_cast<double*>(ring + NST * TILE);        // 2 x NCW x TB
    double* red = csum + 2 * NCW * TB;                                  // NCW x 32
    uint64_t* full = reinterpret_cast<uint64_t*>(red + NCW * 32);       // NST
    uint64_t* empty = full + NST;                                       // NST

    const unsigned G = gridDim.x;
    const long long t0 = (long long)blockIdx.x * a.T / G;
    const long long t1 = (long long)(blockIdx.x + 1) * a.T / G;
    const long long ntiles = t1 - t0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    if (warp == NCW) {
        // ---------------- producer: stream this CTA's tiles of every level, ahead of the math
        if (lane == 0) {
            long long it = 0;
            const int npass = a.levels + (a.refine_f ? 1 : 0);
            for (int L = 0; L < npass; ++L) {
                const T* src = reinterpret_cast<const T*>(a.H) + ((long long)min(L, a.S) * a.T + t0) * TILE;
                for (long long k = 0; k < ntiles; ++k, ++it) {
                    const int slot = (int)(it % NST);
                    if (it >= NST) mbar_wait(&empty[slot], (unsigned)((it / NST - 1) & 1));
                    mbar_expect_tx(&full[slot], TILE * sizeof(T));
                    tma_bulk_g2s(ring + slot * TILE, src + k * TILE, TILE * sizeof(T), &full[slot]);
                }
            }
        }
        return;
    }

    // ---------------- compute warps
    const long long Np = a.Np;
    const long long rows_per = (Np + G - 1) / G;
    const long long r0 = (long long)blockIdx.x * rows_per;
    const long long r1 = min(Np, r0 + rows_per);
    unsigned target = 0;
    long long it = 0;
    int cpar = 0;

    const int npass = a.levels + (a.refine_f ? 1 : 0);
    for (int L = 0; L < npass; ++L) {
        const bool refine = L == a.levels;  // refinement pass of the f-block: y_f += H_f (x_f - cr B y_f)
        if (refine) {
            // ---- phase X': residual of the f-block solve on owned rows (needs every row of y_f)
            grid_sync(a.bar, target, G);
            const double* yf = a.y + (long long)a.S * Np;
            for (long long r = r0 + warp; r < r1; r += NCW) {
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
                if (lane == 0) a.xbuf[r] = i2 < a.n2 ? __ldcg(a.xbuf + r) - a.cr * acc : 0.0;
            }
            compute_bar();
        } else
        // ---- phase X: x_L on owned rows (history sum over this CTA's own y rows)
        for (long long rc = r0; rc < r1; rc += 32) {
            const long long r = rc + lane;
            const bool valid = r < r1;
            double part = 0.0;
            if (L < a.S) {
                if (valid)
                    for (int m = warp; m < L; m += NCW) part += a.e[L - m] * __ldcg(a.y + (long long)m * Np + r);
            }
            red[warp * 32 + lane] = part;
            compute_bar();
            if (warp == 0 && valid) {
                double hist = 0.0;
                for (int w = 0; w < NCW; ++w) hist += red[w * 32 + lane];
                double x;
                if (L < a.S) {
                    const long long o = (long long)L * Np + r;
                    x = (a.z[o] - a.D1[o] * hist) * a.d2inv[o];
                } else {
                    const long long o = (long long)a.S * Np + r;
                    x = (a.z[o] - __ldcg(a.y + (long long)(a.S - 1) * Np + r)) * a.d2inv[(long long)(a.S - 1) * Np + r];
                }
                a.xbuf[r] = x;
            }
            compute_bar();
        }
        grid_sync(a.bar, target, G);

        // ---- phase T: symmetric tile products of H_L with x_L
        for (long long k = 0; k < ntiles; ++k, ++it) {
            int bi, bj;
            tile_coords(t0 + k, bi, bj);
            const int slot = (int)(it % NST);
            const double2 xj = __ldcg(reinterpret_cast<const double2*>(a.xbuf + bj * TB) + lane);
            double xi[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) xi[q] = __ldcg(a.xbuf + bi * TB + 4 * warp + q);
            mbar_wait(&full[slot], (unsigned)((it / NST) & 1));
            const T* tile = ring + slot * TILE;
            double2 hv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const auto v = reinterpret_cast<const typename Vec2<T>::type*>(tile + (4 * warp + q) * TB)[lane];
                hv[q] = make_double2((double)v.x, (double)v.y);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            // row sums: (H x_bj)[4w+q]
            double rs[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) rs[q] = hv[q].x * xj.x + hv[q].y * xj.y;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1)
#pragma unroll
                for (int q = 0; q < 4; ++q) rs[q] += __shfl_xor_sync(0xffffffffu, rs[q], off);
            if (lane < 4) {
                const double v = lane == 0 ? rs[0] : lane == 1 ? rs[1] : lane == 2 ? rs[2] : rs[3];
                a.pbuf[((long long)bi * a.nb + bj) * TB + 4 * warp + lane] = v;
            }
            if (bi != bj) {
                // column sums: (H^T x_bi)[2 lane + c] over this warp's 4 rows, then across warps
                double c0 = 0.0, c1 = 0.0;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    c0 += hv[q].x * xi[q];
                    c1 += hv[q].y * xi[q];
                }
                double* cs = csum + cpar * NCW * TB;
                cs[warp * TB + 2 * lane] = c0;
                cs[warp * TB + 2 * lane + 1] = c1;
                compute_bar();
                if (threadIdx.x < TB) {
                    double s = 0.0;
                    for (int w = 0; w < NCW; ++w) s += cs[w * TB + threadIdx.x];
                    a.pbuf[((long long)bj * a.nb + bi) * TB + threadIdx.x] = s;
                }
                cpar ^= 1;
            }
        }
        grid_sync(a.bar, target, G);

        // ---- phase R: y_L on owned rows = sum of the nb partial products of its row block
        for (long long rc = r0; rc < r1; rc += 32) {
            const long long r = rc + lane;
            const bool valid = r < r1;
            double part = 0.0;
            if (valid) {
                const long long rb = r / TB, ro = r % TB;
                for (int k = warp; k < a.nb; k += NCW) part += __ldcg(a.pbuf + (rb * a.nb + k) * TB + ro);
            }
            red[warp * 32 + lane] = part;
            compute_bar();
            if (warp == 0 && valid) {
                double s = 0.0;
                for (int w = 0; w < NCW; ++w) s += red[w * 32 + lane];
                if (refine) a.y[(long long)a.S * Np + r] += s;
                else a.y[(long long)L * Np + r] = s;
            }
            compute_bar();
        }
        // phase X of the next level reads only this CTA's own y rows: no grid barrier needed
    }
}

// ------------------------------------------------------------------ setup kernels
struct FillArgs {
    OperatorView op;
    double* W;          // batch x Np x Np
    int level0;         // first level of the batch (0-based; S = f-block)
    const double* diag; // S x Np: e0 * D1 / D2 (pads unused)
    const double* bscale; // per level: coefficient of B (cs, cr, or 0 for a D2 == 0 level)
};

__global__ void gj_fill(FillArgs f) {
    const long long Np = f.op.Np;
    const int b = blockIdx.y;
    const int L = f.level0 + b;
    double* W = f.W + (long long)b * Np * Np;
    const double scale = f.bscale[L];
    const int n1 = f.op.n1, n2 = f.op.n2, ld2 = f.op.ld2;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < Np * Np;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long i = idx / Np, j = idx % Np;
        const int i1 = (int)(i / ld2), i2 = (int)(i % ld2), j1 = (int)(j / ld2), j2 = (int)(j % ld2);
        double v;
        if (i2 >= n2 || j2 >= n2) {
            v = i == j ? 1.0 : 0.0;
        } else {
            v = scale * f.op.gen[(long long)(i1 - j1 + n1 - 1) * f.op.gen_stride + (i2 - j2) + ld2];
            if (i == j && L < f.op.S) v += f.diag[(long long)L * Np + i];
        }
        W[idx] = v;
    }
}

// In-place Gauss-Jordan inversion of the 64x64 pivot block of each matrix; records pivots.
__global__ void gj_diag_inv(double* W, long long Np, int K0, double* Dinv, double* piv) {
    __shared__ double D[TB][TB + 1];
    __shared__ double rowp[TB];
    __shared__ double colp[TB];
    const int b = blockIdx.x;
    const double* Wb = W + (long long)b * Np * Np;
    for (int idx = threadIdx.x; idx < TILE; idx += blockDim.x) {
        const int r = idx / TB, c = idx % TB;
        D[r][c] = Wb[(long long)(K0 + r) * Np + K0 + c];
    }
    __syncthreads();
    double pmin = piv[2 * b], pmax = piv[2 * b + 1];
    for (int p = 0; p < TB; ++p) {
        const double pv = D[p][p];
        if (threadIdx.x < TB) {
            const int c = threadIdx.x;
            rowp[c] = (c == p ? 1.0 : D[p][c]) / pv;
            colp[c] = D[c][p];
        }
        __syncthreads();
        for (int idx = threadIdx.x; idx < TILE; idx += blockDim.x) {
            const int r = idx / TB, c = idx % TB;
            D[r][c] = r == p ? rowp[c] : (c == p ? 0.0 : D[r][c]) - colp[r] * rowp[c];
        }
        __syncthreads();
        pmin = fmin(pmin, pv);
        pmax = fmax(pmax, fabs(pv));
    }
    for (int idx = threadIdx.x; idx < TILE; idx += blockDim.x) {
        const int r = idx / TB, c = idx % TB;
        Dinv[(long long)b * TILE + idx] = D[r][c];
    }
    if (threadIdx.x == 0) {
        piv[2 * b] = pmin;
        piv[2 * b + 1] = pmax;
    }
}

// Ftmp = W[:, K]  (Np x 64);  Rtmp = Dinv W[K, :] with Rtmp[:, K] = Dinv  (64 x Np)
__global__ void gj_panels(const double* W, long long Np, int K0, const double* Dinv, double* Ftmp, double* Rtmp) {
    __shared__ double Ds[TB][TB + 1];
    const int b = blockIdx.y;
    const long long j0 = (long long)blockIdx.x * TB;
    const double* Wb = W + (long long)b * Np * Np;
    const double* Db = Dinv + (long long)b * TILE;
    double* Fb = Ftmp + (long long)b * Np * TB;
    double* Rb = Rtmp + (long long)b * TB * Np;
    for (int idx = threadIdx.x; idx < TILE; idx += blockDim.x) {
        const int r = idx / TB, c = idx % TB;
        Ds[r][c] = Db[idx];
        // column panel rows j0 + r, columns K0 + c
        Fb[(j0 + r) * TB + c] = Wb[(j0 + r) * Np + K0 + c];
    }
    __syncthreads();
    const bool pivot_block = j0 == K0;
    for (int idx = threadIdx.x; idx < TILE; idx += blockDim.x) {
        const int r = idx / TB, c = idx % TB;
        double v;
        if (pivot_block) {
            v = Ds[r][c];
        } else {
            v = 0.0;
            const double* wc = Wb + (long long)K0 * Np + j0 + c;
#pragma unroll 8
            for (int l = 0; l < TB; ++l) v += Ds[r][l] * __ldg(wc + (long long)l * Np);
        }
        Rb[(long long)r * Np + j0 + c] = v;
    }
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// W[i][j] = (i in K) ? Rtmp[i-K0][j] : ((j in K) ? 0 : W[i][j]) - sum_k Ftmp[i][k] Rtmp[k][j]
// 64x64 output tile per CTA, 256 threads, DMMA m8n8k4 (warp tile 32x16).
__global__ void __launch_bounds__(256) gj_update(double* W, long long Np, int K0, const double* Ftmp,
                                                 const double* Rtmp) {
    constexpr int KH = TB / 2;
    __shared__ double Fs[TB][KH + 4];  // [i][k]
    __shared__ double Rs[TB][KH + 4];  // [j][k] (transposed)
    const int b = blockIdx.z;
    const long long i0 = (long long)blockIdx.y * TB, j0 = (long long)blockIdx.x * TB;
    double* Wb = W + (long long)b * Np * Np;
    const double* Rb = Rtmp + (long long)b * TB * Np;
    if (i0 == K0) {
        for (int idx = threadIdx.x; idx < TILE; idx += blockDim.x) {
            const int r = idx / TB, c = idx % TB;
            Wb[(i0 + r) * Np + j0 + c] = Rb[(long long)r * Np + j0 + c];
        }
        return;
    }
    const double* Fb = Ftmp + (long long)b * Np * TB;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm0 = (warp & 1) * 32, wn0 = (warp >> 1) * 16;
    double acc[4][2][2] = {};
    for (int kh = 0; kh < TB; kh += KH) {
        __syncthreads();
        for (int idx = threadIdx.x; idx < TB * KH; idx += blockDim.x) {
            const int r = idx / KH, k = idx % KH;
            Fs[r][k] = Fb[(i0 + r) * TB + kh + k];
            const int k2 = idx / TB, c = idx % TB;
            Rs[c][k2] = Rb[(long long)(kh + k2) * Np + j0 + c];
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < KH / 4; ++kk) {
            double av[4], bv[2];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) av[mi] = Fs[wm0 + 8 * mi + g][4 * kk + t];
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) bv[ni] = Rs[wn0 + 8 * ni + g][4 * kk + t];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni], av[mi], bv[ni]);
        }
    }
    const bool pivot_col = j0 == K0;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const long long i = i0 + wm0 + 8 * mi + g;
                const long long j = j0 + wn0 + 8 * ni + 2 * t + c;
                double* p = Wb + i * Np + j;
                *p = (pivot_col ? 0.0 : *p) - acc[mi][ni][c];
            }
}

// Pack the lower-triangular 64x64 tiles of each inverse, zeroing padded rows/columns.
__global__ void pack_tiles(const double* W, long long Np, int n2, int ld2, long long T, double* Hout, float* Hfout) {
    const int b = blockIdx.y;
    const double* Wb = W + (long long)b * Np * Np;
    double* Hb = Hout + (long long)b * T * TILE;
    float* Hfb = Hfout + (long long)b * T * TILE;
    for (long long t = blockIdx.x; t < T; t += gridDim.x) {
        int bi, bj;
        tile_coords(t, bi, bj);
        for (int idx = threadIdx.x; idx < TILE; idx += blockDim.x) {
            const int r = idx / TB, c = idx % TB;
            const long long i = (long long)bi * TB + r, j = (long long)bj * TB + c;
            const bool pad = (int)(i % ld2) >= n2 || (int)(j % ld2) >= n2;
            const double v = pad ? 0.0 : Wb[i * Np + j];
            Hb[t * TILE + idx] = v;
            Hfb[t * TILE + idx] = (float)v;
        }
    }
}

__global__ void fwd_rhs_kernel(long long Np, int S, const double* D1, const double* b, const double* q, double eta,
                               const double* rho, const double* f, double* z) {
    // z_s = b_{s-1} D1_s o rho + eta q_s f   (system.cpp:209-210), padded layout, levels 0..S-1
    const long long n = (long long)S * Np;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        const int s = (int)(idx / Np);
        const long long i = idx % Np;
        z[idx] = b[s] * (D1[idx] * rho[i]) + eta * q[s] * f[i];
    }
}

template <typename T>
int apply_smem_bytes() {
    return NST * TILE * (int)sizeof(T) + 2 * NCW * TB * (int)sizeof(double) + NCW * 32 * (int)sizeof(double) +
           2 * NST * (int)sizeof(uint64_t);
}

__global__ void axpy_kernel(double* y, const double* d, long long n, const int* skip) {
    if (skip && *skip) return;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] += d[i];
}

template <typename T>
void launch_sweep(fi_ctx* ctx, fi_precond* P, const T* H, const double* z, double* y, int levels, int refine_f,
                  const int* skip) {
    static bool configured = false;
    const int smem = apply_smem_bytes<T>();
    if (!configured) {
        FI_CUDA(cudaFuncSetAttribute(precond_apply_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        configured = true;
    }
    const fi_system* sys = P->sys;
    ApplyArgs a;
    a.H = H;
    a.T = P->T;
    a.nb = P->nb;
    a.levels = levels;
    a.S = sys->L.S;
    a.n2 = sys->L.n2;
    a.ld2 = sys->L.ld2;
    a.Np = sys->L.Np;
    a.z = z;
    a.y = y;
    a.D1 = sys->D1.p;
    a.d2inv = P->d2inv.p;
    a.e = sys->e.p;
    a.xbuf = P->xbuf.p;
    a.pbuf = P->pbuf.p;
    a.bar = P->bar.p;
    a.skip = skip;
    a.refine_f = refine_f;
    a.n1 = sys->L.n1;
    a.gen_stride = 2 * sys->L.ld2 + 8;
    a.gen = sys->gen.p;
    a.cr = sys->cr;
    FI_CUDA(cudaMemsetAsync(P->bar.p, 0, sizeof(unsigned), ctx->stream));
    void* args[] = {&a};
    FI_CUDA(cudaLaunchCooperativeKernel((const void*)precond_apply_kernel<T>, dim3(P->G), dim3(APPLY_THREADS), args,
                                        (size_t)smem, ctx->stream));
    FI_LAUNCHED(ctx);
}

}  // namespace

void precond_apply(fi_ctx* ctx, fi_precond* P, const double* z, double* y, int levels, const int* skip) {
    const fi_system* sys = P->sys;
    const bool full = levels == sys->L.S + 1;
    // sweep 1: forward block substitution with the FP64 inverses (+ f-block refinement in-kernel)
    launch_sweep<double>(ctx, P, P->H.p, z, y, levels, full ? 1 : 0, skip);
    if (!P->refine) return;
    // one step of iterative refinement: r = z - P y on all levels at once with K1,
    // d = P^{-1} r with the FP32 copy of the inverses (|d| ~ 1e-12 |y|: FP32 is ample), y += d
    if (!full) FI_CUDA(cudaMemsetAsync(y + (long long)sys->L.S * sys->L.Np, 0, sys->L.Np * sizeof(double), ctx->stream));
    toeplitz_apply(ctx, sys->view(), y, P->rbuf.p, skip, z, true);
    launch_sweep<float>(ctx, P, P->Hf.p, P->rbuf.p, P->dbuf.p, levels, 0, skip);
    const long long n = (long long)levels * sys->L.Np;
    axpy_kernel<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(y, P->dbuf.p, n, skip);
    FI_LAUNCHED(ctx);
}

void precond_build(fi_precond* P) {
    fi_system* sys = P->sys;
    fi_ctx* ctx = sys->ctx;
    const Layout& L = sys->L;
    const int S = L.S;
    const long long N = L.N, Np = L.Np;
    const double e0 = sys->e_h[0];

    // --- block admissibility in the reference's level order (krylov.cpp:35-45).  A level whose
    // D2 vanishes identically has G_s = e0 D1 (diagonal); otherwise D2 must be nonzero with
    // D1/D2 >= 0 so that M = cs B + e0 diag(D1/D2) is symmetric positive definite.
    std::vector<double> diag((size_t)S * Np, 0.0), d2inv((size_t)S * Np, 0.0), bscale((size_t)S + 1, sys->cs);
    bscale[(size_t)S] = sys->cr;
    for (int s = 1; s <= S; ++s) {
        bool all_zero = true;
        for (long long j = 0; j < N; ++j) all_zero = all_zero && sys->D2_h[(size_t)(s - 1) * N + j] == 0.0;
        if (all_zero) bscale[(size_t)s - 1] = 0.0;
        for (long long j = 0; j < N; ++j) {
            const long long i1 = j / L.n2, i2 = j % L.n2;
            const long long p = (long long)(s - 1) * Np + i1 * L.ld2 + i2;
            const double d1 = sys->D1_h[(size_t)(s - 1) * N + j], d2 = sys->D2_h[(size_t)(s - 1) * N + j];
            if (all_zero) {
                if (d1 == 0.0 || e0 == 0.0)
                    throw Error(FI_E_SINGULAR, "precond_build: singular block at time level " + std::to_string(s), s);
                diag[p] = e0 * d1;
                d2inv[p] = 1.0;
                continue;
            }
            if (d2 == 0.0) {
                if (d1 == 0.0 || e0 == 0.0)
                    throw Error(FI_E_SINGULAR, "precond_build: singular block at time level " + std::to_string(s), s);
                throw Error(FI_E_DOMAIN, "precond_build: gamma2 vanishes at part of level " + std::to_string(s) +
                                             "; the symmetric block form needs gamma2 != 0 or gamma2 == 0 everywhere");
            }
            if (d1 / d2 < 0.0)
                throw Error(FI_E_DOMAIN, "precond_build: gamma1/gamma2 < 0 at level " + std::to_string(s) +
                                             "; the symmetric block form needs gamma1/gamma2 >= 0");
            diag[p] = e0 * d1 / d2;
            d2inv[p] = 1.0 / d2;
        }
    }
    for (long long j = 0; j < N; ++j)
        if (sys->D2_h[(size_t)(S - 1) * N + j] == 0.0)
            throw Error(FI_E_SINGULAR, "precond_build: singular block at time level " + std::to_string(S + 1), S + 1);

    P->nb = (int)(Np / TB);
    P->T = (long long)P->nb * (P->nb + 1) / 2;
    P->levels = S + 1;
    P->H.alloc((size_t)(S + 1) * P->T * TILE);
    P->Hf.alloc((size_t)(S + 1) * P->T * TILE);
    P->rbuf.alloc((size_t)L.nI());
    P->dbuf.alloc((size_t)L.nI());
    P->d2inv.alloc((size_t)S * Np);
    P->xbuf.alloc((size_t)Np);
    P->pbuf.alloc((size_t)P->nb * P->nb * TB);
    P->bar.alloc(1);
    FI_CUDA(cudaMemcpyAsync(P->d2inv.p, d2inv.data(), d2inv.size() * sizeof(double), cudaMemcpyHostToDevice,
                            ctx->stream));
    DevBuf<double> diag_d((size_t)S * Np), bscale_d((size_t)S + 1);
    FI_CUDA(cudaMemcpyAsync(diag_d.p, diag.data(), diag.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    FI_CUDA(cudaMemcpyAsync(bscale_d.p, bscale.data(), bscale.size() * sizeof(double), cudaMemcpyHostToDevice,
                            ctx->stream));

    // cooperative grid: one CTA per SM, never more than the work needs
    {
        int per_sm = 0;
        FI_CUDA(cudaFuncSetAttribute(precond_apply_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     apply_smem_bytes<double>()));
        FI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, precond_apply_kernel<double>, APPLY_THREADS,
                                                              apply_smem_bytes<double>()));
        if (per_sm < 1) throw Error(FI_E_CUDA, "precond_apply kernel cannot be resident");
        const long long want = std::max<long long>(P->T, (Np + 31) / 32);
        P->G = (int)std::min<long long>((long long)ctx->sm_count * per_sm, std::max<long long>(1, want));
        P->G = std::min(P->G, ctx->sm_count);
    }

    // --- batched Gauss-Jordan inversion of M_L for all levels
    const size_t mat = (size_t)Np * Np;
    size_t free_b = 0, total_b = 0;
    FI_CUDA(cudaMemGetInfo(&free_b, &total_b));
    long long batch = (long long)std::min<size_t>(16, std::max<size_t>(1, (free_b / 4) / (mat * sizeof(double))));
    batch = std::min<long long>(batch, S + 1);
    DevBuf<double> W((size_t)batch * mat), Ftmp((size_t)batch * Np * TB), Rtmp((size_t)batch * TB * Np),
        Dinv((size_t)batch * TILE), piv((size_t)batch * 2);
    std::vector<double> piv_h((size_t)batch * 2);
    const OperatorView op = sys->view();
    int first_singular = 0;
    for (long long l0 = 0; l0 < S + 1; l0 += batch) {
        const int nbt = (int)std::min<long long>(batch, S + 1 - l0);
        for (int b = 0; b < nbt; ++b) {
            piv_h[2 * b] = INFINITY;
            piv_h[2 * b + 1] = 0.0;
        }
        FI_CUDA(cudaMemcpyAsync(piv.p, piv_h.data(), 2 * nbt * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        FillArgs fa{op, W.p, (int)l0, diag_d.p, bscale_d.p};
        gj_fill<<<dim3((unsigned)std::min<long long>(4096, (Np * Np + 255) / 256), nbt), 256, 0, ctx->stream>>>(fa);
        FI_LAUNCHED(ctx);
        for (int K = 0; K < P->nb; ++K) {
            const int K0 = K * TB;
            gj_diag_inv<<<nbt, 256, 0, ctx->stream>>>(W.p, Np, K0, Dinv.p, piv.p);
            FI_LAUNCHED(ctx);
            gj_panels<<<dim3(P->nb, nbt), 256, 0, ctx->stream>>>(W.p, Np, K0, Dinv.p, Ftmp.p, Rtmp.p);
            FI_LAUNCHED(ctx);
            gj_update<<<dim3(P->nb, P->nb, nbt), 256, 0, ctx->stream>>>(W.p, Np, K0, Ftmp.p, Rtmp.p);
            FI_LAUNCHED(ctx);
        }
        pack_tiles<<<dim3((unsigned)std::min<long long>(P->T, 4096), nbt), 256, 0, ctx->stream>>>(
            W.p, Np, L.n2, L.ld2, P->T, P->H.p + (size_t)l0 * P->T * TILE, P->Hf.p + (size_t)l0 * P->T * TILE);
        FI_LAUNCHED(ctx);
        FI_CUDA(cudaMemcpyAsync(piv_h.data(), piv.p, 2 * nbt * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        FI_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int b = 0; b < nbt && !first_singular; ++b) {
            const double pmin = piv_h[2 * b], pmax = piv_h[2 * b + 1];
            if (!(pmax > 0.0) || !(pmin > 1e-14 * pmax)) first_singular = (int)(l0 + b) + 1;
        }
        if (first_singular)
            throw Error(FI_E_SINGULAR,
                        "precond_build: singular block at time level " + std::to_string(first_singular),
                        first_singular);
    }
}

}  // namespace fib

// forward solve helper (used by abi.cu)
namespace fib {
void forward_rhs(fi_ctx* ctx, const fi_system* sys, const double* rho_pad, const double* f_pad, double* z_pad) {
    fwd_rhs_kernel<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(sys->L.Np, sys->L.S, sys->D1.p, sys->bw.p,
                                                             sys->q.p, sys->eta, rho_pad, f_pad, z_pad);
    FI_LAUNCHED(ctx);
}
}  // namespace fib
