// K2h — the per-level inverses in hierarchical off-diagonal low-rank (HODLR) form, and the forward
// substitution over them.
//
// H_s = M_s^{-1} is dense, but its off-diagonal blocks are numerically low-rank: on
// config 1 a 2048 x 2048 block has rank 19 at 1e-12 ||H||, a 128 x 128 block rank 12.  With 64-row
// leaves and a binary tree over them, each internal node (left child I, right child J) stores
//   H[J, I] ~ Q V^T   (Q: |J| x 32 orthonormal, V = H[I, J] Q: |I| x 32)
// so y = H x is   y_leaf += H[leaf, leaf] x_leaf   and, per node,   y_J += Q (V^T x_I),  y_I += V (Q^T x_J).
// A row therefore needs its 64-entry leaf row and one 32-vector per ancestor node: 256 doubles
// for 64 leaves (depth 6), 8.4 MB per level instead of 67 MB of packed FP64 tiles.
//
// Compression (setup, per batch of levels, from the dense Gauss-Jordan inverses): per depth, a
// randomized range finder  Y = M Omega, Q = CGS2(Y), V = M^T Q  (M = H[J, I]).  Rank 32 against a
// numerical rank <= 19 at 1e-12 keeps the truncation near rounding level.
//
// Sweep (one persistent cooperative kernel, one CTA per 32 rows): per level, a CTA computes x of
// its rows, publishes the partial projections V^T x / Q^T x of its rows for every ancestor node
// (each value carries a level tag in its last mantissa bit, so readers poll the data itself), reads
// the other sides' partials and its leaf sibling's x, and forms y.  One cross-CTA hop per level; the whole y history of the CTA's rows stays in
// shared memory for the L1 time-convolution sums.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "precond.cuh"

namespace fib {
namespace {

constexpr int TB = 64;     // leaf rows
constexpr int RK = 32;     // rank per node
constexpr int HR = 32;     // rows per sweep CTA
constexpr int HPART = 8;   // threads per row in the sweep: 2 leaf halves + up to 6 ancestor depths
constexpr int DMAX = 6;    // tree depth supported (nb <= 64 leaves)
constexpr unsigned kSpin = 1u << 25;
constexpr int PRS = HR * 33 + 2;  // per-depth stride of the projection products (doubles; = 2 mod 16:
                                  // the 12 writers of a half-warp, 6 depths x 2 rows, hit distinct banks)
constexpr int TVS = RK + 1;       // per-depth stride of the summed projections
// y history: row-major [row][level], row stride = nlev rounded up to 2 mod 16 (even: level pairs load
// as double2; 2 mod 16: the rows of a warp write different banks)
__host__ __device__ inline int yh_stride(int nlev) { return (nlev + 13) / 16 * 16 + 2; }

// Values exchanged between CTAs carry their own arrival signal: the least significant mantissa bit
// holds the level tag ((level >> 1) & 1; buffers alternate by level parity), so a reader polls the
// value itself — no counters, no release fences.  (Costs one ulp, 2.2e-16 relative.)
__device__ __forceinline__ void st_tagged(double* p, double v, unsigned tag) {
    const unsigned long long bits = ((unsigned long long)__double_as_longlong(v) & ~1ull) | tag;
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;\n" ::"l"(p), "l"(bits) : "memory");
}
__device__ __forceinline__ unsigned long long ld_bits(const double* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Tree tables (device): per depth d (1..D) and leaf block b: node id and side (0 = I, 1 = J, -1 none)
struct Tree {
    int D, nb, nnodes;
    const int* rb_node;  // [DMAX + 1][nb]
    const int* rb_side;  // [DMAX + 1][nb]
    const int* lo;       // [nnodes] first leaf
    const int* mid;      // [nnodes] first leaf of J
    const int* hi;       // [nnodes] one past the last leaf
};

__device__ __forceinline__ double omega(int d, long long row, int k) {
    // deterministic pseudo-random test matrix (SplitMix64 finaliser -> uniform in [-1, 1))
    unsigned long long x = (unsigned long long)row * 0x9E3779B97F4A7C15ull + (unsigned long long)(k + 64 * d) * 0xBF58476D1CE4E5B9ull;
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return (double)(x >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

// out rows of the nodes at depth d (side `out_side` of each node, 64-row block blockIdx.x):
//   buf[out rows][k] = sum over the node's other side's rows c of  H[row][c] * in(c, k)
// in = Omega (mode 0) or buf of the other side (mode 1).  H is the dense inverse W (pads read as 0).
__global__ void hodlr_gemm(const double* W, long long Np, int n2, int ld2, Tree tr, int d, int out_side, int mode,
                           double* buf) {
    const int b = blockIdx.x, lvb = blockIdx.y;
    const int node = tr.rb_node[d * tr.nb + b];
    if (node < 0 || tr.rb_side[d * tr.nb + b] != out_side) return;
    const double* Wb = W + (long long)lvb * Np * Np;
    double* bf = buf + ((long long)lvb * (DMAX + 1) + d) * Np * RK;
    const int in_lo = out_side == 1 ? tr.lo[node] : tr.mid[node];
    const int in_hi = out_side == 1 ? tr.mid[node] : tr.hi[node];
    __shared__ double Wt[TB][33];
    __shared__ double Bt[32][RK + 1];
    const int tid = threadIdx.x;
    const int orow = tid >> 2, kq = (tid & 3) * 8;
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long r0 = (long long)b * TB;
    for (long long c0 = (long long)in_lo * TB; c0 < (long long)in_hi * TB; c0 += 32) {
        for (int q = tid; q < TB * 32; q += blockDim.x) {
            const int rr = q >> 5, cc = q & 31;
            const long long i = r0 + rr, j = c0 + cc;
            const bool pad = (int)(i % ld2) >= n2 || (int)(j % ld2) >= n2;
            Wt[rr][cc] = pad ? 0.0 : Wb[i * Np + j];
        }
        for (int q = tid; q < 32 * RK; q += blockDim.x) {
            const int cc = q >> 5, k = q & 31;
            const long long j = c0 + cc;
            Bt[cc][k] = mode == 0 ? ((int)(j % ld2) >= n2 ? 0.0 : omega(d, j, k)) : bf[j * RK + k];
        }
        __syncthreads();
#pragma unroll 4
        for (int cc = 0; cc < 32; ++cc) {
            const double w = Wt[orow][cc];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u] += w * Bt[cc][kq + u];
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) bf[(r0 + orow) * RK + kq + u] = acc[u];
}

// CGS2 orthonormalisation of the J-side columns of every node at depth d (in place in buf)
__global__ void hodlr_cgs2(Tree tr, int d, long long Np, double* buf, int nnodes_d, const int* nodes_d) {
    const int node = nodes_d[blockIdx.x];
    const int lvb = blockIdx.y;
    double* bf = buf + ((long long)lvb * (DMAX + 1) + d) * Np * RK;
    const long long j0 = (long long)tr.mid[node] * TB, j1 = (long long)tr.hi[node] * TB;
    __shared__ double red[8][RK];
    __shared__ double coef[RK];
    __shared__ double nrm0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    auto block_sum_vec = [&](double* v, int n) {  // sums v[0..n) over the block into coef[0..n)
        for (int i = 0; i < n; ++i) {
            double s = v[i];
            for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            if (lane == 0) red[warp][i] = s;
        }
        __syncthreads();
        if (tid < n) {
            double s = 0.0;
            for (int w = 0; w < 8; ++w) s += red[w][tid];
            coef[tid] = s;
        }
        __syncthreads();
    };
    for (int j = 0; j < RK; ++j) {
        double part[RK];
        part[0] = 0.0;
        for (long long r = j0 + tid; r < j1; r += blockDim.x) part[0] += bf[r * RK + j] * bf[r * RK + j];
        block_sum_vec(part, 1);
        if (tid == 0) nrm0 = sqrt(coef[0]);
        __syncthreads();
        for (int pass = 0; pass < 2 && j > 0; ++pass) {
            for (int i = 0; i < j; ++i) part[i] = 0.0;
            for (long long r = j0 + tid; r < j1; r += blockDim.x) {
                const double v = bf[r * RK + j];
                for (int i = 0; i < j; ++i) part[i] += bf[r * RK + i] * v;
            }
            block_sum_vec(part, j);
            for (long long r = j0 + tid; r < j1; r += blockDim.x) {
                double v = bf[r * RK + j];
                for (int i = 0; i < j; ++i) v -= coef[i] * bf[r * RK + i];
                bf[r * RK + j] = v;
            }
            __syncthreads();
        }
        part[0] = 0.0;
        for (long long r = j0 + tid; r < j1; r += blockDim.x) part[0] += bf[r * RK + j] * bf[r * RK + j];
        block_sum_vec(part, 1);
        const double nv = sqrt(coef[0]);
        // a direction already spanned (numerical rank < 32) is dropped
        const double sc = nv > 1e-13 * nrm0 && nv > 0.0 ? 1.0 / nv : 0.0;
        for (long long r = j0 + tid; r < j1; r += blockDim.x) bf[r * RK + j] *= sc;
        __syncthreads();
    }
}

// Pack the sweep layout: per level and 32-row CTA block, element (row i, part p, k) at double2
// index (k / 2) * 256 + 8 i + p: p = 0, 1 the leaf row (columns 32 p + k of the row's 64-row leaf),
// p = 2..7 the basis row of the depth-(p-1) ancestor (Q for J rows, V for I rows), 0 if none.
__global__ void hodlr_pack(const double* W, long long Np, int n2, int ld2, Tree tr, const double* buf,
                           double2* out) {
    const int c = blockIdx.x, lvb = blockIdx.y;
    const double* Wb = W + (long long)lvb * Np * Np;
    const double* bf = buf + (long long)lvb * (DMAX + 1) * Np * RK;
    double2* o = out + ((long long)lvb * (Np / HR) + c) * (RK / 2) * 256;
    const int t = threadIdx.x;  // 256 threads
    const int i = t >> 3, p = t & 7;
    const long long r = (long long)c * HR + i;
    const int b = (int)(r / TB);
    const bool prow = (int)(r % ld2) >= n2;
    double v[RK];
#pragma unroll
    for (int k = 0; k < RK; ++k) {
        double val = 0.0;
        if (!prow) {
            if (p < 2) {
                const long long col = (long long)b * TB + 32 * p + k;
                val = (int)(col % ld2) >= n2 ? 0.0 : Wb[r * Np + col];
            } else {
                const int d = p - 1;
                if (d <= tr.D && tr.rb_node[d * tr.nb + b] >= 0) val = bf[((long long)d * Np + r) * RK + k];
            }
        }
        v[k] = val;
    }
#pragma unroll
    for (int k2 = 0; k2 < RK / 2; ++k2) o[k2 * 256 + t] = make_double2(v[2 * k2], v[2 * k2 + 1]);
}

// ------------------------------------------------------------------ sweep
struct HArgs {
    const double2* hd;  // [level][cta][16][256]
    int nlev, S;
    long long Np;
    int n2, ld2;
    Tree tr;
    const double* z;
    double* y;
    const double* D1;
    const double* d2inv;
    const double* epad;  // epad[k] = e_k (0 <= k < S), zeros around
    double* xg;          // [2][Np] x of the level (leaf siblings read it), level-tagged
    double* proj;        // [2][nnodes][2 sides][slots <= nb * 2][RK] partial projections, level-tagged
    const int* skip;
    unsigned long long* trace;  // optional [8]: per-phase time sums of CTA 0 (FI_HODLR_TRACE=1)
};


__global__ void __launch_bounds__(256, 1) hodlr_sweep_kernel(HArgs a) {
    if (a.skip && *a.skip) return;
    extern __shared__ __align__(16) double sm[];
    const int nlev = a.nlev, S = a.S, D = a.tr.D, nb = a.tr.nb;
    const long long Np = a.Np;
    const int c = blockIdx.x, t = threadIdx.x;
    const int i = t >> 3, p = t & 7;
    const long long r0 = (long long)c * HR, r = r0 + i;
    const int b = (int)(r0 / TB);  // leaf block of the CTA (two CTAs per leaf)
    const bool prow = (int)(r % a.ld2) >= a.n2;
    const int maxslots = 2 * nb;
    // shared memory: y history of the CTA's rows [nlev][32], projection products, staging
    // (strides padded so that the 8 threads of a row, which differ in depth, hit different banks)
    const int LS = yh_stride(nlev);
    double* yh = sm;                               // HR x LS: y of the CTA's rows, every level
    double* pr = yh + (long long)HR * LS;          // DMAX x PRS products (row i, k) at i * 33 + k
    double* stage = pr + DMAX * PRS;               // partial projections of the other sides
    double* tvec = stage + 2 * nb * RK;            // DMAX x TVS summed projections
    double* xsb = tvec + DMAX * TVS;               // 2 x 66: x of the leaf block, halves at 0 and 33, by level parity
    double* es = xsb + 2 * (TB + 2);               // nlev + 2: L1 weights e_0.. (history sums)
    double* es1 = es + ((nlev + 3) & ~1);          // nlev + 2: the same shifted by one, es1[k] = e_{k+1}
    // per-depth node, side, slot, and the other side's CTA count
    __shared__ int s_node[DMAX + 1], s_side[DMAX + 1], s_slot[DMAX + 1], s_nother[DMAX + 1], s_ooff[DMAX + 2];
    if (t <= DMAX) {
        int node = -1, side = -1, slot = 0, nother = 0;
        if (t >= 1 && t <= D) {
            node = a.tr.rb_node[t * nb + b];
            side = a.tr.rb_side[t * nb + b];
            if (node >= 0) {
                const int lo = a.tr.lo[node], mid = a.tr.mid[node], hi = a.tr.hi[node];
                slot = side == 0 ? (int)((r0 - (long long)lo * TB) / HR) : (int)((r0 - (long long)mid * TB) / HR);
                nother = side == 0 ? (hi - mid) * (TB / HR) : (mid - lo) * (TB / HR);
            }
        }
        s_node[t] = node;
        s_side[t] = side;
        s_slot[t] = slot;
        s_nother[t] = nother;
    }
    __syncthreads();
    if (t == 0) {
        int off = 0;
        for (int d = 1; d <= DMAX; ++d) {
            s_ooff[d] = off;
            off += s_nother[d] * RK;
        }
        s_ooff[DMAX + 1] = off;  // total staged partials
    }
    __syncthreads();
    for (int q = t; q < nlev + 2; q += blockDim.x) {
        es[q] = a.epad[q];
        es1[q] = a.epad[q + 1];
    }
    __syncthreads();
    const double e1 = es[1];
    const long long lvstride = (Np / HR) * (RK / 2) * 256;
    // this thread's 32 coefficients of the current level (registers), prefetched one level ahead
    double2 cur[RK / 2], nxt[RK / 2];
    auto load_level = [&](int lv, double2* dst) {
        const double2* src = a.hd + (long long)lv * lvstride + (long long)c * (RK / 2) * 256;
#pragma unroll
        for (int k2 = 0; k2 < RK / 2; ++k2) dst[k2] = __ldg(src + k2 * 256 + t);
    };
    // the next level's coefficients in four groups at different points of the level, so that the
    // loads (L2 hits after the prefetch) never throttle a warp's issue
    auto load_quarter = [&](int lv, int q) {
        if (lv >= nlev) return;
        const double2* src = a.hd + (long long)lv * lvstride + (long long)c * (RK / 2) * 256;
#pragma unroll
        for (int k2 = 4 * q; k2 < 4 * q + 4; ++k2) nxt[k2] = __ldg(src + k2 * 256 + t);
    };
    // the other sides' partials this thread stages each level: fixed offsets within a parity block
    constexpr int MAXE = (2 * 64 * RK + 255) / 256;  // <= 2 nb RK staged values / 256 threads
    int soff[MAXE];
#pragma unroll
    for (int u = 0; u < MAXE; ++u) {
        const int e = t + u * 256;
        soff[u] = -1;
        if (e < s_ooff[DMAX + 1]) {
            int d = 1;
            while (d < DMAX && e >= s_ooff[d + 1]) ++d;
            const int le = e - s_ooff[d];
            soff[u] = (((s_node[d] * 2 + (1 - s_side[d])) * maxslots) + le / RK) * RK + le % RK;
        }
    }
    load_level(0, cur);
    double hnext = 0.0;  // (p == 0) history sum of the current level's x numerator
    double hsum = 0.0, xrow = 0.0;
    // (p == 0) z, D1, 1/D2 of the row for level lv, loaded one level ahead
    auto load_coef = [&](int lv, double& cz, double& cd1, double& cdi) {
        cz = cd1 = cdi = 0.0;
        if (p != 0 || prow || lv >= nlev) return;
        if (lv < S) {
            const long long o = (long long)lv * Np + r;
            cz = a.z[o];
            cd1 = a.D1[o];
            cdi = a.d2inv[o];
        } else {
            cz = a.z[(long long)S * Np + r];
            cdi = a.d2inv[(long long)(S - 1) * Np + r];
        }
    };
    double cz, cd1, cdi, nz, nd1, ndi;
    load_coef(0, cz, cd1, cdi);
    // (each stamp is a global read-modify-write of one thread: the phase after it carries its latency;
    // register accumulators would cost the kernel spills)
    unsigned long long tl = 0;
    auto stamp = [&](int ph) {
        if (a.trace && blockIdx.x == 0 && t == 0) {
            const unsigned long long now = clock64();
            if (tl) a.trace[ph] += now - tl;
            tl = now;
        }
    };
    for (int lv = 0; lv < nlev; ++lv) {
        stamp(7);
        const int par = lv & 1;
        const unsigned tag = (unsigned)(lv >> 1) & 1u;
        double* xs = xsb + par * (TB + 2);
        // ---- x of the CTA's rows
        if (p == 0) {
            double x = 0.0;
            if (!prow) {
                if (lv < S) {
                    const double hist = (lv >= 2 ? hnext : 0.0) + (lv >= 1 ? e1 * yh[i * LS + lv - 1] : 0.0);
                    x = (cz - cd1 * hist) * cdi;
                } else {
                    x = (cz - yh[i * LS + S - 1]) * cdi;
                }
            }
            xs[(r0 % TB) + i + (r0 % TB ? 1 : 0)] = x;
            st_tagged(a.xg + (long long)par * Np + r, x, tag);
            xrow = x;
        }
        // x of the row to its 8 threads (no block barrier: the row's threads share a warp)
        xrow = __shfl_sync(0xffffffffu, xrow, (t & 31) & ~7);
        stamp(0);
        load_quarter(lv + 1, 0);
        // ---- partial projections of the CTA's rows for every ancestor node
        if (p >= 2 && p - 1 <= D && s_node[p - 1] >= 0) {
            const double xv = xrow;
            double* pd = pr + (p - 2) * PRS + i * 33;
#pragma unroll
            for (int k2 = 0; k2 < RK / 2; ++k2) {
                pd[2 * k2] = cur[k2].x * xv;
                pd[2 * k2 + 1] = cur[k2].y * xv;
            }
        }
        __syncthreads();
        if (t < D * RK) {
            const int d = t / RK + 1, k = t % RK;
            if (s_node[d] >= 0) {
                const double* pd = pr + (d - 1) * PRS;
                double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int ii = 0; ii < HR; ++ii) s4[ii & 3] += pd[ii * 33 + k];
                const double s = (s4[0] + s4[1]) + (s4[2] + s4[3]);
                const long long slotbase = (((long long)par * a.tr.nnodes + s_node[d]) * 2 + s_side[d]) * maxslots;
                st_tagged(a.proj + (slotbase + s_slot[d]) * RK + k, s, tag);
            }
        }
        stamp(1);
        // next level's coefficients: issued here, off the publish path, consumed at the level's end;
        // the level after that is pulled into L2 now, so these register loads hit L2
        if (lv + 2 < nlev) {
            const char* pf = reinterpret_cast<const char*>(a.hd + (long long)(lv + 2) * lvstride +
                                                           (long long)c * (RK / 2) * 256);
            for (int q = t; q < (RK / 2) * 256 * 16 / 128; q += blockDim.x)
                asm volatile("prefetch.global.L2 [%0];\n" ::"l"(pf + (long long)q * 128));
        }
        load_quarter(lv + 1, 1);
        load_coef(lv + 1, nz, nd1, ndi);
        // ---- history of the next level (rows' y up to lv - 1): sum_{m <= lv-1} e_{lv+1-m} y_m
        {
            // level pairs (m, m + 1), m even, thread p takes m = 2p + 16j; weights (e_{lv+1-m}, e_{lv-m})
            // as one double2 from es (lv even) or es1 (lv odd); a lone last level m = lv - 1 separately
            double h4[4] = {0.0, 0.0, 0.0, 0.0};
            if (lv + 1 < S) {
                const double* yr = yh + i * LS;
                const double* eb = (lv & 1) ? es1 - 1 : es;  // eb + (lv - m) is 16-byte aligned
                int m = 2 * p;
                for (; m + 48 + 1 <= lv - 1; m += 64)
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const double2 yv = *reinterpret_cast<const double2*>(yr + m + 16 * u);
                        const double2 ev = *reinterpret_cast<const double2*>(eb + lv - m - 16 * u);
                        h4[u] = fma(yv.x, ev.y, fma(yv.y, ev.x, h4[u]));
                    }
                for (; m + 1 <= lv - 1; m += 16) {
                    const double2 yv = *reinterpret_cast<const double2*>(yr + m);
                    const double2 ev = *reinterpret_cast<const double2*>(eb + lv - m);
                    h4[0] = fma(yv.x, ev.y, fma(yv.y, ev.x, h4[0]));
                }
                if (((lv - 1) & 1) == 0 && lv >= 1 && 2 * p == ((lv - 1) & 15)) h4[1] += es[2] * yr[lv - 1];
            }
            double h = (h4[0] + h4[1]) + (h4[2] + h4[3]);
            h += __shfl_xor_sync(0xffffffffu, h, 1);
            h += __shfl_xor_sync(0xffffffffu, h, 2);
            h += __shfl_xor_sync(0xffffffffu, h, 4);
            hsum = h;  // (all 8 threads of the row hold the sum)
        }
        stamp(2);
        stamp(3);
        load_quarter(lv + 1, 2);
        // ---- the other sides' partials and the leaf sibling's x: load all, re-poll the ones whose
        // level tag is not current yet
        {
            const long long pbase = (long long)par * a.tr.nnodes * 2 * maxslots * RK;
            unsigned long long bv[MAXE];
            unsigned long long xb = 0;
            const long long rr = (long long)b * TB + t;
            const bool xsib = t < TB && (rr < r0 || rr >= r0 + HR);
#pragma unroll
            for (int u = 0; u < MAXE; ++u) bv[u] = soff[u] >= 0 ? ld_bits(a.proj + pbase + soff[u]) : tag;
            if (xsib) xb = ld_bits(a.xg + (long long)par * Np + rr);
            for (unsigned n = 0;; ++n) {
                bool ok = !xsib || (unsigned)(xb & 1ull) == tag;
#pragma unroll
                for (int u = 0; u < MAXE; ++u) ok = ok && (unsigned)(bv[u] & 1ull) == tag;
                if (ok) break;
                __nanosleep(32);
                if (n == kSpin) __trap();
#pragma unroll
                for (int u = 0; u < MAXE; ++u)
                    if (soff[u] >= 0 && (unsigned)(bv[u] & 1ull) != tag) bv[u] = ld_bits(a.proj + pbase + soff[u]);
                if (xsib && (unsigned)(xb & 1ull) != tag) xb = ld_bits(a.xg + (long long)par * Np + rr);
            }
#pragma unroll
            for (int u = 0; u < MAXE; ++u)
                if (soff[u] >= 0) stage[t + u * 256] = __longlong_as_double((long long)bv[u]);
            if (xsib) xs[t + (t >= 32 ? 1 : 0)] = __longlong_as_double((long long)xb);
        }
        __syncthreads();
        if (t < D * RK) {
            const int d = t / RK + 1, k = t % RK;
            double s4[4] = {0.0, 0.0, 0.0, 0.0};
            if (s_node[d] >= 0) {
                const double* st = stage + s_ooff[d] + k;
                const int no = s_nother[d];
                int j = 0;
                for (; j + 4 <= no; j += 4) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) s4[u] += st[(j + u) * RK];
                }
                for (; j < no; ++j) s4[j & 3] += st[j * RK];
            }
            tvec[(d - 1) * TVS + k] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
        }
        __syncthreads();
        stamp(4);
        load_quarter(lv + 1, 3);
        // ---- y of the CTA's rows: leaf product + low-rank terms, 8 threads per row
        // (one branch-free loop for both kinds of part, four independent FMA chains)
        double part;
        {
            const bool act = p < 2 || (p - 1 <= D && s_node[p - 1] >= 0);
            const double* src = p < 2 ? xs + 33 * p : tvec + (p - 2) * TVS;
            double q4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int k2 = 0; k2 < RK / 2; ++k2) {
                q4[(2 * k2) & 3] = fma(cur[k2].x, src[2 * k2], q4[(2 * k2) & 3]);
                q4[(2 * k2 + 1) & 3] = fma(cur[k2].y, src[2 * k2 + 1], q4[(2 * k2 + 1) & 3]);
            }
            part = act ? (q4[0] + q4[1]) + (q4[2] + q4[3]) : 0.0;
        }
        part += __shfl_xor_sync(0xffffffffu, part, 1);
        part += __shfl_xor_sync(0xffffffffu, part, 2);
        part += __shfl_xor_sync(0xffffffffu, part, 4);
        if (p == 0) {
            const double yv = prow ? 0.0 : part;
            yh[i * LS + lv] = yv;
            a.y[(long long)lv * Np + r] = yv;
            hnext = hsum;
        }
        stamp(5);
#pragma unroll
        for (int k2 = 0; k2 < RK / 2; ++k2) cur[k2] = nxt[k2];
        cz = nz;
        cd1 = nd1;
        cdi = ndi;
    }
}

// ------------------------------------------------------------------ a-posteriori accuracy check
// For every level of the batch: y = H x with the dense inverse and with the packed HODLR form for a
// fixed pseudo-random x; acc[level] += (|y_dense - y_hodlr|^2, |y_dense|^2).  Rank 32 is ample for
// the 1D BASELINE blocks; where it is not (the build checks every batch), the preconditioner falls
// back to packed tiles.
__device__ __forceinline__ double probe(long long r, int n2, int ld2) {
    return (int)(r % ld2) >= n2 ? 0.0 : omega(7, r, 3);
}
__global__ void hodlr_check_proj(const double2* hd, long long Np, int n2, int ld2, Tree tr, double* pj) {
    const int c = blockIdx.x, lvb = blockIdx.y, t = threadIdx.x;
    const int i = t >> 3, p = t & 7;
    const long long r = (long long)c * HR + i;
    const int b = (int)(r / TB);
    if (p < 2 || p - 1 > tr.D) return;
    const int d = p - 1, node = tr.rb_node[d * tr.nb + b];
    if (node < 0) return;
    const int side = tr.rb_side[d * tr.nb + b];
    const double2* o = hd + ((long long)lvb * (Np / HR) + c) * (RK / 2) * 256;
    const double xv = probe(r, n2, ld2);
    double* dst = pj + (((long long)lvb * tr.nnodes + node) * 2 + side) * RK;
    for (int k2 = 0; k2 < RK / 2; ++k2) {
        const double2 v = o[k2 * 256 + t];
        atomicAdd(dst + 2 * k2, v.x * xv);
        atomicAdd(dst + 2 * k2 + 1, v.y * xv);
    }
}
__global__ void hodlr_check_apply(const double* W, const double2* hd, long long Np, int n2, int ld2, Tree tr,
                                  const double* pj, double* acc) {
    const int c = blockIdx.x, lvb = blockIdx.y, t = threadIdx.x;
    const int i = t >> 3, p = t & 7;
    const long long r = (long long)c * HR + i;
    const int b = (int)(r / TB);
    const double* Wb = W + (long long)lvb * Np * Np;
    const double2* o = hd + ((long long)lvb * (Np / HR) + c) * (RK / 2) * 256;
    const bool prow = (int)(r % ld2) >= n2;
    double yh = 0.0, yd = 0.0;
    if (p < 2) {
        for (int k2 = 0; k2 < RK / 2; ++k2) {
            const double2 v = o[k2 * 256 + t];
            const long long c0 = (long long)b * TB + 32 * p + 2 * k2;
            yh += v.x * probe(c0, n2, ld2) + v.y * probe(c0 + 1, n2, ld2);
        }
    } else if (p - 1 <= tr.D && tr.rb_node[(p - 1) * tr.nb + b] >= 0) {
        const int d = p - 1, node = tr.rb_node[d * tr.nb + b], side = tr.rb_side[d * tr.nb + b];
        const double* tv = pj + (((long long)lvb * tr.nnodes + node) * 2 + (1 - side)) * RK;
        for (int k2 = 0; k2 < RK / 2; ++k2) {
            const double2 v = o[k2 * 256 + t];
            yh += v.x * tv[2 * k2] + v.y * tv[2 * k2 + 1];
        }
    }
    if (!prow)
        for (long long col = p; col < Np; col += HPART)
            if ((int)(col % ld2) < n2) yd += Wb[r * Np + col] * probe(col, n2, ld2);
    for (int off = 1; off < HPART; off <<= 1) {
        yh += __shfl_xor_sync(0xffffffffu, yh, off);
        yd += __shfl_xor_sync(0xffffffffu, yd, off);
    }
    if (p == 0 && !prow) {
        atomicAdd(acc + 2 * lvb, (yd - yh) * (yd - yh));
        atomicAdd(acc + 2 * lvb + 1, yd * yd);
    }
}

size_t hodlr_sweep_smem(int nlev, int nb) {
    return ((size_t)HR * yh_stride(nlev) + DMAX * PRS + 2 * (size_t)nb * RK + DMAX * TVS + 2 * (TB + 2) +
            2 * (size_t)((nlev + 3) & ~1)) *
           sizeof(double);
}

}  // namespace

// --------------------------------------------------------------------------- host side
struct HodlrData {
    int D = 0, nb = 0, nnodes = 0;
    DevBuf<int> rb_node, rb_side, lo, mid, hi, nodes_by_depth;
    std::vector<int> depth_off, depth_cnt;  // nodes of each depth in nodes_by_depth
    DevBuf<double2> hd;                     // [levels][Np/32][16][256]
    DevBuf<double> proj, xg;
    Tree tree() const {
        return Tree{D, nb, nnodes, rb_node.p, rb_side.p, lo.p, mid.p, hi.p};
    }
};

bool hodlr_supported(const Layout& L, int levels, int sm_count) {
    const long long nb = L.Np / TB;
    if (nb < 2 || nb > 64) return false;
    if (L.Np / HR > sm_count) return false;
    return hodlr_sweep_smem(levels, (int)nb) <= 227 * 1024;
}

HodlrData* hodlr_create(const Layout& L, int levels) {
    auto* h = new HodlrData();
    const int nb = (int)(L.Np / TB);
    h->nb = nb;
    std::vector<int> lo, mid, hi, dep;
    std::vector<int> rbn((size_t)(DMAX + 1) * nb, -1), rbs((size_t)(DMAX + 1) * nb, -1);
    // recursive bisection of [0, nb): node (lo, mid, hi) at depth d covers leaves lo..hi-1
    std::vector<std::array<int, 3>> stack{{0, nb, 1}};
    int D = 0;
    while (!stack.empty()) {
        auto [l, hh, d] = stack.back();
        stack.pop_back();
        if (hh - l < 2) continue;
        const int m = (l + hh) / 2;
        const int id = (int)lo.size();
        lo.push_back(l);
        mid.push_back(m);
        hi.push_back(hh);
        dep.push_back(d);
        D = std::max(D, d);
        for (int bb = l; bb < hh; ++bb) {
            rbn[(size_t)d * nb + bb] = id;
            rbs[(size_t)d * nb + bb] = bb < m ? 0 : 1;
        }
        stack.push_back({l, m, d + 1});
        stack.push_back({m, hh, d + 1});
    }
    if (D > DMAX) throw Error(FI_E_RESOURCE, "hodlr: tree too deep");
    h->D = D;
    h->nnodes = (int)lo.size();
    std::vector<int> byd;
    h->depth_off.assign(DMAX + 2, 0);
    h->depth_cnt.assign(DMAX + 2, 0);
    for (int d = 1; d <= D; ++d) {
        h->depth_off[d] = (int)byd.size();
        for (int n = 0; n < h->nnodes; ++n)
            if (dep[n] == d) byd.push_back(n);
        h->depth_cnt[d] = (int)byd.size() - h->depth_off[d];
    }
    auto up = [](DevBuf<int>& dst, const std::vector<int>& v) {
        dst.alloc(std::max<size_t>(v.size(), 1));
        FI_CUDA(cudaMemcpy(dst.p, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice));
    };
    up(h->rb_node, rbn);
    up(h->rb_side, rbs);
    up(h->lo, lo);
    up(h->mid, mid);
    up(h->hi, hi);
    up(h->nodes_by_depth, byd);
    h->hd.alloc((size_t)levels * (L.Np / HR) * (RK / 2) * 256);
    h->proj.alloc((size_t)2 * h->nnodes * 2 * (2 * nb) * RK);
    h->xg.alloc((size_t)2 * L.Np);
    return h;
}

void hodlr_destroy(HodlrData* h) { delete h; }

size_t hodlr_bytes(const HodlrData* h) { return h ? h->hd.bytes() : 0; }

// Compress the dense inverses W[0..nbt) of levels l0.. into the sweep layout.
void hodlr_compress(fi_ctx* ctx, HodlrData* h, const Layout& L, const double* W, int nbt, int l0, double* work) {
    const long long Np = L.Np;
    const Tree tr = h->tree();
    // work: nbt x (DMAX + 1) x Np x RK doubles
    for (int d = 1; d <= h->D; ++d) {
        const dim3 g((unsigned)h->nb, (unsigned)nbt);
        // (no power iteration: without re-orthonormalisation it would wash the small singular
        // directions out of Y; rank 32 against a numerical rank <= 19 needs none)
        hodlr_gemm<<<g, 256, 0, ctx->stream>>>(W, Np, L.n2, L.ld2, tr, d, 1, 0, work);  // Y_J = M Omega
        FI_LAUNCHED(ctx);
        hodlr_cgs2<<<dim3((unsigned)h->depth_cnt[d], (unsigned)nbt), 256, 0, ctx->stream>>>(
            tr, d, Np, work, h->depth_cnt[d], h->nodes_by_depth.p + h->depth_off[d]);  // Q_J
        FI_LAUNCHED(ctx);
        hodlr_gemm<<<g, 256, 0, ctx->stream>>>(W, Np, L.n2, L.ld2, tr, d, 0, 1, work);  // V_I = M^T Q_J
        FI_LAUNCHED(ctx);
    }
    hodlr_pack<<<dim3((unsigned)(Np / HR), (unsigned)nbt), 256, 0, ctx->stream>>>(
        W, Np, L.n2, L.ld2, tr, work, h->hd.p + (size_t)l0 * (Np / HR) * (RK / 2) * 256);
    FI_LAUNCHED(ctx);
}

size_t hodlr_work_doubles(const Layout& L, int nbt) { return (size_t)nbt * (DMAX + 1) * L.Np * RK; }

// Largest relative error |H x - H_hodlr x| / |H x| over the batch's levels (probe vector x).
double hodlr_check(fi_ctx* ctx, HodlrData* h, const Layout& L, const double* W, int nbt, int l0, double* work) {
    const long long Np = L.Np;
    const Tree tr = h->tree();
    const double2* hd = h->hd.p + (size_t)l0 * (Np / HR) * (RK / 2) * 256;
    double* pj = work;                                          // nbt x nnodes x 2 x RK
    double* acc = work + (size_t)nbt * h->nnodes * 2 * RK;      // nbt x 2
    FI_CUDA(cudaMemsetAsync(work, 0, ((size_t)nbt * h->nnodes * 2 * RK + 2 * nbt) * sizeof(double), ctx->stream));
    hodlr_check_proj<<<dim3((unsigned)(Np / HR), (unsigned)nbt), 256, 0, ctx->stream>>>(hd, Np, L.n2, L.ld2, tr, pj);
    FI_LAUNCHED(ctx);
    hodlr_check_apply<<<dim3((unsigned)(Np / HR), (unsigned)nbt), 256, 0, ctx->stream>>>(W, hd, Np, L.n2, L.ld2, tr,
                                                                                        pj, acc);
    FI_LAUNCHED(ctx);
    std::vector<double> hacc((size_t)2 * nbt);
    FI_CUDA(cudaMemcpyAsync(hacc.data(), acc, hacc.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    FI_CUDA(cudaStreamSynchronize(ctx->stream));
    double worst = 0.0;
    for (int q = 0; q < nbt; ++q)
        worst = std::max(worst, hacc[(size_t)2 * q + 1] > 0 ? std::sqrt(hacc[(size_t)2 * q] / hacc[(size_t)2 * q + 1]) : 0.0);
    return worst;
}

void hodlr_sweep(fi_ctx* ctx, HodlrData* h, const fi_system* sys, const double* d2inv, const double* z, double* y,
                 int levels, const int* skip) {
    const Layout& L = sys->L;
    const size_t smem = hodlr_sweep_smem(levels, h->nb);
    static size_t configured = 0;
    if (smem > configured) {
        FI_CUDA(cudaFuncSetAttribute(hodlr_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    HArgs a;
    a.hd = h->hd.p;
    a.nlev = levels;
    a.S = L.S;
    a.Np = L.Np;
    a.n2 = L.n2;
    a.ld2 = L.ld2;
    a.tr = h->tree();
    a.z = z;
    a.y = y;
    a.D1 = sys->D1.p;
    a.d2inv = d2inv;
    a.epad = sys->epad.p + kEOFF;
    a.xg = h->xg.p;
    a.proj = h->proj.p;
    a.skip = skip;
    static const bool tracing = std::getenv("FI_HODLR_TRACE") != nullptr;
    DevBuf<unsigned long long> trace;
    a.trace = nullptr;
    if (tracing) {
        trace.alloc(8);
        FI_CUDA(cudaMemsetAsync(trace.p, 0, trace.bytes(), ctx->stream));
        a.trace = trace.p;
    }
    FI_CUDA(cudaMemsetAsync(h->proj.p, 0xff, h->proj.bytes(), ctx->stream));
    FI_CUDA(cudaMemsetAsync(h->xg.p, 0xff, h->xg.bytes(), ctx->stream));
    void* args[] = {&a};
    FI_CUDA(cudaLaunchCooperativeKernel((const void*)hodlr_sweep_kernel, dim3((unsigned)(L.Np / HR)), dim3(256), args,
                                        smem, ctx->stream));
    FI_LAUNCHED(ctx);
    if (tracing) {
        unsigned long long hv[8];
        FI_CUDA(cudaMemcpyAsync(hv, trace.p, sizeof(hv), cudaMemcpyDeviceToHost, ctx->stream));
        FI_CUDA(cudaStreamSynchronize(ctx->stream));
        std::fprintf(stderr,
                     "[hodlr_sweep] kcycles/level: x %.2f | proj+release %.2f | history %.2f | wait %.2f | stage+sum %.2f | "
                     "y %.2f | loop %.2f\n",
                     hv[0] * 1e-3 / levels, hv[1] * 1e-3 / levels, hv[2] * 1e-3 / levels, hv[3] * 1e-3 / levels,
                     hv[4] * 1e-3 / levels, hv[5] * 1e-3 / levels, hv[7] * 1e-3 / levels);
    }
}

}  // namespace fib
