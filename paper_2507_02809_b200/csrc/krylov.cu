// K3/K4 — device-resident GMRES (replaces gmres(), krylov.cpp:72-209).
//
// One Arnoldi step is the operator application (K1 / the preconditioner, or the fused split step) and
// ONE cooperative kernel, mgs_step_kernel, that runs the whole rest of the step on the device:
//   * the reference's modified Gram-Schmidt (krylov.cpp:127-132): k + 2 fused rounds
//     "w -= h_{i-1} v_{i-1}; h_i = v_i . w" over the grid, each closed by a deterministic grid reduction
//     (block partials summed in the same fixed order by every CTA: bit-reproducible);
//   * the conditional second pass when ||w|| < ||w_pre|| / sqrt 2 (krylov.cpp:134-140), decided on device;
//   * h_{k+1} = ||w||, v_{k+1} = w / h_{k+1} (krylov.cpp:141-144);
//   * the Givens update, the residual history, the convergence and breakdown tests (krylov.cpp:149-185),
//     by one thread once the grid is done.
// Two drivers:
//   * solve_device (fi_gmres with the system operators): the whole solve is one CUDA graph — a conditional
//     WHILE node over restart cycles around a WHILE node over Arnoldi steps (mgs_step_kernel sets its
//     condition), an IF node for the restart residual — launched once, one host synchronisation per solve;
//   * solve (generic LinearOp callbacks, and full GMRES whose basis must grow): the host enqueues the steps
//     two ahead of the device's convergence flag, read from host-mapped memory.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>

#include "krylov.cuh"

namespace fib {
namespace {

constexpr int RT = 256;  // reduce_kernel block size
constexpr int MT = 512;  // mgs_step_kernel block size

enum ReduceMode : int {
    RM_ROUND = 1,  // out[slot] = y.w       (after w -= coef x)
    RM_NORM = 4,   // scal[slot] = w.w (no update)
};

struct ReduceArgs {
    double* w;
    const double* x;        // w -= (*coef) x   (nullptr: no update)
    const double* coef;
    const double* y;        // dot partner      (nullptr: none)
    long long n;
    int mode;
    int slot;
    double* out;
    GmresState* st;
    double* partials;       // 2 * gridDim.x
    unsigned* ticket;
    const int* done;        // skip if *done != 0
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// one fused axpy + dot/norm pass; the last block to arrive finishes the cross-block sum in fixed order
__global__ void __launch_bounds__(RT) reduce_kernel(ReduceArgs a) {
    if (a.done && *a.done) return;
    __shared__ double s1[RT / 32], s2[RT / 32];
    __shared__ bool last;
    const double alpha = a.x ? *a.coef : 0.0;
    double d = 0.0, nn = 0.0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
        double wv = a.w[i];
        if (a.x) {
            wv -= alpha * a.x[i];
            a.w[i] = wv;
        }
        if (a.y) d += a.y[i] * wv;
        nn += wv * wv;
    }
    d = warp_sum(d);
    nn = warp_sum(nn);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        s1[warp] = d;
        s2[warp] = nn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double bd = 0.0, bn = 0.0;
        for (int w = 0; w < RT / 32; ++w) {
            bd += s1[w];
            bn += s2[w];
        }
        a.partials[2 * blockIdx.x] = bd;
        a.partials[2 * blockIdx.x + 1] = bn;
        __threadfence();
        const unsigned t = atomicAdd(a.ticket, 1u);
        last = t == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double bd = 0.0, bn = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += RT) {
        bd += __ldcg(a.partials + 2 * b);
        bn += __ldcg(a.partials + 2 * b + 1);
    }
    bd = warp_sum(bd);
    bn = warp_sum(bn);
    __syncthreads();
    if (lane == 0) {
        s1[warp] = bd;
        s2[warp] = bn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double D = 0.0, Nn = 0.0;
        for (int w = 0; w < RT / 32; ++w) {
            D += s1[w];
            Nn += s2[w];
        }
        if (a.mode == RM_ROUND) a.out[a.slot] = D;
        else a.st->scal[a.slot] = Nn;
        *a.ticket = 0;
    }
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

struct MgsArgs {
    double* w;
    double* V;
    long long ldv, n;
    int k;      // >= 0: the step (host-driven); -1: st->k (device-driven)
    int maxit;
    GmresState* st;
    double* hist;
    double* parts;  // 2 parities x G x 2 block partials
    unsigned* bar;  // [0] grid-barrier counter, [1] exit counter (the last CTA out re-arms both)
    double* vcur;   // device-driven: copy of v_{k+1}, the operators' fixed input
    volatile int* done_host;
    cudaGraphConditionalHandle cond;
    int use_cond;
};

// K3 + K4: everything of Arnoldi step k after the operator application (see the file comment).
__global__ void __launch_bounds__(MT) mgs_step_kernel(MgsArgs a) {
    GmresState* st = a.st;
    if (st->done) {  // a look-ahead step past convergence (no barrier is used: the counters stay armed)
        if (a.use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(a.cond, 0u);
        return;
    }
    const int k = a.k >= 0 ? a.k : st->k;
    const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ double wsum[MT / 32][2];
    __shared__ double bres[2];
    unsigned target = 0;
    int rk = 0;
    const long long n2 = a.n >> 1, stride = (long long)G * MT, i0 = (long long)cta * MT + tid;
    double2* __restrict__ w2 = reinterpret_cast<double2*>(a.w);
    // w -= coef x (x != nullptr); returns (y . w, w . w) over the grid, identical in every CTA
    auto round = [&](const double* x, double coef, const double* y, double& dot, double& nrm) {
        const double2* __restrict__ x2 = reinterpret_cast<const double2*>(x);
        const double2* __restrict__ y2 = reinterpret_cast<const double2*>(y);
        double d = 0.0, nn = 0.0;
        long long i = i0;
        for (; i + stride < n2; i += 2 * stride) {  // two elements per thread in flight
            double2 wa = w2[i], wb = w2[i + stride];
            double2 xa = make_double2(0.0, 0.0), xb = xa, ya = xa, yb = xa;
            if (x) {
                xa = __ldg(x2 + i);
                xb = __ldg(x2 + i + stride);
            }
            if (y) {
                ya = __ldg(y2 + i);
                yb = __ldg(y2 + i + stride);
            }
            if (x) {
                wa.x -= coef * xa.x;
                wa.y -= coef * xa.y;
                wb.x -= coef * xb.x;
                wb.y -= coef * xb.y;
                w2[i] = wa;
                w2[i + stride] = wb;
            }
            d += ya.x * wa.x;
            d += ya.y * wa.y;
            d += yb.x * wb.x;
            d += yb.y * wb.y;
            nn += wa.x * wa.x;
            nn += wa.y * wa.y;
            nn += wb.x * wb.x;
            nn += wb.y * wb.y;
        }
        for (; i < n2; i += stride) {
            double2 wa = w2[i];
            if (x) {
                const double2 xa = __ldg(x2 + i);
                wa.x -= coef * xa.x;
                wa.y -= coef * xa.y;
                w2[i] = wa;
            }
            if (y) {
                const double2 ya = __ldg(y2 + i);
                d += ya.x * wa.x;
                d += ya.y * wa.y;
            }
            nn += wa.x * wa.x;
            nn += wa.y * wa.y;
        }
        if ((a.n & 1) && cta == 0 && tid == 0) {  // odd length (generic LinearOp): the last element
            const long long t = a.n - 1;
            double wv = a.w[t];
            if (x) {
                wv -= coef * x[t];
                a.w[t] = wv;
            }
            if (y) d += y[t] * wv;
            nn += wv * wv;
        }
        d = warp_sum(d);
        nn = warp_sum(nn);
        if (lane == 0) {
            wsum[warp][0] = d;
            wsum[warp][1] = nn;
        }
        __syncthreads();
        double* pp = a.parts + (size_t)(rk & 1) * G * 2;
        if (tid < 2) {
            double b = 0.0;
            for (int q = 0; q < MT / 32; ++q) b += wsum[q][tid];
            __stcg(pp + 2 * cta + tid, b);
        }
        __syncthreads();
        if (tid == 0) {
            target += (unsigned)G;
            __threadfence();
            atomicAdd(a.bar, 1u);
            unsigned n = 0;
            while (ld_relaxed_u32(a.bar) < target)
                if (++n == (1u << 28)) __trap();
            (void)ld_acquire_u32(a.bar);
        }
        __syncthreads();
        if (warp == 0) {
            // every CTA sums the G partials in the same fixed order (G <= 10 * 32)
            double pv[10][2];
#pragma unroll
            for (int u = 0; u < 10; ++u) {
                const int q = lane + 32 * u;
                pv[u][0] = q < G ? __ldcg(pp + 2 * q) : 0.0;
                pv[u][1] = q < G ? __ldcg(pp + 2 * q + 1) : 0.0;
            }
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int u = 0; u < 10; ++u) {
                s0 += pv[u][0];
                s1 += pv[u][1];
            }
            s0 = warp_sum(s0);
            s1 = warp_sum(s1);
            if (lane == 0) {
                bres[0] = s0;
                bres[1] = s1;
            }
        }
        __syncthreads();
        ++rk;
        dot = bres[0];
        nrm = bres[1];
    };
    const bool writer = cta == 0 && tid == 0;
    const double* V = a.V;
    const long long ldv = a.ldv;
    // first pass (krylov.cpp:127-132)
    double coef = 0.0, pre2 = 0.0, post2 = 0.0, dummy = 0.0;
    round(nullptr, 0.0, V, coef, pre2);
    if (writer) st->h[0] = coef;
    for (int i = 1; i <= k; ++i) {
        double hi;
        round(V + (long long)(i - 1) * ldv, coef, V + (long long)i * ldv, hi, dummy);
        coef = hi;
        if (writer) st->h[i] = hi;
    }
    round(V + (long long)k * ldv, coef, nullptr, dummy, post2);
    double nn2 = post2;
    // conditional second pass (krylov.cpp:134-140)
    const bool reorth = sqrt(post2) < sqrt(pre2) * 0.70710678118654752;
    if (writer) st->reorth = reorth ? 1 : 0;
    if (reorth) {
        round(nullptr, 0.0, V, coef, dummy);
        if (writer) st->c[0] = coef;
        for (int i = 1; i <= k; ++i) {
            double ci;
            round(V + (long long)(i - 1) * ldv, coef, V + (long long)i * ldv, ci, dummy);
            coef = ci;
            if (writer) st->c[i] = ci;
        }
        round(V + (long long)k * ldv, coef, nullptr, dummy, nn2);
        if (writer)
            for (int i = 0; i <= k; ++i) st->h[i] += st->c[i];
    }
    // v_{k+1} = w / h_{k+1} (krylov.cpp:141-144)
    const double hnext = sqrt(nn2);
    if (hnext > st->breakdown_tol) {
        const double inv = 1.0 / hnext;
        double2* __restrict__ vn = reinterpret_cast<double2*>(a.V + (long long)(k + 1) * ldv);
        double2* __restrict__ vc = reinterpret_cast<double2*>(a.vcur);
        for (long long i = i0; i < n2; i += stride) {
            const double2 wv = w2[i];
            const double2 v = make_double2(wv.x * inv, wv.y * inv);
            vn[i] = v;
            if (vc) vc[i] = v;
        }
        if ((a.n & 1) && cta == 0 && tid == 0) {
            a.V[(long long)(k + 1) * ldv + a.n - 1] = a.w[a.n - 1] * inv;
            if (a.vcur) a.vcur[a.n - 1] = a.w[a.n - 1] * inv;
        }
    }
    if (writer) {
        // Hessenberg column + Givens update (krylov.cpp:141-185)
        double* h = st->h;
        h[k + 1] = hnext;
        st->hnorm2 = nn2;
        st->vnext_ok = hnext > st->breakdown_tol ? 1 : 0;
        double col_scale = 0.0;
        for (int i = 0; i <= k + 1; ++i) col_scale = fmax(col_scale, fabs(h[i]));
        for (int i = 0; i < k; ++i) {
            const double t = st->cs[i] * h[i] + st->sn[i] * h[i + 1];
            h[i + 1] = -st->sn[i] * h[i] + st->cs[i] * h[i + 1];
            h[i] = t;
        }
        const double denom = hypot(h[k], h[k + 1]);
        if (denom <= 1e-14 * col_scale || denom == 0.0) {
            st->breakdown = 1;
            st->done = 1;
        } else {
            st->cs[k] = h[k] / denom;
            st->sn[k] = h[k + 1] / denom;
            h[k] = denom;
            double* col = st->R + (long long)k * (k + 1) / 2;  // packed: k + 1 entries
            for (int i = 0; i <= k; ++i) col[i] = h[i];
            st->g[k + 1] = -st->sn[k] * st->g[k];
            st->g[k] *= st->cs[k];
            const double relres = fabs(st->g[k + 1]) / st->bnorm;
            st->iters += 1;
            st->kc = k + 1;
            a.hist[st->iters] = relres;
            if (relres <= st->tol) {
                st->converged = 1;
                st->done = 1;
            } else if (hnext <= st->breakdown_tol) {
                st->breakdown = 1;
                st->done = 1;
            } else if (st->iters >= a.maxit) {
                st->done = 1;
            }
        }
        st->k = k + 1;
        if (st->done && a.done_host) {
            __threadfence_system();
            *a.done_host = 1;  // host-mapped: the host-driven loop stops enqueueing without a device sync
        }
        if (a.use_cond) cudaGraphSetConditional(a.cond, (!st->done && st->k < st->steps) ? 1u : 0u);
    }
    // re-arm the barrier counters for the next launch: the last CTA out resets them (every CTA has
    // finished polling when it increments the exit counter)
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(a.bar + 1, 1u) == (unsigned)G - 1) {
            a.bar[0] = 0u;
            a.bar[1] = 0u;
            __threadfence();
        }
    }
}

// Back substitution R y = g (krylov.cpp:188-197) for the kc completed columns (R packed by column).
__global__ void backsub_kernel(GmresState* st) {
    const int kc = st->kc;
    for (int i = kc - 1; i >= 0; --i) {
        double acc = st->g[i];
        for (int j = i + 1; j < kc; ++j) acc -= st->R[(long long)j * (j + 1) / 2 + i] * st->ycoef[j];
        st->ycoef[i] = acc / st->R[(long long)i * (i + 1) / 2 + i];
    }
}

// x += sum_j y_j V_j in the reference's order (krylov.cpp:198-199)
__global__ void update_x_kernel(double* x, const double* V, long long n, long long ldV, const GmresState* st) {
    const int kc = st->kc;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double xi = x[i];
        for (int j = 0; j < kc; ++j) xi += st->ycoef[j] * V[(long long)j * ldV + i];
        x[i] = xi;
    }
}

__global__ void sub_kernel(const double* b, const double* ax, double* r, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        r[i] = b[i] - ax[i];
}

// dst = src / sqrt(scal[slot]) (and a second copy when dst2 != nullptr)
__global__ void scale_by_kernel(const double* src, double* dst, double* dst2, long long n, const double* scal, int slot) {
    const double inv = 1.0 / sqrt(scal[slot]);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double v = src[i] * inv;
        dst[i] = v;
        if (dst2) dst2[i] = v;
    }
}

// ---- device-driven solve: the scalar steps between the graph's vector kernels
// after M^{-1} b (scal[0] = |M^{-1} b|^2, scal[1] = |b|^2): bnorm, the breakdown threshold
__global__ void g_norms_kernel(GmresState* st) {
    st->bnorm = sqrt(st->scal[0]);
    st->bnorm_true = sqrt(st->scal[1]);
    st->breakdown_tol = 1e-14 * st->bnorm;
}
// after r0 (scal[0] = |r0|^2 when x0 was given; |M^{-1} b|^2 otherwise): history[0], the outer condition
__global__ void g_start_kernel(GmresState* st, double* hist, cudaGraphConditionalHandle outer) {
    st->iters = 0;
    st->converged = st->breakdown = st->done = 0;
    st->flags = 0;
    if (st->bnorm == 0.0) {  // zero right-hand side (krylov.cpp:88-98)
        st->flags = 1;
        hist[0] = 0.0;
        cudaGraphSetConditional(outer, 0u);
        return;
    }
    st->beta = sqrt(st->scal[0]);
    hist[0] = st->beta / st->bnorm;
    if (st->beta / st->bnorm <= st->tol) {  // already converged (krylov.cpp:100-106)
        st->flags = 2;
        st->converged = 1;
        cudaGraphSetConditional(outer, 0u);
        return;
    }
    cudaGraphSetConditional(outer, 1u);
}
// start of a restart cycle: g = beta e_1, the step counter, the Arnoldi loop's condition
__global__ void g_cycle_kernel(GmresState* st, int cycle, int maxit, cudaGraphConditionalHandle inner) {
    st->ncycles += 1;
    st->k = 0;
    st->kc = 0;
    st->done = 0;
    st->g[0] = st->beta;
    st->steps = min(cycle, maxit - st->iters);
    cudaGraphSetConditional(inner, st->steps > 0 ? 1u : 0u);
}
// end of a cycle (after x is updated): stop, or restart from r = M^{-1}(b - A x)
__global__ void g_cycle_end_kernel(GmresState* st, int maxit, cudaGraphConditionalHandle outer,
                                   cudaGraphConditionalHandle resid) {
    const bool stop = st->converged || st->breakdown || st->iters >= maxit;
    cudaGraphSetConditional(outer, stop ? 0u : 1u);
    cudaGraphSetConditional(resid, stop ? 0u : 1u);
}
// after the restart residual (scal[0] = |r|^2): converged without a new history entry, or a new cycle
__global__ void g_restart_kernel(GmresState* st, cudaGraphConditionalHandle outer) {
    st->nresid += 1;
    const double beta = sqrt(st->scal[0]);
    st->beta = beta;
    if (beta / st->bnorm <= st->tol || beta == 0.0) {
        st->converged = 1;
        cudaGraphSetConditional(outer, 0u);
    }
}

void check_graph(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw Error(FI_E_CUDA, std::string("gmres graph: ") + what + ": " + cudaGetErrorString(e));
    }
}

}  // namespace

GmresEngine::GmresEngine(fi_ctx* ctx, long long n) : ctx_(ctx), n_(n), ldv_((n + 1) & ~1LL) {
    grid_ = ctx->sm_count * 4;
    FI_CUDA(cudaHostAlloc((void**)&done_host_, sizeof(int), cudaHostAllocMapped));
    FI_CUDA(cudaHostGetDevicePointer((void**)&done_hmap_, (void*)done_host_, 0));
    for (auto& e : iter_ev_) FI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    partials_.alloc((size_t)2 * grid_);
    ticket_.alloc(1);
    FI_CUDA(cudaMemsetAsync(ticket_.p, 0, sizeof(unsigned), ctx->stream));
    // the fused MGS step: two CTAs of MT threads per SM, all resident (cooperative launch)
    int per_sm = 0;
    FI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mgs_step_kernel, MT, 0));
    if (per_sm < 1) throw Error(FI_E_CUDA, "mgs_step_kernel cannot be resident");
    mgs_grid_ = ctx->sm_count * std::min(per_sm, 2);
    if (mgs_grid_ > 320) mgs_grid_ = 320;
    mparts_.alloc((size_t)4 * mgs_grid_);
    mbar_.alloc(2);
    FI_CUDA(cudaMemsetAsync(mbar_.p, 0, mbar_.bytes(), ctx->stream));
    st_buf_.alloc(1);
    st_ = st_buf_.p;
}

void GmresEngine::reduce(double* w, const double* x, const double* coef, const double* y, int mode, int slot,
                         const int* done) {
    ReduceArgs a;
    a.w = w;
    a.x = x;
    a.coef = coef;
    a.y = y;
    a.n = n_;
    a.mode = mode;
    a.slot = slot;
    a.out = mode == RM_ROUND ? const_cast<double*>(coef) + 16 : nullptr;
    a.st = st_;
    a.partials = partials_.p;
    a.ticket = ticket_.p;
    a.done = done;
    reduce_kernel<<<grid_, RT, 0, ctx_->stream>>>(a);
    FI_LAUNCHED(ctx_);
}

// reads a buffer larger than L2 (leaves L2 full of clean lines: a write flush would leave dirty lines
// whose write-back the timed kernel would pay for)
__global__ void flush_read_kernel(const double2* p, long long n2, double* sink) {
    double acc = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) {
        const double2 v = __ldcg(p + i);
        acc += v.x + v.y;
    }
    if (acc == 12345.678) *sink = acc;  // never true for the zero buffer: keeps the loads
}

double GmresEngine::time_mgs_round(double* w, const double* x, const double* y, int reps) {
    DevBuf<double> arr(64), flush((size_t)48 << 20);  // 384 MB: larger than L2
    cudaEvent_t e0, e1;
    FI_CUDA(cudaEventCreate(&e0));
    FI_CUDA(cudaEventCreate(&e1));
    float total = 0.f;
    FI_CUDA(cudaMemsetAsync(arr.p, 0, arr.bytes(), ctx_->stream));
    FI_CUDA(cudaMemsetAsync(flush.p, 0, flush.bytes(), ctx_->stream));
    for (int r = 0; r <= reps; ++r) {
        flush_read_kernel<<<ctx_->sm_count * 8, 256, 0, ctx_->stream>>>(reinterpret_cast<const double2*>(flush.p),
                                                                        (long long)(flush.n / 2), arr.p + 48);
        FI_CUDA(cudaEventRecord(e0, ctx_->stream));
        reduce(w, x, arr.p, y, RM_ROUND, 0, nullptr);
        FI_CUDA(cudaEventRecord(e1, ctx_->stream));
        FI_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        FI_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        if (r > 0) total += ms;  // (round 0: warm-up)
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return total / reps;
}

__global__ void fill_random_kernel(double* p, long long n, unsigned long long seed) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        unsigned long long x = (unsigned long long)i * 0x9E3779B97F4A7C15ull + seed * 0xBF58476D1CE4E5B9ull;
        x ^= x >> 30;
        x *= 0xBF58476D1CE4E5B9ull;
        x ^= x >> 27;
        x *= 0x94D049BB133111EBull;
        x ^= x >> 31;
        p[i] = (double)(x >> 11) * (2.0 / 9007199254740992.0) - 1.0;
    }
}

double GmresEngine::time_mgs_step(int k, int reps, int* reorth) {
    reserve(k + 2, false);
    ensure(w_, (size_t)n_);
    ensure(hist_, 8);
    DevBuf<double> flush((size_t)48 << 20), sink(1);  // 384 MB: larger than L2
    FI_CUDA(cudaMemsetAsync(flush.p, 0, flush.bytes(), ctx_->stream));
    fill_random_kernel<<<ctx_->sm_count * 4, 256, 0, ctx_->stream>>>(V_.p, (long long)(k + 1) * ldv_, 11);
    FI_LAUNCHED(ctx_);
    GmresState hs{};
    hs.h = h_.p;
    hs.c = c_.p;
    hs.cs = cs_.p;
    hs.sn = sn_.p;
    hs.g = g_.p;
    hs.ycoef = ycoef_.p;
    hs.R = R_.p;
    hs.bnorm = 1.0;
    hs.tol = 0.0;
    hs.breakdown_tol = 0.0;
    std::vector<double> zeros((size_t)k + 2, 0.0);
    FI_CUDA(cudaMemcpyAsync(cs_.p, zeros.data(), zeros.size() * sizeof(double), cudaMemcpyHostToDevice, ctx_->stream));
    FI_CUDA(cudaMemcpyAsync(sn_.p, zeros.data(), zeros.size() * sizeof(double), cudaMemcpyHostToDevice, ctx_->stream));
    cudaEvent_t e0, e1;
    FI_CUDA(cudaEventCreate(&e0));
    FI_CUDA(cudaEventCreate(&e1));
    float total = 0.f;
    for (int r = 0; r <= reps; ++r) {
        fill_random_kernel<<<ctx_->sm_count * 4, 256, 0, ctx_->stream>>>(w_.p, n_, 17 + r);
        FI_LAUNCHED(ctx_);
        FI_CUDA(cudaMemcpyAsync(st_, &hs, sizeof(GmresState), cudaMemcpyHostToDevice, ctx_->stream));
        flush_read_kernel<<<ctx_->sm_count * 8, 256, 0, ctx_->stream>>>(reinterpret_cast<const double2*>(flush.p),
                                                                        (long long)(flush.n / 2), sink.p);
        FI_CUDA(cudaEventRecord(e0, ctx_->stream));
        mgs_step(k, 1 << 30, false, 0);
        FI_CUDA(cudaEventRecord(e1, ctx_->stream));
        FI_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        FI_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        if (r > 0) total += ms;  // (round 0: warm-up)
    }
    GmresState out{};
    FI_CUDA(cudaMemcpy(&out, st_, sizeof(GmresState), cudaMemcpyDeviceToHost));
    if (reorth) *reorth = out.reorth;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return total / reps;
}

double GmresEngine::norm2(const double* v, int slot) {
    reduce(const_cast<double*>(v), nullptr, nullptr, nullptr, RM_NORM, slot, nullptr);
    double out = 0.0;
    FI_CUDA(cudaMemcpyAsync(&out, scal_dev(st_) + slot, sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream));
    FI_CUDA(cudaStreamSynchronize(ctx_->stream));
    return out;
}

void GmresEngine::bind_state_pointers() {
    double* ptrs[kStatePointers] = {h_.p, c_.p, cs_.p, sn_.p, g_.p, ycoef_.p, R_.p};
    FI_CUDA(cudaMemcpyAsync(st_, ptrs, sizeof(ptrs), cudaMemcpyHostToDevice, ctx_->stream));
}

void GmresEngine::reserve(int vectors, bool keep) {
    if (vectors <= cap_) return;
    const size_t nv = (size_t)vectors;
    const size_t need = nv * (size_t)ldv_ * sizeof(double);
    size_t free_b = 0, total_b = 0;
    FI_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if (need > free_b + V_.bytes())
        throw Error(FI_E_RESOURCE, "gmres: Krylov basis of " + std::to_string(vectors) + " vectors (" +
                                       std::to_string(need) + " bytes) exceeds free device memory; use restart");
    FI_CUDA(cudaStreamSynchronize(ctx_->stream));
    auto grow = [&](DevBuf<double>& b, size_t count, size_t keep_count) {
        DevBuf<double> nb(count);
        if (keep && b.p && keep_count)
            FI_CUDA(cudaMemcpyAsync(nb.p, b.p, std::min(keep_count, b.n) * sizeof(double), cudaMemcpyDeviceToDevice,
                                    ctx_->stream));
        FI_CUDA(cudaStreamSynchronize(ctx_->stream));
        b = std::move(nb);
    };
    const size_t oc = (size_t)cap_;
    grow(V_, nv * (size_t)ldv_, oc * (size_t)ldv_);
    grow(h_, nv + 1, oc + 1);
    grow(c_, nv + 1, oc + 1);
    grow(cs_, nv + 1, oc + 1);
    grow(sn_, nv + 1, oc + 1);
    grow(g_, nv + 1, oc + 1);
    grow(ycoef_, nv, oc);
    grow(R_, nv * (nv + 1) / 2, oc * (oc + 1) / 2);
    cap_ = vectors;
    bind_state_pointers();
    if (gexec_) {  // the captured graph points at the old buffers
        cudaGraphExecDestroy(gexec_);
        cudaGraphDestroy(graph_);
        gexec_ = nullptr;
        graph_ = nullptr;
        gkey_.clear();
    }
}

void GmresEngine::mgs_step(int k, int maxit, bool graph, unsigned long long cond) {
    MgsArgs a;
    a.w = w_.p;
    a.V = V_.p;
    a.ldv = ldv_;
    a.n = n_;
    a.k = graph ? -1 : k;
    a.maxit = maxit;
    a.st = st_;
    a.hist = hist_.p;
    a.parts = mparts_.p;
    a.bar = mbar_.p;
    a.vcur = graph ? vcur_.p : nullptr;
    a.done_host = graph ? nullptr : done_hmap_;
    a.cond = (cudaGraphConditionalHandle)cond;
    a.use_cond = graph ? 1 : 0;
    void* args[] = {&a};
    FI_CUDA(cudaLaunchCooperativeKernel((const void*)mgs_step_kernel, dim3(mgs_grid_), dim3(MT), args, 0,
                                        ctx_->stream));
    FI_LAUNCHED(ctx_);
}

void GmresEngine::solve(const Op& A, const Op* M, const double* b, const double* x0, double* x, double tol, int maxit,
                        int restart, fi_gmres_report* rep, std::vector<double>& history) {
    const auto t_start = std::chrono::steady_clock::now();
    if (!(tol > 0.0)) throw Error(FI_E_DOMAIN, "gmres requires tol > 0");
    const long long n = n_;
    if (maxit <= 0) maxit = (int)std::min<long long>(n, 0x7fffffff);
    const int cycle = restart > 0 ? std::min(restart, maxit) : maxit;
    cudaStream_t s = ctx_->stream;
    const int blocks = ctx_->sm_count * 4;

    // the basis grows on demand: full GMRES (cycle = maxit = n by default) allocates as it goes
    reserve(std::min(cycle + 1, 64), true);
    ensure(w_, (size_t)n);
    ensure(t1_, (size_t)n);
    ensure(t2_, (size_t)n);
    ensure(hist_, (size_t)maxit + 1);
    GmresState hs{};
    auto upload_state = [&]() {
        hs.h = h_.p;
        hs.c = c_.p;
        hs.cs = cs_.p;
        hs.sn = sn_.p;
        hs.g = g_.p;
        hs.ycoef = ycoef_.p;
        hs.R = R_.p;
        FI_CUDA(cudaMemcpyAsync(st_, &hs, sizeof(GmresState), cudaMemcpyHostToDevice, s));
    };
    auto download_state = [&]() {
        FI_CUDA(cudaMemcpyAsync(&hs, st_, sizeof(GmresState), cudaMemcpyDeviceToHost, s));
        FI_CUDA(cudaStreamSynchronize(s));
    };
    upload_state();
    auto precondition = [&](const double* in, double* out) {
        if (M) (*M)(in, out, nullptr);
        else FI_CUDA(cudaMemcpyAsync(out, in, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    };

    history.clear();
    // pb = M^{-1} b (kept in w until the first cycle scales it into V_0) ; bnorm
    double* pb = w_.p;
    precondition(b, pb);
    const double bnorm = std::sqrt(norm2(pb, 0));
    const double bnorm_true = std::sqrt(norm2(b, 1));
    if (bnorm == 0.0) {
        FI_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));
        FI_CUDA(cudaStreamSynchronize(s));
        rep->iterations = 0;
        rep->converged = 1;
        rep->breakdown = 0;
        rep->final_true_residual = 0.0;
        history.push_back(0.0);
        rep->history_len = 1;
        rep->wall_time_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
        return;
    }
    if (x0) FI_CUDA(cudaMemcpyAsync(x, x0, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    else FI_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));

    // r0 = x0 ? M^{-1}(b - A x0) : pb   (krylov.cpp:100)
    auto residual_into = [&](double* r_out) {
        A(x, t1_.p, nullptr);
        sub_kernel<<<blocks, 256, 0, s>>>(b, t1_.p, t2_.p, n);
        FI_LAUNCHED(ctx_);
        precondition(t2_.p, r_out);
    };
    if (x0) residual_into(pb);
    double beta = std::sqrt(norm2(pb, 0));
    history.push_back(beta / bnorm);

    auto finish = [&](bool converged, bool breakdown, int iters) {
        // final_true_residual = ||b - A x|| / ||b|| (krylov.cpp:205)
        A(x, t1_.p, nullptr);
        sub_kernel<<<blocks, 256, 0, s>>>(b, t1_.p, t2_.p, n);
        FI_LAUNCHED(ctx_);
        const double rn = std::sqrt(norm2(t2_.p, 1));
        rep->iterations = iters;
        rep->converged = converged || (breakdown && history.back() <= tol) ? 1 : 0;
        rep->breakdown = (breakdown && !rep->converged) ? 1 : 0;
        rep->final_true_residual = rn / bnorm_true;
        rep->history_len = (int)history.size();
        rep->wall_time_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    };
    if (beta / bnorm <= tol) {
        finish(true, false, 0);
        return;
    }

    int iters = 0;
    bool converged = false, breakdown = false;
    hs.bnorm = bnorm;
    hs.tol = tol;
    hs.breakdown_tol = 1e-14 * bnorm;
    while (true) {
        // V_0 = r0 / beta
        scale_by_kernel<<<blocks, 256, 0, s>>>(pb, V_.p, nullptr, n, scal_dev(st_), 0);
        FI_LAUNCHED(ctx_);
        hs.done = 0;
        hs.kc = 0;
        hs.iters = iters;
        hs.converged = 0;
        hs.breakdown = 0;
        upload_state();
        FI_CUDA(cudaMemcpyAsync(g_.p, &beta, sizeof(double), cudaMemcpyHostToDevice, s));
        const int steps = std::min(cycle, maxit - iters);
        const int* done = field_dev<int>(st_, offsetof(GmresState, done));
        *done_host_ = 0;
        for (int k = 0; k < steps; ++k) {
            // Look-ahead: before enqueueing step k, wait (host side) only for step k - kLook to have
            // finished and read its convergence flag from host-mapped memory.  The GPU always has
            // kLook steps queued, and at most kLook no-op steps are enqueued past convergence.
            if (k >= kLook) {
                FI_CUDA(cudaEventSynchronize(iter_ev_[k % kLook]));
                if (*(volatile int*)done_host_) break;
            }
            if (k + 2 > cap_) {  // step k writes v_{k+1}: grow the basis (full GMRES)
                FI_CUDA(cudaStreamSynchronize(s));
                if (*(volatile int*)done_host_) break;
                reserve(std::min(cycle + 1, 2 * cap_), true);
            }
            const double* vk = V_.p + (long long)k * ldv_;
            if (M && fused_) {
                (*fused_)(vk, w_.p, done);
            } else if (M) {
                A(vk, t1_.p, done);
                (*M)(t1_.p, w_.p, done);
            } else {
                A(vk, w_.p, done);
            }
            mgs_step(k, maxit, false, 0);
            FI_CUDA(cudaEventRecord(iter_ev_[k % kLook], s));
        }
        download_state();
        // history entries of this cycle
        if (hs.iters > iters) {
            std::vector<double> hh((size_t)(hs.iters - iters));
            FI_CUDA(cudaMemcpyAsync(hh.data(), hist_.p + iters + 1, hh.size() * sizeof(double),
                                    cudaMemcpyDeviceToHost, s));
            FI_CUDA(cudaStreamSynchronize(s));
            history.insert(history.end(), hh.begin(), hh.end());
        }
        iters = hs.iters;
        converged = hs.converged != 0;
        breakdown = hs.breakdown != 0;
        if (hs.kc > 0) {
            backsub_kernel<<<1, 1, 0, s>>>(st_);
            FI_LAUNCHED(ctx_);
            update_x_kernel<<<blocks, 256, 0, s>>>(x, V_.p, n, ldv_, st_);
            FI_LAUNCHED(ctx_);
        }
        const bool stop = converged || breakdown;
        if (stop || iters >= maxit) break;
        // restart: r = M^{-1}(b - A x)
        residual_into(pb);
        beta = std::sqrt(norm2(pb, 0));
        if (beta / bnorm <= tol || beta == 0.0) {
            converged = true;
            break;
        }
    }
    finish(converged, breakdown, iters);
}

bool GmresEngine::solve_device(const Op& A, const Op* M, const double* b, const double* x0, double* x, double tol,
                               int maxit, int restart, const std::vector<long long>& key, fi_gmres_report* rep,
                               std::vector<double>& history) {
    const auto t_start = std::chrono::steady_clock::now();
    if (!(tol > 0.0)) throw Error(FI_E_DOMAIN, "gmres requires tol > 0");
    const long long n = n_;
    if (maxit <= 0) maxit = (int)std::min<long long>(n, 0x7fffffff);
    if (restart <= 0) return false;  // full GMRES: the basis grows on demand (solve)
    const int cycle = std::min(restart, maxit);
    cudaStream_t s = ctx_->stream;
    const int blocks = ctx_->sm_count * 4;
    try {
        reserve(cycle + 1, false);
    } catch (const Error&) {
        return false;
    }
    ensure(w_, (size_t)n);
    ensure(t1_, (size_t)n);
    ensure(t2_, (size_t)n);
    ensure(vcur_, (size_t)n);
    if (hist_.n < (size_t)maxit + 1) {
        ensure(hist_, (size_t)maxit + 1);
        if (gexec_) {
            cudaGraphExecDestroy(gexec_);
            cudaGraphDestroy(graph_);
            gexec_ = nullptr;
            graph_ = nullptr;
        }
    }
    std::vector<long long> k2 = key;
    k2.insert(k2.end(), {(long long)(const void*)b, (long long)(const void*)x, (long long)(const void*)x0, maxit, cycle,
                         (long long)(M != nullptr), (long long)(fused_ != nullptr)});
    if (!gexec_ || k2 != gkey_) {
        if (gexec_) {
            cudaGraphExecDestroy(gexec_);
            cudaGraphDestroy(graph_);
            gexec_ = nullptr;
            graph_ = nullptr;
        }
        // ---- capture the solve (relaxed mode: the operators' setup calls are not stream work)
        auto precondition = [&](const double* in, double* out) {
            if (M) (*M)(in, out, nullptr);
            else FI_CUDA(cudaMemcpyAsync(out, in, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
        };
        auto norm_into = [&](const double* v, int slot) {
            ReduceArgs ra{};
            ra.w = const_cast<double*>(v);
            ra.n = n;
            ra.mode = RM_NORM;
            ra.slot = slot;
            ra.st = st_;
            ra.partials = partials_.p;
            ra.ticket = ticket_.p;
            reduce_kernel<<<grid_, RT, 0, s>>>(ra);
            FI_LAUNCHED(ctx_);
        };
        auto add_conditional = [&](cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type) -> cudaGraph_t {
            cudaStreamCaptureStatus cst;
            const cudaGraphNode_t* deps = nullptr;
            size_t ndeps = 0;
            cudaGraph_t capg;
            check_graph(cudaStreamGetCaptureInfo(s, &cst, nullptr, &capg, &deps, &ndeps), "capture info");
            cudaGraphNodeParams p = {};
            p.type = cudaGraphNodeTypeConditional;
            p.conditional.handle = h;
            p.conditional.type = type;
            p.conditional.size = 1;
            cudaGraphNode_t node;
            check_graph(cudaGraphAddNode(&node, capg, deps, ndeps, &p), "conditional node");
            check_graph(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies), "deps");
            return p.conditional.phGraph_out[0];
        };
        cudaGraph_t g;
        check_graph(cudaGraphCreate(&g, 0), "create");
        cudaGraphConditionalHandle h_outer, h_resid, h_inner;
        check_graph(cudaGraphConditionalHandleCreate(&h_outer, g, 0, cudaGraphCondAssignDefault), "outer handle");
        cudaGraph_t outer_body = nullptr, inner_body = nullptr, resid_body = nullptr;
        try {
            // top level: M^{-1} b, the norms, x, r0, the cycle loop, the final true residual
            long long l0 = ctx_->launches;
            check_graph(cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed),
                        "capture top");
            precondition(b, w_.p);
            norm_into(w_.p, 0);
            norm_into(b, 1);
            g_norms_kernel<<<1, 1, 0, s>>>(st_);
            FI_LAUNCHED(ctx_);
            if (x0) {
                FI_CUDA(cudaMemcpyAsync(x, x0, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
                A(x, t1_.p, nullptr);
                sub_kernel<<<blocks, 256, 0, s>>>(b, t1_.p, t2_.p, n);
                FI_LAUNCHED(ctx_);
                precondition(t2_.p, w_.p);
                norm_into(w_.p, 0);
            } else {
                FI_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));
            }
            g_start_kernel<<<1, 1, 0, s>>>(st_, hist_.p, h_outer);
            FI_LAUNCHED(ctx_);
            outer_body = add_conditional(h_outer, cudaGraphCondTypeWhile);
            A(x, t1_.p, nullptr);  // final true residual (krylov.cpp:205)
            sub_kernel<<<blocks, 256, 0, s>>>(b, t1_.p, t2_.p, n);
            FI_LAUNCHED(ctx_);
            norm_into(t2_.p, 2);
            check_graph(cudaStreamEndCapture(s, &g), "end top");
            glaunch_[0] = ctx_->launches - l0;
            l0 = ctx_->launches;

            // one restart cycle: V_0 = r0 / beta, the Arnoldi loop, x update, the restart residual
            check_graph(cudaGraphConditionalHandleCreate(&h_inner, outer_body, 0, cudaGraphCondAssignDefault),
                        "inner handle");
            check_graph(cudaGraphConditionalHandleCreate(&h_resid, outer_body, 0, cudaGraphCondAssignDefault),
                        "resid handle");
            check_graph(cudaStreamBeginCaptureToGraph(s, outer_body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed),
                        "capture cycle");
            scale_by_kernel<<<blocks, 256, 0, s>>>(w_.p, V_.p, vcur_.p, n, scal_dev(st_), 0);
            FI_LAUNCHED(ctx_);
            g_cycle_kernel<<<1, 1, 0, s>>>(st_, cycle, maxit, h_inner);
            FI_LAUNCHED(ctx_);
            inner_body = add_conditional(h_inner, cudaGraphCondTypeWhile);
            backsub_kernel<<<1, 1, 0, s>>>(st_);
            FI_LAUNCHED(ctx_);
            update_x_kernel<<<blocks, 256, 0, s>>>(x, V_.p, n, ldv_, st_);
            FI_LAUNCHED(ctx_);
            g_cycle_end_kernel<<<1, 1, 0, s>>>(st_, maxit, h_outer, h_resid);
            FI_LAUNCHED(ctx_);
            resid_body = add_conditional(h_resid, cudaGraphCondTypeIf);
            check_graph(cudaStreamEndCapture(s, &outer_body), "end cycle");
            glaunch_[1] = ctx_->launches - l0;
            l0 = ctx_->launches;

            // one Arnoldi step: the operators on vcur (= v_k), then the fused MGS / Givens / scale kernel
            check_graph(cudaStreamBeginCaptureToGraph(s, inner_body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed),
                        "capture step");
            if (M && fused_) {
                (*fused_)(vcur_.p, w_.p, nullptr);
            } else if (M) {
                A(vcur_.p, t1_.p, nullptr);
                (*M)(t1_.p, w_.p, nullptr);
            } else {
                A(vcur_.p, w_.p, nullptr);
            }
            mgs_step(0, maxit, true, (unsigned long long)h_inner);
            check_graph(cudaStreamEndCapture(s, &inner_body), "end step");
            glaunch_[2] = ctx_->launches - l0;
            l0 = ctx_->launches;

            // the restart residual r = M^{-1}(b - A x) and the restart decision
            check_graph(cudaStreamBeginCaptureToGraph(s, resid_body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed),
                        "capture residual");
            A(x, t1_.p, nullptr);
            sub_kernel<<<blocks, 256, 0, s>>>(b, t1_.p, t2_.p, n);
            FI_LAUNCHED(ctx_);
            precondition(t2_.p, w_.p);
            norm_into(w_.p, 0);
            g_restart_kernel<<<1, 1, 0, s>>>(st_, h_outer);
            FI_LAUNCHED(ctx_);
            check_graph(cudaStreamEndCapture(s, &resid_body), "end residual");
            glaunch_[3] = ctx_->launches - l0;
            ctx_->launches -= glaunch_[0] + glaunch_[1] + glaunch_[2] + glaunch_[3];  // counted when they run
            check_graph(cudaGraphInstantiate(&gexec_, g, 0), "instantiate");
        } catch (...) {
            cudaStreamCaptureStatus cst;
            if (cudaStreamIsCapturing(s, &cst) == cudaSuccess && cst != cudaStreamCaptureStatusNone) {
                cudaGraph_t junk = nullptr;
                cudaStreamEndCapture(s, &junk);
                if (junk) cudaGraphDestroy(junk);
            }
            cudaGetLastError();
            cudaGraphDestroy(g);
            gexec_ = nullptr;
            static const bool verbose = std::getenv("FI_GMRES_VERBOSE") != nullptr;
            if (verbose) std::fprintf(stderr, "[gmres] device-driven graph unavailable; host-driven loop\n");
            return false;
        }
        graph_ = g;
        gkey_ = k2;
    }
    // ---- run: state, one launch, one synchronisation
    GmresState hs{};
    hs.h = h_.p;
    hs.c = c_.p;
    hs.cs = cs_.p;
    hs.sn = sn_.p;
    hs.g = g_.p;
    hs.ycoef = ycoef_.p;
    hs.R = R_.p;
    hs.tol = tol;
    FI_CUDA(cudaMemcpyAsync(st_, &hs, sizeof(GmresState), cudaMemcpyHostToDevice, s));
    FI_CUDA(cudaGraphLaunch(gexec_, s));
    FI_CUDA(cudaMemcpyAsync(&hs, st_, sizeof(GmresState), cudaMemcpyDeviceToHost, s));
    FI_CUDA(cudaStreamSynchronize(s));
    // the kernels the graph ran: the top level, every cycle, every Arnoldi step, every restart residual
    ctx_->launches += glaunch_[0] + (long long)hs.ncycles * glaunch_[1] + (long long)hs.iters * glaunch_[2] +
                      (long long)hs.nresid * glaunch_[3];
    history.clear();
    if (hs.flags & 1) {  // zero right-hand side: x = 0, history {0}
        FI_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));
        FI_CUDA(cudaStreamSynchronize(s));
        rep->iterations = 0;
        rep->converged = 1;
        rep->breakdown = 0;
        rep->final_true_residual = 0.0;
        history.push_back(0.0);
        rep->history_len = 1;
        rep->wall_time_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
        return true;
    }
    history.resize((size_t)hs.iters + 1);
    FI_CUDA(cudaMemcpyAsync(history.data(), hist_.p, history.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    FI_CUDA(cudaStreamSynchronize(s));
    const bool converged = hs.converged != 0, breakdown = hs.breakdown != 0;
    rep->iterations = hs.iters;
    rep->converged = converged || (breakdown && history.back() <= tol) ? 1 : 0;
    rep->breakdown = (breakdown && !rep->converged) ? 1 : 0;
    rep->final_true_residual = std::sqrt(hs.scal[2]) / hs.bnorm_true;
    rep->history_len = (int)history.size();
    rep->wall_time_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    return true;
}

GmresEngine::~GmresEngine() {
    if (gexec_) cudaGraphExecDestroy(gexec_);
    if (graph_) cudaGraphDestroy(graph_);
    for (auto& e : iter_ev_)
        if (e) cudaEventDestroy(e);
    if (done_host_) cudaFreeHost(done_host_);
}

}  // namespace fib
