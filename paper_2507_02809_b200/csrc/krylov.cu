// K3/K4 — device-resident GMRES (replaces gmres(), krylov.cpp:72-209).
//
// The Arnoldi step keeps every scalar on the device:
//   * MGS rounds are fused "w -= h_{i-1} v_{i-1}; h_i = v_i . w" kernels (K3): a grid-stride
//     vector pass with warp-shuffle + block reductions, the cross-block reduction finished
//     deterministically by the last block to arrive (fixed summation order, so results are
//     bit-reproducible run to run).  The coefficient h_{i-1} is read from device memory.
//   * the reference's conditional second MGS pass (krylov.cpp:134-140) is a device flag
//     that gates the second-pass kernels;
//   * the Hessenberg column, Givens rotations, g, the residual history, convergence and
//     breakdown tests (krylov.cpp:141-185) are one single-thread kernel (K4).
// Every kernel of an enqueued iteration checks a device `done` flag, so a whole restart
// cycle is enqueued without host synchronisation; the host reads the state once per cycle.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <functional>

#include "krylov.cuh"

namespace fib {
namespace {

constexpr int RT = 256;  // reduction kernel block size

enum ReduceMode : int {
    RM_FIRST = 0,   // h[0] = v0.w ; pre_norm2 = w.w
    RM_ROUND = 1,   // out[i] = vi.w       (after w -= coef[i-1] v_{i-1})
    RM_FINAL1 = 2,  // post_norm2 = w.w ; reorth flag  (after w -= h[k] v_k)
    RM_FINAL2 = 3,  // h[i] += c[i] for i<=k ; hnorm2 = w.w  (after w -= c[k] v_k)
    RM_NORM = 4,    // scal[slot] = w.w (no update)
};

struct ReduceArgs {
    double* w;
    const double* x;        // w -= (*coef) x   (nullptr: no update)
    const double* coef;
    const double* y;        // dot partner      (nullptr: none)
    long long n;
    int mode;
    int k;                  // column index (FINAL2 adds c[0..k])
    int slot;               // RM_ROUND output index / RM_NORM scal slot
    double* out;            // RM_ROUND: array receiving the dot
    GmresState* st;
    double* partials;       // 2 * gridDim.x
    unsigned* ticket;
    const int* gate_on;     // run only if *gate_on != 0
    const int* done;        // skip if *done != 0
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

__global__ void __launch_bounds__(RT) reduce_kernel(ReduceArgs a) {
    if (a.done && *a.done) return;
    if (a.gate_on && !*a.gate_on) return;
    __shared__ double s1[RT / 32], s2[RT / 32];
    __shared__ bool last;
    const double alpha = a.x ? *a.coef : 0.0;
    double d = 0.0, nn = 0.0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(a.w) | reinterpret_cast<uintptr_t>(a.x) |
                       reinterpret_cast<uintptr_t>(a.y)) & 15) == 0;
    long long tail = 0;
    if (vec) {
        const long long n2 = a.n / 2;
        double2* w2 = reinterpret_cast<double2*>(a.w);
        const double2* x2 = reinterpret_cast<const double2*>(a.x);
        const double2* y2 = reinterpret_cast<const double2*>(a.y);
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
            double2 wv = w2[i];
            if (a.x) {
                const double2 xv = __ldg(x2 + i);
                wv.x -= alpha * xv.x;
                wv.y -= alpha * xv.y;
                w2[i] = wv;
            }
            if (a.y) {
                const double2 yv = __ldg(y2 + i);
                d += yv.x * wv.x;
                d += yv.y * wv.y;
            }
            nn += wv.x * wv.x;
            nn += wv.y * wv.y;
        }
        tail = 2 * n2;
    }
    for (long long i = tail + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
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
    // deterministic cross-block reduction: per-thread strided sums in fixed order, then a
    // fixed-order warp/block tree
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
        GmresState* st = a.st;
        switch (a.mode) {
            case RM_FIRST:
                st->h[0] = D;
                st->pre_norm2 = Nn;
                break;
            case RM_ROUND:
                a.out[a.slot] = D;
                break;
            case RM_FINAL1:
                st->hnorm2 = Nn;
                st->reorth = sqrt(Nn) < sqrt(st->pre_norm2) * 0.70710678118654752 ? 1 : 0;
                break;
            case RM_FINAL2:
                for (int i = 0; i <= a.k; ++i) st->h[i] += st->c[i];
                st->hnorm2 = Nn;
                break;
            case RM_NORM:
                st->scal[a.slot] = Nn;
                break;
        }
        *a.ticket = 0;
    }
}

// K4: Hessenberg column + Givens update for Arnoldi step k of the cycle (krylov.cpp:141-185).
__global__ void givens_kernel(GmresState* st, int k, int maxit, double* hist, volatile int* done_host) {
    if (st->done) return;
    const double hnext = sqrt(st->hnorm2);
    double* h = st->h;
    h[k + 1] = hnext;
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
        __threadfence_system();
        *done_host = 1;
        return;
    }
    st->cs[k] = h[k] / denom;
    st->sn[k] = h[k + 1] / denom;
    h[k] = denom;
    double* col = st->R + (long long)k * st->ldR;  // rotated column k holds k+1 entries
    for (int i = 0; i <= k; ++i) col[i] = h[i];
    st->g[k + 1] = -st->sn[k] * st->g[k];
    st->g[k] *= st->cs[k];
    const double relres = fabs(st->g[k + 1]) / st->bnorm;
    st->iters += 1;
    st->kc = k + 1;
    hist[st->iters] = relres;
    if (relres <= st->tol) {
        st->converged = 1;
        st->done = 1;
    } else if (hnext <= st->breakdown_tol) {
        st->breakdown = 1;
        st->done = 1;
    } else if (st->iters >= maxit) {
        st->done = 1;
    }
    if (st->done) {
        __threadfence_system();
        *done_host = 1;  // host-mapped: lets the host stop enqueueing without a device sync
    }
}

// v_{k+1} = w / h_{k+1}
__global__ void scale_kernel(const double* w, double* v, long long n, const GmresState* st) {
    if (st->done) return;
    const double inv = 1.0 / sqrt(st->hnorm2);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        v[i] = w[i] * inv;
}

// Back substitution R y = g (krylov.cpp:188-197) for the kc completed columns.
__global__ void backsub_kernel(GmresState* st) {
    const int kc = st->kc;
    for (int i = kc - 1; i >= 0; --i) {
        double acc = st->g[i];
        for (int j = i + 1; j < kc; ++j) acc -= st->R[(long long)j * st->ldR + i] * st->ycoef[j];
        st->ycoef[i] = acc / st->R[(long long)i * st->ldR + i];
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

__global__ void scale_by_kernel(const double* src, double* dst, long long n, const double* scal, int slot) {
    const double inv = 1.0 / sqrt(scal[slot]);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dst[i] = src[i] * inv;
}

}  // namespace

GmresEngine::GmresEngine(fi_ctx* ctx, long long n) : ctx_(ctx), n_(n) {
    grid_ = ctx->sm_count * 4;
    FI_CUDA(cudaHostAlloc((void**)&done_host_, sizeof(int), cudaHostAllocMapped));
    FI_CUDA(cudaHostGetDevicePointer((void**)&done_hmap_, (void*)done_host_, 0));
    for (auto& e : iter_ev_) FI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    partials_.alloc((size_t)2 * grid_);
    ticket_.alloc(1);
    FI_CUDA(cudaMemsetAsync(ticket_.p, 0, sizeof(unsigned), ctx->stream));
}

void GmresEngine::reduce(double* w, const double* x, const double* coef, const double* y, int mode, int k, int slot,
                         double* out, const int* gate_on, const int* done) {
    ReduceArgs a;
    a.w = w;
    a.x = x;
    a.coef = coef;
    a.y = y;
    a.n = n_;
    a.mode = mode;
    a.k = k;
    a.slot = slot;
    a.out = out;
    a.st = st_;
    a.partials = partials_.p;
    a.ticket = ticket_.p;
    a.gate_on = gate_on;
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
    // the state's h[] and coefficients: a scratch GmresState on the device
    DevBuf<GmresState> st(1);
    DevBuf<double> arr(64), flush((size_t)48 << 20);  // 384 MB: larger than L2
    GmresState hs{};
    hs.h = arr.p;
    hs.c = arr.p + 16;
    FI_CUDA(cudaMemsetAsync(arr.p, 0, arr.bytes(), ctx_->stream));
    FI_CUDA(cudaMemcpyAsync(st.p, &hs, sizeof(GmresState), cudaMemcpyHostToDevice, ctx_->stream));
    GmresState* keep = st_;
    st_ = st.p;
    cudaEvent_t e0, e1;
    FI_CUDA(cudaEventCreate(&e0));
    FI_CUDA(cudaEventCreate(&e1));
    float total = 0.f;
    FI_CUDA(cudaMemsetAsync(flush.p, 0, flush.bytes(), ctx_->stream));
    for (int r = 0; r <= reps; ++r) {
        flush_read_kernel<<<ctx_->sm_count * 8, 256, 0, ctx_->stream>>>(reinterpret_cast<const double2*>(flush.p),
                                                                        (long long)(flush.n / 2), arr.p + 48);
        FI_CUDA(cudaEventRecord(e0, ctx_->stream));
        reduce(w, x, arr.p, y, RM_ROUND, 1, 1, arr.p + 32, nullptr, nullptr);
        FI_CUDA(cudaEventRecord(e1, ctx_->stream));
        FI_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        FI_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        if (r > 0) total += ms;  // (round 0: warm-up)
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    st_ = keep;
    return total / reps;
}

double GmresEngine::norm2(const double* v, int slot) {
    // RM_NORM never writes w (x == nullptr)
    reduce(const_cast<double*>(v), nullptr, nullptr, nullptr, RM_NORM, 0, slot, nullptr, nullptr, nullptr);
    double out = 0.0;
    FI_CUDA(cudaMemcpyAsync(&out, scal_dev(st_) + slot, sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream));
    FI_CUDA(cudaStreamSynchronize(ctx_->stream));
    return out;
}

void GmresEngine::solve(const Op& A, const Op* M, const double* b, const double* x0, double* x, double tol, int maxit,
                        int restart, fi_gmres_report* rep, std::vector<double>& history) {
    const auto t_start = std::chrono::steady_clock::now();
    static const bool htrace = std::getenv("FI_GMRES_HOSTTRACE") != nullptr;
    auto hstamp = [&](const char* what) {
        if (htrace)
            std::fprintf(stderr, "[gmres host] %-14s %8.3f ms\n", what,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
    };
    if (!(tol > 0.0)) throw Error(FI_E_DOMAIN, "gmres requires tol > 0");
    const long long n = n_;
    if (maxit <= 0) maxit = (int)std::min<long long>(n, 0x7fffffff);
    const int cycle = restart > 0 ? std::min(restart, maxit) : maxit;
    cudaStream_t s = ctx_->stream;
    const int blocks = ctx_->sm_count * 4;

    // basis V (cycle + 1 vectors) + work vectors
    const long long ldv = (n + 1) & ~1LL;
    if (V_.n < (size_t)(cycle + 1) * ldv) {
        // (only when the workspace must grow: cudaMemGetInfo costs milliseconds of host time, which
        // would idle the GPU at the start of every solve)
        const size_t need = ((size_t)cycle + 1 + 3) * (size_t)n * sizeof(double);
        size_t free_b = 0, total_b = 0;
        FI_CUDA(cudaMemGetInfo(&free_b, &total_b));
        if (need > free_b + V_.bytes() + w_.bytes() + t1_.bytes() + t2_.bytes())
            throw Error(FI_E_RESOURCE, "gmres: Krylov basis of " + std::to_string(cycle + 1) + " vectors (" +
                                           std::to_string(need) + " bytes) exceeds free device memory; use restart");
    }
    // workspaces persist across solves (no cudaMalloc/cudaFree inside a timed solve)
    DevBuf<double>&V = V_, &w = w_, &t1 = t1_, &t2 = t2_, &hist_d = hist_, &arr = arr_, &ycoef = ycoef_;
    DevBuf<GmresState>& st_d = st_buf_;
    ensure(V, (size_t)(cycle + 1) * ldv);
    ensure(w, (size_t)n);
    ensure(t1, (size_t)n);
    ensure(t2, (size_t)n);
    ensure(hist_d, (size_t)maxit + 1);
    // device state
    ensure(st_d, 1);
    ensure(arr, (size_t)(cycle + 2) * 5 + (size_t)(cycle + 1) * (cycle + 1));
    GmresState hs{};
    hs.h = arr.p;
    hs.c = hs.h + (cycle + 2);
    hs.cs = hs.c + (cycle + 2);
    hs.sn = hs.cs + (cycle + 2);
    hs.g = hs.sn + (cycle + 2);
    hs.R = hs.g + (cycle + 2);
    hs.ldR = cycle + 1;
    st_ = st_d.p;
    ensure(ycoef, (size_t)cycle + 1);
    hs.ycoef = ycoef.p;

    auto upload_state = [&]() {
        FI_CUDA(cudaMemcpyAsync(st_d.p, &hs, sizeof(GmresState), cudaMemcpyHostToDevice, s));
    };
    auto download_state = [&]() {
        FI_CUDA(cudaMemcpyAsync(&hs, st_d.p, sizeof(GmresState), cudaMemcpyDeviceToHost, s));
        FI_CUDA(cudaStreamSynchronize(s));
    };
    hstamp("workspaces");
    upload_state();
    hstamp("upload_state");

    auto precondition = [&](const double* in, double* out) {
        if (M) (*M)(in, out, nullptr);
        else FI_CUDA(cudaMemcpyAsync(out, in, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    };

    history.clear();
    // pb = M^{-1} b ; bnorm
    double* pb = V.p;  // V_0 receives r0 / beta below
    precondition(b, pb);
    hstamp("precondition");
    const double bnorm = std::sqrt(norm2(pb, 0));
    hstamp("bnorm");
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
        rep->wall_time_seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
        return;
    }
    if (x0) FI_CUDA(cudaMemcpyAsync(x, x0, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    else FI_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));

    // r0 = x0 ? M^{-1}(b - A x0) : pb   (krylov.cpp:100)
    auto residual_into = [&](double* r_out) {
        A(x, t1.p, nullptr);
        sub_kernel<<<blocks, 256, 0, s>>>(b, t1.p, t2.p, n);
        FI_LAUNCHED(ctx_);
        precondition(t2.p, r_out);
    };
    if (x0) residual_into(pb);
    double beta = std::sqrt(norm2(pb, 0));
    history.push_back(beta / bnorm);

    auto finish = [&](bool converged, bool breakdown, int iters) {
        // final_true_residual = ||b - A x|| / ||b|| (krylov.cpp:205)
        A(x, t1.p, nullptr);
        sub_kernel<<<blocks, 256, 0, s>>>(b, t1.p, t2.p, n);
        FI_LAUNCHED(ctx_);
        const double rn = std::sqrt(norm2(t2.p, 1));
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
        scale_by_kernel<<<blocks, 256, 0, s>>>(pb, V.p, n, scal_dev(st_d.p), 0);
        FI_LAUNCHED(ctx_);
        hs.done = 0;
        hs.kc = 0;
        hs.iters = iters;
        hs.converged = 0;
        hs.breakdown = 0;
        upload_state();
        FI_CUDA(cudaMemcpyAsync(hs.g, &beta, sizeof(double), cudaMemcpyHostToDevice, s));
        const int steps = std::min(cycle, maxit - iters);
        const int* done = field_dev<int>(st_d.p, offsetof(GmresState, done));
        const int* reorth = field_dev<int>(st_d.p, offsetof(GmresState, reorth));
        *done_host_ = 0;
        for (int k = 0; k < steps; ++k) {
            // Look-ahead: before enqueueing step k, wait (host side) only for step k - kLook to have
            // finished and read its convergence flag from host-mapped memory.  The GPU always has
            // kLook steps queued, and at most kLook no-op steps are enqueued past convergence.
            if (k >= kLook) {
                FI_CUDA(cudaEventSynchronize(iter_ev_[k % kLook]));
                if (*(volatile int*)done_host_) break;
            }
            const double* vk = V.p + (long long)k * ldv;
            if (M && fused_) {
                (*fused_)(vk, w.p, done);
            } else if (M) {
                A(vk, t1.p, done);
                (*M)(t1.p, w.p, done);
            } else {
                A(vk, w.p, done);
            }
            // first MGS pass (krylov.cpp:127-132)
            reduce(w.p, nullptr, nullptr, V.p, RM_FIRST, k, 0, nullptr, nullptr, done);
            for (int i = 1; i <= k; ++i)
                reduce(w.p, V.p + (long long)(i - 1) * ldv, hs.h + (i - 1), V.p + (long long)i * ldv, RM_ROUND, k, i,
                       hs.h, nullptr, done);
            reduce(w.p, V.p + (long long)k * ldv, hs.h + k, nullptr, RM_FINAL1, k, 0, nullptr, nullptr, done);
            // conditional second pass (krylov.cpp:134-140)
            reduce(w.p, nullptr, nullptr, V.p, RM_ROUND, k, 0, hs.c, reorth, done);
            for (int i = 1; i <= k; ++i)
                reduce(w.p, V.p + (long long)(i - 1) * ldv, hs.c + (i - 1), V.p + (long long)i * ldv, RM_ROUND, k, i,
                       hs.c, reorth, done);
            reduce(w.p, V.p + (long long)k * ldv, hs.c + k, nullptr, RM_FINAL2, k, 0, nullptr, reorth, done);
            givens_kernel<<<1, 1, 0, s>>>(st_d.p, k, maxit, hist_d.p, done_hmap_);
            FI_LAUNCHED(ctx_);
            scale_kernel<<<blocks, 256, 0, s>>>(w.p, V.p + (long long)(k + 1) * ldv, n, st_d.p);
            FI_LAUNCHED(ctx_);
            FI_CUDA(cudaEventRecord(iter_ev_[k % kLook], s));
        }
        download_state();
        // history entries of this cycle
        if (hs.iters > iters) {
            std::vector<double> hh((size_t)(hs.iters - iters));
            FI_CUDA(cudaMemcpyAsync(hh.data(), hist_d.p + iters + 1, hh.size() * sizeof(double),
                                    cudaMemcpyDeviceToHost, s));
            FI_CUDA(cudaStreamSynchronize(s));
            history.insert(history.end(), hh.begin(), hh.end());
        }
        iters = hs.iters;
        converged = hs.converged != 0;
        breakdown = hs.breakdown != 0;
        if (hs.kc > 0) {
            backsub_kernel<<<1, 1, 0, s>>>(st_d.p);
            FI_LAUNCHED(ctx_);
            update_x_kernel<<<blocks, 256, 0, s>>>(x, V.p, n, ldv, st_d.p);
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

}  // namespace fib

namespace fib {
GmresEngine::~GmresEngine() {
    for (auto& e : iter_ev_)
        if (e) cudaEventDestroy(e);
    if (done_host_) cudaFreeHost(done_host_);
}
}  // namespace fib
