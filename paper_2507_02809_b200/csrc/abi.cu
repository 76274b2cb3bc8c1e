// C-ABI entry points (include/fracinv_b200.h).  Every call converts library exceptions
// into status codes; the message and SingularBlockError time index are kept per host
// thread (fi_last_error, fi_last_error_time_index).
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "krylov.cuh"
#include "precond.cuh"

namespace fib {
double gamma_fn(double x);
void l1_weights(double beta, int S, double* b, double* e);
void time_grid(double beta, int S, double T, double* dt, double* eta);
void symbol_coeffs_1d(double omega, int n, double* coeffs);
void symbol_coeffs_md(double omega, int d, const int* n, long long sample_cap, double* coeffs);
void symbol_coeffs_2d_dev(fi_ctx* ctx, double omega, int n1, int n2, long long sample_cap, double* coeffs);
void assemble_dense(fi_ctx* ctx, const fi_system* sys, int kind, long long cap, double* M);
void add_noise(const double* mu, long long n, double eps, uint64_t seed, double* out);
void add_gaussian_noise(const double* mu, long long n, double rel_eps, uint64_t seed, double* out);
}  // namespace fib

namespace {

thread_local std::string g_err;
thread_local int g_time_index = 0;

template <class F>
int guard(F&& f) {
    try {
        f();
        g_err.clear();
        g_time_index = 0;
        return FI_OK;
    } catch (const fib::Error& e) {
        g_err = e.what();
        g_time_index = e.time_index;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        g_time_index = 0;
        return FI_E_RESOURCE;
    } catch (const std::exception& e) {
        g_err = e.what();
        g_time_index = 0;
        return FI_E_CUDA;
    }
}

void require(bool ok, int code, const std::string& msg) {
    if (!ok) throw fib::Error(code, msg);
}

// every context-bound entry point runs on the context's device, whatever the calling thread's
// current device is (a host thread may drive contexts on several devices)
void bind(const fi_ctx* ctx) {
    if (ctx) FI_CUDA(cudaSetDevice(ctx->device));
}

__global__ void pack_kernel(const double* ref, double* pad, long long total, long long Np, long long N, int n2,
                            int ld2) {
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long s = idx / Np, i = idx % Np;
        const long long i1 = i / ld2, i2 = i % ld2;
        pad[idx] = i2 < n2 ? ref[s * N + i1 * n2 + i2] : 0.0;
    }
}

__global__ void unpack_kernel(const double* pad, double* ref, long long total, long long Np, long long N, int n2,
                              int ld2) {
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long s = idx / N, j = idx % N;
        const long long i1 = j / n2, i2 = j % n2;
        ref[idx] = pad[s * Np + i1 * ld2 + i2];
    }
}

void pack_levels(fi_ctx* ctx, const fib::Layout& L, const double* ref, double* pad, int levels) {
    const long long total = (long long)levels * L.Np;
    pack_kernel<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(ref, pad, total, L.Np, L.N, L.n2, L.ld2);
    FI_LAUNCHED(ctx);
}

void unpack_levels(fi_ctx* ctx, const fib::Layout& L, const double* pad, double* ref, int levels) {
    const long long total = (long long)levels * L.N;
    unpack_kernel<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(pad, ref, total, L.Np, L.N, L.n2, L.ld2);
    FI_LAUNCHED(ctx);
}

// mode: 0 = dense inverses (the reference's per-block direct solve), 1 = tau-PCG per block,
//       -1 = automatic: dense up to the cap; above it, tau-PCG for 2D (the reference raises
//       ResourceLimitError there), ResourceLimitError for 1D as in the reference.
fi_precond* build_precond(fi_system* sys, long long block_cap, int mode = -1, double tol = 1e-14, int maxit = 200) {
    if (block_cap <= 0) block_cap = 4096;  // BlockTriangularPreconditioner::kDefaultBlockCap
    if (mode < 0) mode = (sys->L.N > block_cap && fib::iterative_supported(sys->L)) ? 1 : 0;
    if (mode == 0 && sys->L.N > block_cap)
        throw fib::Error(FI_E_RESOURCE, "BlockTriangularPreconditioner: block dimension " + std::to_string(sys->L.N) +
                                            " exceeds cap " + std::to_string(block_cap));
    if (mode == 1 && !(sys->omega > 0.0))
        throw fib::Error(FI_E_DOMAIN, "tau-PCG preconditioner needs fi_system_desc.omega");
    fi_precond* P = new fi_precond();
    P->sys = sys;
    static std::atomic<unsigned long long> next_uid{1};
    P->uid = next_uid++;
    try {
        if (mode == 1) fib::precond_build_iterative(P, tol, maxit);
        else fib::precond_build(P);
        P->zbuf.alloc((size_t)sys->L.nI());
        P->ybuf.alloc((size_t)sys->L.nI());
        FI_CUDA(cudaStreamSynchronize(sys->ctx->stream));
    } catch (...) {
        delete P;
        throw;
    }
    return P;
}

}  // namespace

namespace fib {
void ensure_smem_attr(const void* func, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> set;  // (device, kernel) -> bytes allowed
    int dev = 0;
    FI_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    size_t& have = set[{dev, func}];
    if (bytes <= have) return;
    FI_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    have = bytes;
}

void pack_vector(fi_ctx* ctx, const Layout& L, const double* ref, double* pad) { pack_levels(ctx, L, ref, pad, L.S + 1); }
void unpack_vector(fi_ctx* ctx, const Layout& L, const double* pad, double* ref) {
    unpack_levels(ctx, L, pad, ref, L.S + 1);
}
}  // namespace fib

extern "C" {

// ------------------------------------------------------------------ context
int fi_ctx_create(int device, fi_ctx** out) {
    return guard([&] {
        require(out != nullptr, FI_E_DOMAIN, "fi_ctx_create: out is NULL");
        int count = 0;
        FI_CUDA(cudaGetDeviceCount(&count));
        require(device >= 0 && device < count, FI_E_CUDA, "fi_ctx_create: no CUDA device " + std::to_string(device));
        FI_CUDA(cudaSetDevice(device));
        fi_ctx* c = new fi_ctx();
        c->device = device;
        FI_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
        FI_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        FI_CUDA(cudaEventCreate(&c->ev0));
        FI_CUDA(cudaEventCreate(&c->ev1));
        FI_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
        FI_CUDA(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming));
        FI_CUDA(cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming));
        *out = c;
    });
}

void fi_ctx_destroy(fi_ctx* ctx) {
    if (!ctx || --ctx->refs > 0) return;
    cudaStreamSynchronize(ctx->stream);
    cudaEventDestroy(ctx->ev0);
    cudaEventDestroy(ctx->ev1);
    cudaEventDestroy(ctx->fork);
    cudaEventDestroy(ctx->join);
    cudaStreamDestroy(ctx->side);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
}

void* fi_ctx_stream(fi_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int fi_ctx_synchronize(fi_ctx* ctx) {
    return guard([&] {
        require(ctx != nullptr, FI_E_DOMAIN, "fi_ctx_synchronize: NULL context");
        bind(ctx);
        FI_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

const char* fi_last_error(void) { return g_err.c_str(); }
int fi_last_error_time_index(void) { return g_time_index; }
long long fi_ctx_kernel_launches(fi_ctx* ctx) { return ctx ? ctx->launches : 0; }

// ------------------------------------------------------------------ host setup numerics
int fi_gamma(double x, double* out) {
    return guard([&] { *out = fib::gamma_fn(x); });
}
int fi_l1_weights(double beta, int S, double* b, double* e) {
    return guard([&] { fib::l1_weights(beta, S, b, e); });
}
int fi_time_grid(double beta, int S, double T, double* dt, double* eta) {
    return guard([&] { fib::time_grid(beta, S, T, dt, eta); });
}
int fi_symbol_coeffs_1d(double omega, int n, double* coeffs) {
    return guard([&] { fib::symbol_coeffs_1d(omega, n, coeffs); });
}
int fi_symbol_coeffs_md(double omega, int d, const int* n, long long sample_cap, double* coeffs) {
    return guard([&] { fib::symbol_coeffs_md(omega, d, n, sample_cap <= 0 ? (1LL << 26) : sample_cap, coeffs); });
}
int fi_symbol_coeffs_md_dev(fi_ctx* ctx, double omega, int d, const int* n, long long sample_cap, double* coeffs) {
    return guard([&] {
        require(ctx && n && coeffs, FI_E_DOMAIN, "fi_symbol_coeffs_md_dev: NULL argument");
        bind(ctx);
        const long long cap = sample_cap <= 0 ? (1LL << 26) : sample_cap;
        if (d == 2) fib::symbol_coeffs_2d_dev(ctx, omega, n[0], n[1], cap, coeffs);
        else fib::symbol_coeffs_md(omega, d, n, cap, coeffs);  // d = 1: the host sum (1D uses the recursion)
    });
}
int fi_add_gaussian_noise(const double* mu, long long n, double rel_eps, unsigned long long seed, double* out) {
    return guard([&] { fib::add_gaussian_noise(mu, n, rel_eps, seed, out); });
}
int fi_add_noise(const double* mu, long long n, double eps, unsigned long long seed, double* out) {
    return guard([&] { fib::add_noise(mu, n, eps, seed, out); });
}

// ------------------------------------------------------------------ system
int fi_system_create(fi_ctx* ctx, const fi_system_desc* desc, fi_system** out) {
    return guard([&] {
        require(ctx && desc && out, FI_E_DOMAIN, "fi_system_create: NULL argument");
        require(desc->d == 1 || desc->d == 2, FI_E_DOMAIN, "fi_system_create: d must be 1 or 2");
        require(desc->n[0] >= 1 && (desc->d == 1 || desc->n[1] >= 1), FI_E_DOMAIN, "fi_system_create: n_i >= 1");
        require(desc->S >= 1, FI_E_DOMAIN, "fi_system_create: S >= 1");
        require(desc->gen && desc->e && desc->b && desc->q && desc->D1 && desc->D2, FI_E_DOMAIN,
                "fi_system_create: NULL array");
        const int S = desc->S;
        for (int s = 1; s <= S; ++s)
            require(desc->q[s - 1] > 0.0, FI_E_DOMAIN,
                    "q(t) must be positive at every time level, violated at s = " + std::to_string(s));
        bind(ctx);
        fi_system* sys = new fi_system();
        try {
            sys->ctx = ctx;
            sys->L = fib::make_layout(desc->d, desc->n, S);
            const fib::Layout& L = sys->L;
            sys->h = desc->h;
            sys->eta = desc->eta;
            sys->cs = desc->scale_space;
            sys->cr = desc->scale_reg;
            sys->omega = desc->omega;
            const int n1 = L.n1, n2 = L.n2;
            const size_t gsz = (size_t)(2 * n1 - 1) * (2 * n2 - 1);
            sys->gen_h.assign(desc->gen, desc->gen + gsz);
            sys->e_h.assign(desc->e, desc->e + S);
            sys->b_h.assign(desc->b, desc->b + S);
            sys->q_h.assign(desc->q, desc->q + S);
            sys->D1_h.assign(desc->D1, desc->D1 + (size_t)S * L.N);
            sys->D2_h.assign(desc->D2, desc->D2 + (size_t)S * L.N);
            // padded generating tensor: row r = l1 + n1 - 1, a[l1][l2] at column l2 + ld2
            const int gs = 2 * L.ld2 + 8;
            std::vector<double> gpad((size_t)(2 * n1 - 1) * gs, 0.0);
            for (int r = 0; r < 2 * n1 - 1; ++r)
                for (int l2 = -(n2 - 1); l2 <= n2 - 1; ++l2)
                    gpad[(size_t)r * gs + l2 + L.ld2] = sys->gen_h[(size_t)r * (2 * n2 - 1) + l2 + n2 - 1];
            std::vector<double> epad((size_t)fib::kEOFF + S + 256, 0.0);
            for (int k = 0; k < S; ++k) epad[(size_t)fib::kEOFF + k] = sys->e_h[(size_t)k];
            std::vector<double> D1p((size_t)S * L.Np, 0.0), D2p((size_t)S * L.Np, 0.0);
            for (int s = 0; s < S; ++s)
                for (long long j = 0; j < L.N; ++j) {
                    const long long p = (long long)s * L.Np + (j / n2) * L.ld2 + j % n2;
                    D1p[(size_t)p] = sys->D1_h[(size_t)s * L.N + j];
                    D2p[(size_t)p] = sys->D2_h[(size_t)s * L.N + j];
                }
            auto up = [&](fib::DevBuf<double>& buf, const std::vector<double>& v) {
                buf.alloc(v.size());
                FI_CUDA(cudaMemcpy(buf.p, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice));
            };
            up(sys->gen, gpad);
            up(sys->epad, epad);
            up(sys->D1, D1p);
            up(sys->D2, D2p);
            up(sys->q, sys->q_h);
            up(sys->e, sys->e_h);
            up(sys->bw, sys->b_h);
            sys->ubuf.alloc((size_t)L.nI());
            sys->zbuf.alloc((size_t)L.nI());
            FI_CUDA(cudaMemset(sys->ubuf.p, 0, sys->ubuf.bytes()));
            // operator realisation: FI_APPLY=dmma|fft overrides the default (AUTO: K1f where supported)
            sys->fft_ok = fib::fft_apply_supported(L);
            if (const char* m = std::getenv("FI_APPLY")) {
                if (std::string(m) == "dmma") sys->apply_mode = FI_APPLY_DMMA;
                else if (std::string(m) == "fft") sys->apply_mode = FI_APPLY_FFT;
            }
            if (sys->use_fft()) fib::fft_apply_prepare(sys);
        } catch (...) {
            delete sys;
            throw;
        }
        ctx->refs++;
        *out = sys;
    });
}

void fi_system_destroy(fi_system* sys) {
    if (!sys || --sys->refs > 0) return;
    fi_ctx* ctx = sys->ctx;
    cudaStreamSynchronize(ctx->stream);
    delete sys->engine;
    delete sys;
    fi_ctx_destroy(ctx);
}

long long fi_system_dim(const fi_system* sys) { return sys ? sys->L.nRef() : 0; }
long long fi_system_space_dim(const fi_system* sys) { return sys ? sys->L.N : 0; }

int fi_system_apply(fi_system* sys, const double* y_dev, double* z_dev) {
    return guard([&] {
        require(sys && y_dev && z_dev, FI_E_DOMAIN, "fi_system_apply: NULL argument");
        bind(sys->ctx);
        fi_ctx* ctx = sys->ctx;
        fib::pack_vector(ctx, sys->L, y_dev, sys->ubuf.p);
        fib::system_apply(ctx, sys, sys->ubuf.p, sys->zbuf.p, nullptr);
        fib::unpack_vector(ctx, sys->L, sys->zbuf.p, z_dev);
    });
}

int fi_system_apply_host(fi_system* sys, const double* y_host, double* z_host) {
    return guard([&] {
        require(sys && y_host && z_host, FI_E_DOMAIN, "fi_system_apply_host: NULL argument");
        bind(sys->ctx);
        fi_ctx* ctx = sys->ctx;
        const size_t bytes = (size_t)sys->L.nRef() * sizeof(double);
        fib::DevBuf<double> y((size_t)sys->L.nRef()), z((size_t)sys->L.nRef());
        FI_CUDA(cudaMemcpyAsync(y.p, y_host, bytes, cudaMemcpyHostToDevice, ctx->stream));
        fib::pack_vector(ctx, sys->L, y.p, sys->ubuf.p);
        fib::system_apply(ctx, sys, sys->ubuf.p, sys->zbuf.p, nullptr);
        fib::unpack_vector(ctx, sys->L, sys->zbuf.p, z.p);
        FI_CUDA(cudaMemcpyAsync(z_host, z.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        FI_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int fi_system_apply_timed(fi_system* sys, const double* y_dev, double* z_dev, int reps, double* ms_avg) {
    return guard([&] {
        require(sys && y_dev && z_dev && ms_avg && reps > 0, FI_E_DOMAIN, "fi_system_apply_timed: bad argument");
        bind(sys->ctx);
        fi_ctx* ctx = sys->ctx;
        fib::pack_vector(ctx, sys->L, y_dev, sys->ubuf.p);
        fib::system_apply(ctx, sys, sys->ubuf.p, sys->zbuf.p, nullptr);  // warm-up
        FI_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
        for (int r = 0; r < reps; ++r) fib::system_apply(ctx, sys, sys->ubuf.p, sys->zbuf.p, nullptr);
        FI_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
        FI_CUDA(cudaEventSynchronize(ctx->ev1));
        float ms = 0.f;
        FI_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        *ms_avg = ms / reps;
        fib::unpack_vector(ctx, sys->L, sys->zbuf.p, z_dev);
        FI_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// ------------------------------------------------------------------ preconditioner
int fi_precond_create(fi_system* sys, long long block_cap, fi_precond** out) {
    return guard([&] {
        require(sys && out, FI_E_DOMAIN, "fi_precond_create: NULL argument");
        bind(sys->ctx);
        *out = build_precond(sys, block_cap);
        sys->refs++;
    });
}

int fi_precond_create_ex(fi_system* sys, long long block_cap, int inner, double tol, int maxit, fi_precond** out) {
    return guard([&] {
        require(sys && out, FI_E_DOMAIN, "fi_precond_create_ex: NULL argument");
        bind(sys->ctx);
        require(inner >= -1 && inner <= 1, FI_E_DOMAIN, "fi_precond_create_ex: inner must be -1, 0 or 1");
        require(tol > 0.0 && maxit > 0, FI_E_DOMAIN, "fi_precond_create_ex: tol > 0 and maxit > 0 required");
        *out = build_precond(sys, block_cap, inner, tol, maxit);
        sys->refs++;
    });
}

int fi_precond_inner(const fi_precond* P) { return P ? P->mode : -1; }
int fi_precond_form(const fi_precond* P) { return P ? (P->mode == 1 ? 1 : (P->hodlr ? 2 : 0)) : -1; }

void fi_precond_destroy(fi_precond* P) {
    if (!P) return;
    fi_system* sys = P->sys;
    cudaStreamSynchronize(sys->ctx->stream);
    delete P;
    fi_system_destroy(sys);
}

long long fi_precond_bytes(const fi_precond* P) {
    return P ? (long long)(P->H.bytes() + P->Hf.bytes() + fib::hodlr_bytes(P->hodlr)) : 0;
}

int fi_precond_set_refine(fi_precond* P, int refine) {
    return guard([&] {
        require(P != nullptr, FI_E_DOMAIN, "fi_precond_set_refine: NULL preconditioner");
        P->refine = refine ? 1 : 0;
    });
}

int fi_precond_apply(fi_precond* P, const double* z_dev, double* y_dev) {
    return guard([&] {
        require(P && z_dev && y_dev, FI_E_DOMAIN, "fi_precond_apply: NULL argument");
        bind(P->sys->ctx);
        fi_ctx* ctx = P->sys->ctx;
        fib::pack_vector(ctx, P->sys->L, z_dev, P->zbuf.p);
        fib::precond_apply(ctx, P, P->zbuf.p, P->ybuf.p, P->sys->L.S + 1, nullptr);
        fib::unpack_vector(ctx, P->sys->L, P->ybuf.p, y_dev);
    });
}

int fi_precond_apply_host(fi_precond* P, const double* z_host, double* y_host) {
    return guard([&] {
        require(P && z_host && y_host, FI_E_DOMAIN, "fi_precond_apply_host: NULL argument");
        bind(P->sys->ctx);
        fi_ctx* ctx = P->sys->ctx;
        const fib::Layout& L = P->sys->L;
        const size_t bytes = (size_t)L.nRef() * sizeof(double);
        unsigned long long before[4] = {0, 0, 0, 0}, after[4] = {0, 0, 0, 0};
        if (P->mode == 1) fib::precond_iterative_stats(P, before, false);
        fib::DevBuf<double> z((size_t)L.nRef()), y((size_t)L.nRef());
        FI_CUDA(cudaMemcpyAsync(z.p, z_host, bytes, cudaMemcpyHostToDevice, ctx->stream));
        fib::pack_vector(ctx, L, z.p, P->zbuf.p);
        fib::precond_apply(ctx, P, P->zbuf.p, P->ybuf.p, L.S + 1, nullptr);
        fib::unpack_vector(ctx, L, P->ybuf.p, y.p);
        FI_CUDA(cudaMemcpyAsync(y_host, y.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        FI_CUDA(cudaStreamSynchronize(ctx->stream));
        if (P->mode == 1) {
            fib::precond_iterative_stats(P, after, false);
            if (after[1] > before[1])
                throw fib::Error(FI_E_NOCONV, "precond_apply: " + std::to_string(after[1] - before[1]) +
                                                  " tau-PCG block solve(s) stopped at maxit = " +
                                                  std::to_string(P->it_maxit) + " above tol");
        }
    });
}

int fi_precond_build_check(const fi_precond* P, double out[2]) {
    return guard([&] {
        require(P && out, FI_E_DOMAIN, "fi_precond_build_check: NULL argument");
        out[0] = P->hodlr_check_fwd;
        out[1] = P->hodlr_check_bwd;
    });
}

int fi_precond_stats(fi_precond* P, long long out[4], int reset) {
    return guard([&] {
        require(P && out, FI_E_DOMAIN, "fi_precond_stats: NULL argument");
        bind(P->sys->ctx);
        unsigned long long v[4] = {0, 0, 0, 0};
        if (P->mode == 1) fib::precond_iterative_stats(P, v, reset != 0);
        for (int i = 0; i < 4; ++i) out[i] = (long long)v[i];
    });
}

int fi_precond_apply_timed(fi_precond* P, const double* z_dev, double* y_dev, int reps, double* ms_avg) {
    return guard([&] {
        require(P && z_dev && y_dev && ms_avg && reps > 0, FI_E_DOMAIN, "fi_precond_apply_timed: bad argument");
        bind(P->sys->ctx);
        fi_ctx* ctx = P->sys->ctx;
        const fib::Layout& L = P->sys->L;
        fib::pack_vector(ctx, L, z_dev, P->zbuf.p);
        fib::precond_apply(ctx, P, P->zbuf.p, P->ybuf.p, L.S + 1, nullptr);
        FI_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
        for (int r = 0; r < reps; ++r) fib::precond_apply(ctx, P, P->zbuf.p, P->ybuf.p, L.S + 1, nullptr);
        FI_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
        FI_CUDA(cudaEventSynchronize(ctx->ev1));
        float ms = 0.f;
        FI_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        *ms_avg = ms / reps;
        fib::unpack_vector(ctx, L, P->ybuf.p, y_dev);
        FI_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// ------------------------------------------------------------------ assembly helpers
int fi_build_rhs(const fi_system* sys, const double* rho_host, const double* mu_eps_host, double* z_host) {
    return guard([&] {
        require(sys && rho_host && mu_eps_host && z_host, FI_E_DOMAIN, "fi_build_rhs: NULL argument");
        const long long N = sys->L.N;
        const int S = sys->L.S;
        for (int s = 1; s <= S; ++s)
            for (long long j = 0; j < N; ++j)
                z_host[(long long)(s - 1) * N + j] =
                    sys->b_h[(size_t)s - 1] * (sys->D1_h[(size_t)(s - 1) * N + j] * rho_host[j]);
        std::memcpy(z_host + (long long)S * N, mu_eps_host, (size_t)N * sizeof(double));
    });
}

int fi_forward_solve(fi_system* sys, fi_precond* P, const double* rho_host, const double* f_host, double* states_host,
                     double* mu_host) {
    return guard([&] {
        require(sys && rho_host && f_host && mu_host, FI_E_DOMAIN, "fi_forward_solve: NULL argument");
        bind(sys->ctx);
        fi_ctx* ctx = sys->ctx;
        const fib::Layout& L = sys->L;
        fi_precond* own = nullptr;
        if (!P) {
            // forward_solve assembles its blocks regardless of the preconditioner cap
            // (system.cpp:198: dense(N)), so the temporary build uses cap = N
            own = fib::iterative_supported(L) && L.N > 4096 ? build_precond(sys, 4096) : build_precond(sys, L.N);
            P = own;
        }
        try {
            fib::DevBuf<double> rf((size_t)2 * L.N), rfp((size_t)2 * L.Np), states((size_t)L.S * L.N);
            FI_CUDA(cudaMemcpyAsync(rf.p, rho_host, L.N * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
            FI_CUDA(cudaMemcpyAsync(rf.p + L.N, f_host, L.N * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
            pack_levels(ctx, L, rf.p, rfp.p, 2);
            fib::forward_rhs(ctx, sys, rfp.p, rfp.p + L.Np, P->zbuf.p);
            fib::precond_apply(ctx, P, P->zbuf.p, P->ybuf.p, L.S, nullptr);
            unpack_levels(ctx, L, P->ybuf.p, states.p, L.S);
            if (states_host)
                FI_CUDA(cudaMemcpyAsync(states_host, states.p, (size_t)L.S * L.N * sizeof(double),
                                        cudaMemcpyDeviceToHost, ctx->stream));
            FI_CUDA(cudaMemcpyAsync(mu_host, states.p + (long long)(L.S - 1) * L.N, L.N * sizeof(double),
                                    cudaMemcpyDeviceToHost, ctx->stream));
            FI_CUDA(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            delete own;
            throw;
        }
        delete own;
    });
}

// ------------------------------------------------------------------ GMRES
static void copy_history(const std::vector<double>& h, double* out, int cap) {
    if (!out) return;
    const int m = std::min<int>(cap, (int)h.size());
    for (int i = 0; i < m; ++i) out[i] = h[(size_t)i];
}

int fi_gmres(fi_system* sys, fi_precond* P, const double* b_dev, const double* x0_dev, double* x_dev,
             const fi_gmres_opts* opts, fi_gmres_report* report, double* history_host, int history_cap) {
    return guard([&] {
        require(sys && b_dev && x_dev && opts && report, FI_E_DOMAIN, "fi_gmres: NULL argument");
        bind(sys->ctx);
        require(!P || P->sys == sys, FI_E_DIM, "fi_gmres: preconditioner belongs to another system");
        fi_ctx* ctx = sys->ctx;
        const fib::Layout& L = sys->L;
        const long long n = L.nI();
        if (sys->gb.n < (size_t)n) {
            sys->gb.alloc((size_t)n);
            sys->gx.alloc((size_t)n);
        }
        fib::DevBuf<double>& b = sys->gb;
        fib::DevBuf<double>& x = sys->gx;
        fib::DevBuf<double>& x0 = sys->gx0;
        fib::pack_vector(ctx, L, b_dev, b.p);
        if (x0_dev) {
            if (x0.n < (size_t)n) x0.alloc((size_t)n);
            fib::pack_vector(ctx, L, x0_dev, x0.p);
        }
        fib::Op A = [ctx, sys](const double* in, double* out, const int* skip) {
            fib::system_apply(ctx, sys, in, out, skip);
        };
        fib::Op M = [ctx, P](const double* in, double* out, const int* skip) {
            fib::precond_apply(ctx, P, in, out, P->sys->L.S + 1, skip);
        };
        // maxit = 0 selects the matrix dimension (krylov.hpp:56), i.e. the reference's n
        const int maxit = opts->maxit > 0 ? opts->maxit : (int)std::min<long long>(L.nRef(), 0x7fffffff);
        if (!sys->engine) sys->engine = new fib::GmresEngine(ctx, n);
        // optional split apply: P^{-1} A v = v + P^{-1}((A - P) v), one sweep per Arnoldi step
        static const bool split_env = !(std::getenv("FI_SPLIT_APPLY") && std::atoi(std::getenv("FI_SPLIT_APPLY")) == 0);
        const bool split = split_env && sys->split_apply;
        fib::Op Fz = [ctx, P, sys](const double* in, double* out, const int* skip) {
            fib::precond_times_operator(ctx, P, in, out, sys->sp_u.p, sys->sp_t.p, skip);
        };
        if (split && P) {
            if (sys->sp_u.n < (size_t)n) {
                sys->sp_u.alloc((size_t)n);
                sys->sp_t.alloc((size_t)n);
            }
        }
        sys->engine->set_fused(split && P ? &Fz : nullptr);
        std::vector<double> hist;
        if (P && P->mode == 1) FI_CUDA(cudaMemsetAsync(P->it_stats.p, 0, P->it_stats.bytes(), ctx->stream));
        // device-driven (one CUDA graph per solve, one host synchronisation) unless the restart cycle's
        // basis does not fit or full GMRES was asked for (its basis grows on demand: host-driven loop)
        static const bool device_env = !(std::getenv("FI_GMRES_DEVICE") && std::atoi(std::getenv("FI_GMRES_DEVICE")) == 0);
        const std::vector<long long> key = {(long long)(P ? P->uid : 0), P ? P->refine : -1, split ? 1 : 0, sys->use_fft() ? 1 : 0,
                                            (long long)(P ? P->mode : -1)};
        const bool done = device_env && sys->engine->solve_device(A, P ? &M : nullptr, b.p, x0_dev ? x0.p : nullptr,
                                                                  x.p, opts->tol, maxit, opts->restart, key, report,
                                                                  hist);
        if (!done)
            sys->engine->solve(A, P ? &M : nullptr, b.p, x0_dev ? x0.p : nullptr, x.p, opts->tol, maxit,
                               opts->restart, report, hist);
        sys->engine->set_fused(nullptr);
        report->inner_nonconverged = 0;
        if (P && P->mode == 1) {
            unsigned long long st[4];
            fib::precond_iterative_stats(P, st, false);
            report->inner_nonconverged = (int)st[1];
        }
        fib::unpack_vector(ctx, L, x.p, x_dev);
        FI_CUDA(cudaStreamSynchronize(ctx->stream));
        copy_history(hist, history_host, history_cap);
    });
}

int fi_mgs_round_timed(fi_ctx* ctx, long long n, double* w_dev, const double* x_dev, const double* y_dev, int reps,
                       double* ms_avg) {
    return guard([&] {
        require(ctx && w_dev && x_dev && y_dev && ms_avg && n > 0 && reps > 0, FI_E_DOMAIN,
                "fi_mgs_round_timed: bad argument");
        bind(ctx);
        fib::GmresEngine eng(ctx, n);
        *ms_avg = eng.time_mgs_round(w_dev, x_dev, y_dev, reps);
    });
}

int fi_mgs_step_timed(fi_ctx* ctx, long long n, int k, int reps, double* ms_avg, int* reorth) {
    return guard([&] {
        require(ctx && ms_avg && n > 0 && k >= 0 && reps > 0, FI_E_DOMAIN, "fi_mgs_step_timed: bad argument");
        bind(ctx);
        fib::GmresEngine eng(ctx, n);
        *ms_avg = eng.time_mgs_step(k, reps, reorth);
    });
}

int fi_assemble_dense(fi_system* sys, int kind, long long cap, double* M_dev) {
    return guard([&] {
        require(sys && M_dev, FI_E_DOMAIN, "fi_assemble_dense: NULL argument");
        bind(sys->ctx);
        fib::assemble_dense(sys->ctx, sys, kind, cap <= 0 ? 4096 : cap, M_dev);
    });
}

int fi_system_set_apply_mode(fi_system* sys, int mode) {
    return guard([&] {
        require(sys, FI_E_DOMAIN, "fi_system_set_apply_mode: NULL system");
        require(mode == FI_APPLY_AUTO || mode == FI_APPLY_DMMA || mode == FI_APPLY_FFT, FI_E_DOMAIN,
                "fi_system_set_apply_mode: unknown mode");
        require(mode != FI_APPLY_FFT || sys->fft_ok, FI_E_DOMAIN,
                "fi_system_set_apply_mode: the FFT apply needs a 2D grid with n_i + 1 a power of two");
        bind(sys->ctx);
        sys->apply_mode = mode;
        if (sys->use_fft()) fib::fft_apply_prepare(sys);
    });
}

int fi_system_get_apply_mode(const fi_system* sys) {
    if (!sys) return -1;
    return sys->use_fft() ? FI_APPLY_FFT : FI_APPLY_DMMA;
}

int fi_system_set_split_apply(fi_system* sys, int on) {
    return guard([&] {
        require(sys, FI_E_DOMAIN, "fi_system_set_split_apply: NULL system");
        sys->split_apply = on ? 1 : 0;
    });
}

int fi_gmres_host(fi_system* sys, fi_precond* P, const double* b_host, const double* x0_host, double* x_host,
                  const fi_gmres_opts* opts, fi_gmres_report* report, double* history_host, int history_cap) {
    int rc = FI_OK;
    int rc2 = guard([&] {
        require(sys && b_host && x_host, FI_E_DOMAIN, "fi_gmres_host: NULL argument");
        bind(sys->ctx);
        fi_ctx* ctx = sys->ctx;
        const size_t n = (size_t)sys->L.nRef();
        // staging for the reference-layout host vectors: [b | x | x0], kept across calls
        if (sys->gio.n < 3 * n) sys->gio.alloc(3 * n);
        double* b = sys->gio.p;
        double* x = b + n;
        double* x0 = x + n;
        FI_CUDA(cudaMemcpyAsync(b, b_host, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        if (x0_host)
            FI_CUDA(cudaMemcpyAsync(x0, x0_host, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        rc = fi_gmres(sys, P, b, x0_host ? x0 : nullptr, x, opts, report, history_host, history_cap);
        if (rc != FI_OK) throw fib::Error(rc, g_err, g_time_index);
        FI_CUDA(cudaMemcpyAsync(x_host, x, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        FI_CUDA(cudaStreamSynchronize(ctx->stream));
    });
    return rc2;
}

int fi_gmres_op(fi_ctx* ctx, long long n, fi_linop_fn apply_A, void* user_A, fi_linop_fn apply_M, void* user_M,
                const double* b_dev, const double* x0_dev, double* x_dev, const fi_gmres_opts* opts,
                fi_gmres_report* report, double* history_host, int history_cap) {
    return guard([&] {
        require(ctx && apply_A && b_dev && x_dev && opts && report && n > 0, FI_E_DOMAIN, "fi_gmres_op: bad argument");
        bind(ctx);
        fib::Op A = [apply_A, user_A](const double* in, double* out, const int*) {
            if (apply_A(user_A, in, out) != 0) throw fib::Error(FI_E_DOMAIN, "fi_gmres_op: apply_A callback failed");
        };
        fib::Op M = [apply_M, user_M](const double* in, double* out, const int*) {
            if (apply_M(user_M, in, out) != 0) throw fib::Error(FI_E_DOMAIN, "fi_gmres_op: apply_M callback failed");
        };
        const int maxit = opts->maxit > 0 ? opts->maxit : (int)std::min<long long>(n, 0x7fffffff);
        fib::GmresEngine eng(ctx, n);
        std::vector<double> hist;
        eng.solve(A, apply_M ? &M : nullptr, b_dev, x0_dev, x_dev, opts->tol, maxit, opts->restart, report, hist);
        report->inner_nonconverged = 0;
        FI_CUDA(cudaStreamSynchronize(ctx->stream));
        copy_history(hist, history_host, history_cap);
    });
}

}  // extern "C"
