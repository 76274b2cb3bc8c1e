// fracinv_b200.hpp — header-only C++ façade over the C-ABI (fracinv_b200.h), mirroring the
// reference library's API (/root/reference/proj/include/fracinv/{system,krylov,errors}.hpp) so a
// reference user switches by changing the include and namespace:
//
//   fracinv::SystemOperator A(spec);                      ->  fracinv::b200::SystemOperator A(ctx, spec);
//   fracinv::BlockTriangularPreconditioner P(A);          ->  fracinv::b200::BlockTriangularPreconditioner P(A);
//   auto [y, rep] = fracinv::gmres(opA, opP, z, {tol});   ->  auto [y, rep] = fracinv::b200::gmres(A, &P, z, {tol, 0, 50});
//
// Errors are rethrown as the reference's exception types.  Vectors are std::vector<double> in
// the reference's stacked layout (block s at (s-1)*N, f last).
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fracinv_b200.h"

namespace fracinv {
namespace b200 {

// ------------------------------------------------------------------ errors (errors.hpp:9-43)
class DimensionError : public std::invalid_argument {
public:
    using std::invalid_argument::invalid_argument;
};
class ResourceLimitError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class SingularBlockError : public std::runtime_error {
public:
    SingularBlockError(const std::string& what, int time_index) : std::runtime_error(what), time_index_(time_index) {}
    int time_index() const noexcept { return time_index_; }

private:
    int time_index_;
};
class ConfigError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
// EXTENSION: a tau-PCG block solve stopped at maxit above its tolerance (FI_E_NOCONV)
class NoConvergenceError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class CudaError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

inline void check(int rc) {
    if (rc == FI_OK) return;
    const std::string msg = fi_last_error();
    switch (rc) {
        case FI_E_DIM: throw DimensionError(msg);
        case FI_E_RESOURCE: throw ResourceLimitError(msg);
        case FI_E_SINGULAR: throw SingularBlockError(msg, fi_last_error_time_index());
        case FI_E_DOMAIN: throw std::domain_error(msg);
        case FI_E_CONFIG: throw ConfigError(msg);
        case FI_E_NOCONV: throw NoConvergenceError(msg);
        default: throw CudaError(msg);
    }
}

// ------------------------------------------------------------------ context
class Context {
public:
    explicit Context(int device = 0) { check(fi_ctx_create(device, &h_)); }
    ~Context() { fi_ctx_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    fi_ctx* handle() const noexcept { return h_; }
    void synchronize() const { check(fi_ctx_synchronize(h_)); }

private:
    fi_ctx* h_ = nullptr;
};

// ------------------------------------------------------------------ problem (system.hpp:26-55)
using SpaceTimeField = std::function<double(const std::vector<double>& x, double t)>;
using TimeField = std::function<double(double t)>;

struct SpaceGrid {  // symbol.hpp:13-31
    std::vector<int> n;
    std::vector<double> lo, hi;
    double h = 0.0;
    SpaceGrid(std::vector<int> n_, std::vector<double> lo_, std::vector<double> hi_)
        : n(std::move(n_)), lo(std::move(lo_)), hi(std::move(hi_)) {
        if (n.empty() || n.size() > 2) throw std::domain_error("SpaceGrid: the B200 path supports d in {1, 2}");
        if (lo.size() != n.size() || hi.size() != n.size())
            throw DimensionError("SpaceGrid: box bounds must match the number of directions");
        for (size_t i = 0; i < n.size(); ++i) {
            if (n[i] < 1) throw std::domain_error("SpaceGrid requires n_i >= 1");
            if (!(hi[i] > lo[i])) throw std::domain_error("SpaceGrid requires box_hi > box_lo in every direction");
        }
        h = (hi[0] - lo[0]) / (n[0] + 1);
        for (size_t i = 1; i < n.size(); ++i)
            if (std::abs((hi[i] - lo[i]) / (n[i] + 1) - h) > 1e-12 * std::abs(h))
                throw std::domain_error("SpaceGrid: mesh width must be common to all directions");
    }
    int d() const { return (int)n.size(); }
    int64_t total() const { return n.size() == 1 ? n[0] : (int64_t)n[0] * n[1]; }
    // interior nodes, lexicographic order, last direction fastest (symbol.cpp:43-57)
    std::vector<std::vector<double>> nodes() const {
        std::vector<std::vector<double>> out;
        out.reserve((size_t)total());
        if (d() == 1) {
            for (int j = 1; j <= n[0]; ++j) out.push_back({lo[0] + j * h});
        } else {
            for (int j1 = 1; j1 <= n[0]; ++j1)
                for (int j2 = 1; j2 <= n[1]; ++j2) out.push_back({lo[0] + j1 * h, lo[1] + j2 * h});
        }
        return out;
    }
};

struct ProblemSpec {
    double beta, omega;  // FractionalOrders
    SpaceGrid sgrid;
    int S;
    double T;
    SpaceTimeField gamma1, gamma2;
    TimeField q;
    std::vector<double> rho, f_true;
    double lambda = 5e-3;
    double noise_eps = 0.0;
};

// ------------------------------------------------------------------ operators
class SystemOperator {
public:
    SystemOperator(Context& ctx, const ProblemSpec& spec) : ctx_(&ctx), spec_(spec) {
        const int S = spec.S;
        const int64_t N = spec.sgrid.total();
        if ((int64_t)spec.rho.size() != N || (int64_t)spec.f_true.size() != N)
            throw DimensionError("SystemOperator: rho/f_true must have length N(n)");
        if (!(spec.beta > 0.0 && spec.beta < 1.0)) throw std::domain_error("time order beta must lie in (0,1)");
        if (!(spec.omega > 1.0 && spec.omega < 2.0)) throw std::domain_error("space order omega must lie in (1,2)");
        double dt = 0.0, eta = 0.0;
        check(fi_time_grid(spec.beta, S, spec.T, &dt, &eta));
        b_.resize((size_t)S);
        e_.resize((size_t)S);
        check(fi_l1_weights(spec.beta, S, b_.data(), e_.data()));
        const int d = spec.sgrid.d();
        std::vector<double> gen;
        if (d == 1) {
            gen.resize((size_t)(2 * spec.sgrid.n[0] - 1));
            check(fi_symbol_coeffs_1d(spec.omega, spec.sgrid.n[0], gen.data()));
        } else {
            gen.resize((size_t)(2 * spec.sgrid.n[0] - 1) * (2 * spec.sgrid.n[1] - 1));
            check(fi_symbol_coeffs_md(spec.omega, 2, spec.sgrid.n.data(), 0, gen.data()));
        }
        // sample_fields (system.cpp:104-119)
        const auto nodes = spec.sgrid.nodes();
        D1_.resize((size_t)S * N);
        D2_.resize((size_t)S * N);
        q_.resize((size_t)S);
        for (int s = 1; s <= S; ++s) {
            const double t = s * dt;
            q_[(size_t)s - 1] = spec.q(t);
            for (int64_t j = 0; j < N; ++j) {
                D1_[(size_t)(s - 1) * N + j] = spec.gamma1(nodes[(size_t)j], t);
                D2_[(size_t)(s - 1) * N + j] = spec.gamma2(nodes[(size_t)j], t);
            }
        }
        const double hw = std::pow(spec.sgrid.h, spec.omega);
        fi_system_desc desc{};
        desc.d = d;
        desc.n[0] = spec.sgrid.n[0];
        desc.n[1] = d == 2 ? spec.sgrid.n[1] : 0;
        desc.S = S;
        desc.h = spec.sgrid.h;
        desc.eta = eta;
        desc.scale_space = eta / hw;
        desc.scale_reg = spec.lambda / hw;
        desc.gen = gen.data();
        desc.e = e_.data();
        desc.b = b_.data();
        desc.q = q_.data();
        desc.D1 = D1_.data();
        desc.D2 = D2_.data();
        desc.omega = spec.omega;
        check(fi_system_create(ctx.handle(), &desc, &h_));
    }
    ~SystemOperator() { fi_system_destroy(h_); }
    SystemOperator(const SystemOperator&) = delete;
    SystemOperator& operator=(const SystemOperator&) = delete;

    fi_system* handle() const noexcept { return h_; }
    const ProblemSpec& spec() const noexcept { return spec_; }
    int64_t space_dim() const { return fi_system_space_dim(h_); }
    int steps() const { return spec_.S; }
    int64_t dim() const { return fi_system_dim(h_); }
    // EXTENSION: Arnoldi steps of gmres() with this system's preconditioner compute P^{-1} A v as
    // v + P^{-1}((A - P) v) (default, one sweep per step) or in the reference's order (K1, then P^{-1})
    void set_split_apply(bool on) { check(fi_system_set_split_apply(h_, on ? 1 : 0)); }
    // EXTENSION: realisation of apply() (and of A inside gmres()): Dmma = K1, the dense FP64 DMMA contraction
    // K U (north-star (a)); Fft = K1f, the reference's circulant-embedded FFT Toeplitz products as batched 2D
    // transforms (2D grids with n_i + 1 a power of two; std::domain_error elsewhere); Auto = Fft where supported
    enum class ApplyMode { Auto = FI_APPLY_AUTO, Dmma = FI_APPLY_DMMA, Fft = FI_APPLY_FFT };
    void set_apply_mode(ApplyMode m) { check(fi_system_set_apply_mode(h_, (int)m)); }
    ApplyMode apply_mode() const { return (ApplyMode)fi_system_get_apply_mode(h_); }

    // z = A y (system.cpp:144-174)
    std::vector<double> apply(const std::vector<double>& y) const {
        if ((int64_t)y.size() != dim())
            throw DimensionError("SystemOperator::apply: vector length " + std::to_string(y.size()) +
                                 " does not match operator dimension " + std::to_string(dim()));
        std::vector<double> z(y.size());
        check(fi_system_apply_host(h_, y.data(), z.data()));
        return z;
    }
    // device-pointer overload (async on the context stream)
    void apply_device(const double* y_dev, double* z_dev) const { check(fi_system_apply(h_, y_dev, z_dev)); }

    // build_rhs (system.cpp:176-190)
    std::vector<double> build_rhs(const std::vector<double>& mu_eps) const {
        if ((int64_t)mu_eps.size() != space_dim()) throw DimensionError("build_rhs: mu_eps must have length N(n)");
        std::vector<double> z((size_t)dim());
        check(fi_build_rhs(h_, spec_.rho.data(), mu_eps.data(), z.data()));
        return z;
    }

private:
    Context* ctx_;
    ProblemSpec spec_;
    std::vector<double> b_, e_, q_, D1_, D2_;
    fi_system* h_ = nullptr;
};

class BlockTriangularPreconditioner {
public:
    static constexpr int64_t kDefaultBlockCap = 4096;
    // per-block solve: Auto = the reference's dense solve up to block_cap, and above it (2D only)
    // the substituted tau-preconditioned CG; Dense / TauPCG force one (fi_precond_create_ex)
    enum class Inner : int { Auto = -1, Dense = 0, TauPCG = 1 };
    explicit BlockTriangularPreconditioner(const SystemOperator& A, int64_t block_cap = kDefaultBlockCap) : A_(&A) {
        check(fi_precond_create(A.handle(), block_cap, &h_));
    }
    BlockTriangularPreconditioner(const SystemOperator& A, int64_t block_cap, Inner inner, double tol = 1e-14,
                                  int maxit = 200)
        : A_(&A) {
        check(fi_precond_create_ex(A.handle(), block_cap, static_cast<int>(inner), tol, maxit, &h_));
    }
    Inner inner() const { return static_cast<Inner>(fi_precond_inner(h_)); }
    ~BlockTriangularPreconditioner() { fi_precond_destroy(h_); }
    BlockTriangularPreconditioner(const BlockTriangularPreconditioner&) = delete;
    BlockTriangularPreconditioner& operator=(const BlockTriangularPreconditioner&) = delete;
    fi_precond* handle() const noexcept { return h_; }
    int64_t dim() const { return A_->dim(); }
    // y = P^{-1} z (krylov.cpp:48-70)
    std::vector<double> apply(const std::vector<double>& z) const {
        if ((int64_t)z.size() != dim())
            throw DimensionError("precond_apply: vector length " + std::to_string(z.size()) +
                                 " does not match preconditioner dimension " + std::to_string(dim()));
        std::vector<double> y(z.size());
        check(fi_precond_apply_host(h_, z.data(), y.data()));
        return y;
    }
    void apply_device(const double* z_dev, double* y_dev) const { check(fi_precond_apply(h_, z_dev, y_dev)); }
    // tau-PCG inner-solve counters since the last reset: CG steps, block solves stopped at maxit, most steps
    // of one block solve, applies (fi_precond_stats)
    std::array<long long, 4> stats(bool reset = false) const {
        std::array<long long, 4> out{};
        check(fi_precond_stats(h_, out.data(), reset ? 1 : 0));
        return out;
    }
    // the build's HODLR check: forward error vs the uncompressed inverse, backward error in the block matrix
    std::array<double, 2> build_check() const {
        std::array<double, 2> out{};
        check(fi_precond_build_check(h_, out.data()));
        return out;
    }

private:
    const SystemOperator* A_;
    fi_precond* h_ = nullptr;
};

// forward_solve (system.cpp:192-224): mu = v^(S) for the source f_true
inline std::vector<double> forward_solve_mu(SystemOperator& A, const BlockTriangularPreconditioner* P = nullptr) {
    std::vector<double> mu((size_t)A.space_dim());
    check(fi_forward_solve(A.handle(), P ? P->handle() : nullptr, A.spec().rho.data(), A.spec().f_true.data(),
                           nullptr, mu.data()));
    return mu;
}

inline std::vector<double> add_noise(const std::vector<double>& mu, double eps, uint64_t seed) {
    std::vector<double> out(mu.size());
    check(fi_add_noise(mu.data(), (long long)mu.size(), eps, seed, out.data()));
    return out;
}
inline std::vector<double> add_gaussian_noise(const std::vector<double>& mu, double rel_eps, uint64_t seed) {
    std::vector<double> out(mu.size());
    check(fi_add_gaussian_noise(mu.data(), (long long)mu.size(), rel_eps, seed, out.data()));
    return out;
}

// ------------------------------------------------------------------ GMRES (krylov.hpp:14-69)
struct GmresOptions {
    double tol = 1e-8;
    int maxit = 0;    // 0 selects the matrix dimension
    int restart = 0;  // EXTENSION: 0 = full GMRES (reference)
};

struct SolveReport {
    int iterations = 0;
    std::vector<double> residual_history;
    bool converged = false;
    bool breakdown = false;
    double wall_time_seconds = 0.0;
    double final_true_residual = 0.0;
    int inner_nonconverged = 0;  // EXTENSION: tau-PCG block solves that stopped at maxit above tol
};

inline std::pair<std::vector<double>, SolveReport> gmres(const SystemOperator& A,
                                                         const BlockTriangularPreconditioner* P,
                                                         const std::vector<double>& b, const GmresOptions& opts = {},
                                                         const std::vector<double>* x0 = nullptr) {
    if ((int64_t)b.size() != A.dim()) throw DimensionError("gmres: right-hand side length does not match the operator");
    std::vector<double> x(b.size());
    const int cap = (opts.maxit > 0 ? opts.maxit : (int)std::min<int64_t>(A.dim(), 1 << 20)) + 1;
    std::vector<double> hist((size_t)cap);
    fi_gmres_opts o{opts.tol, opts.maxit, opts.restart};
    fi_gmres_report r{};
    check(fi_gmres_host(A.handle(), P ? P->handle() : nullptr, b.data(), x0 ? x0->data() : nullptr, x.data(), &o, &r,
                        hist.data(), cap));
    SolveReport rep;
    rep.iterations = r.iterations;
    rep.converged = r.converged != 0;
    rep.breakdown = r.breakdown != 0;
    rep.wall_time_seconds = r.wall_time_seconds;
    rep.final_true_residual = r.final_true_residual;
    rep.inner_nonconverged = r.inner_nonconverged;
    rep.residual_history.assign(hist.begin(), hist.begin() + std::min(r.history_len, cap));
    return {std::move(x), std::move(rep)};
}

inline std::vector<double> extract_reconstruction(const std::vector<double>& y, int64_t space_dim) {
    if ((int64_t)y.size() % space_dim != 0 || (int64_t)y.size() < 2 * space_dim)
        throw DimensionError("extract_reconstruction: vector is not a stacked block vector");
    return std::vector<double>(y.end() - space_dim, y.end());
}

inline double relative_error(const std::vector<double>& truth, const std::vector<double>& approx) {
    if (truth.size() != approx.size()) throw DimensionError("relative_error: size mismatch");
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < truth.size(); ++i) {
        num += (truth[i] - approx[i]) * (truth[i] - approx[i]);
        den += truth[i] * truth[i];
    }
    return std::sqrt(num) / std::sqrt(den);
}

}  // namespace b200
}  // namespace fracinv
