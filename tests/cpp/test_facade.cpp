// Reference-style C++ host program over the C++ façade (include/fracinv_b200.hpp): BASELINE
// config 0 end to end, the canonical call sequence of the reference (acceptance.cpp:185-193):
//   SystemOperator A(spec); BlockTriangularPreconditioner P(A);
//   mu = add_noise(forward_solve(A).mu); z = build_rhs(A, mu); gmres(A, P, z, {tol, maxit, restart})
// plus the reference's error contract.  Writes f~ (binary doubles) to argv[1] and one JSON line
// to stdout; tests/test_gpu_facade.py compares both with the CPU oracle.
#include <cmath>
#include <cstdio>
#include <fstream>

#include "fracinv_b200.hpp"

using namespace fracinv::b200;

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s f_out.bin\n", argv[0]);
        return 2;
    }
    const double pi = 3.14159265358979323846;
    Context ctx(0);
    const int n = 255, S = 64;
    SpaceGrid grid({n}, {0.0}, {1.0});
    std::vector<double> rho((size_t)n), f((size_t)n);
    const auto nodes = grid.nodes();
    for (int j = 0; j < n; ++j) {
        const double x = nodes[(size_t)j][0];
        rho[(size_t)j] = x * x * (1 - x) * (1 - x);
        f[(size_t)j] = std::sin(pi * x);
    }
    ProblemSpec spec{0.5, 1.5, grid, S, 1.0,
                     [pi](const std::vector<double>& x, double t) { return 1 + 0.5 * std::sin(pi * x[0]) * std::exp(-t); },
                     [](const std::vector<double>& x, double t) { return 1 + x[0] * (1 - x[0]) * (1 + t); },
                     [](double t) { return 1 + t; }, rho, f, 1e-3, 0.01};
    SystemOperator A(ctx, spec);
    BlockTriangularPreconditioner P(A);
    const auto mu = add_gaussian_noise(forward_solve_mu(A, &P), 0.01, 1000);
    const auto z = A.build_rhs(mu);
    const auto [y, rep] = gmres(A, &P, z, {1e-10, 0, 50});
    const auto frec = extract_reconstruction(y, A.space_dim());
    std::ofstream(argv[1], std::ios::binary).write(reinterpret_cast<const char*>(frec.data()),
                                                  (std::streamsize)(frec.size() * sizeof(double)));

    // error contract: vanishing gamma2 at t_S -> SingularBlockError(S+1) (test_krylov.cpp:49-63)
    int singular_index = 0;
    {
        SpaceGrid g4({4}, {0.0}, {pi});
        ProblemSpec bad{0.5, 1.5, g4, 2, 1.0, [](const std::vector<double>&, double) { return 1.0; },
                        [](const std::vector<double>&, double t) { return 1.0 - t; }, [](double) { return 1.0; },
                        std::vector<double>(4, 0.0), std::vector<double>(4, 0.0), 1e-2, 0.0};
        SystemOperator B(ctx, bad);
        try {
            BlockTriangularPreconditioner PB(B);
        } catch (const SingularBlockError& ex) {
            singular_index = ex.time_index();
        }
    }
    bool dim_error = false;
    try {
        A.apply(std::vector<double>(3, 0.0));
    } catch (const DimensionError&) {
        dim_error = true;
    }
    // the substituted 2D block solve (tau-PCG) against the dense inverses on a 15x15 grid
    double tau_vs_dense = 1.0, fft_vs_dmma = 1.0;
    int tau_inner = -1;
    bool fft_default = false, fft_refused_1d = false;
    {
        SpaceGrid g2({15, 15}, {0.0, 0.0}, {1.0, 1.0});
        const auto nodes2 = g2.nodes();
        std::vector<double> rho2(nodes2.size(), 0.0), f2(nodes2.size());
        for (size_t j = 0; j < nodes2.size(); ++j) f2[j] = std::sin(pi * nodes2[j][0]) * std::sin(pi * nodes2[j][1]);
        ProblemSpec s2{0.3, 1.2, g2, 8, 1.0,
                       [](const std::vector<double>& x, double) { return 1 + x[0] * x[1]; },
                       [](const std::vector<double>& x, double t) { return 1 + x[0] * (1 + t); },
                       [](double t) { return 1 + t * t; }, rho2, f2, 1e-3, 0.01};
        SystemOperator A2(ctx, s2);
        using Inner = BlockTriangularPreconditioner::Inner;
        BlockTriangularPreconditioner Pt(A2, 4096, Inner::TauPCG), Pd(A2, 4096, Inner::Dense);
        tau_inner = static_cast<int>(Pt.inner());
        std::vector<double> v((size_t)A2.dim());
        for (size_t i = 0; i < v.size(); ++i) v[i] = std::sin(0.37 * (double)i) + 0.25;
        const auto yt = Pt.apply(v), yd = Pd.apply(v);
        double num = 0.0, den = 0.0;
        for (size_t i = 0; i < v.size(); ++i) {
            num += (yt[i] - yd[i]) * (yt[i] - yd[i]);
            den += yd[i] * yd[i];
        }
        tau_vs_dense = std::sqrt(num / den);
        // the operator's two realisations: K1f (FFT, the default on this 2D grid) against K1 (DMMA)
        fft_default = A2.apply_mode() == SystemOperator::ApplyMode::Fft;
        const auto zf = A2.apply(v);
        A2.set_apply_mode(SystemOperator::ApplyMode::Dmma);
        const auto zd = A2.apply(v);
        A2.set_apply_mode(SystemOperator::ApplyMode::Auto);
        num = den = 0.0;
        for (size_t i = 0; i < v.size(); ++i) {
            num += (zf[i] - zd[i]) * (zf[i] - zd[i]);
            den += zd[i] * zd[i];
        }
        fft_vs_dmma = std::sqrt(num / den);
        try {
            A.set_apply_mode(SystemOperator::ApplyMode::Fft);  // 1D: no FFT realisation
        } catch (const std::domain_error&) {
            fft_refused_1d = true;
        }
    }
    std::printf("{\"iterations\": %d, \"converged\": %s, \"final_true_residual\": %.17g, \"recon_error\": %.17g, "
                "\"singular_index\": %d, \"dimension_error\": %s, \"history_len\": %zu, \"tau_inner\": %d, "
                "\"tau_vs_dense\": %.17g, \"fft_default\": %s, \"fft_vs_dmma\": %.17g, \"fft_refused_1d\": %s}\n",
                rep.iterations, rep.converged ? "true" : "false", rep.final_true_residual,
                relative_error(f, frec), singular_index, dim_error ? "true" : "false", rep.residual_history.size(),
                tau_inner, tau_vs_dense, fft_default ? "true" : "false", fft_vs_dmma, fft_refused_1d ? "true" : "false");
    return 0;
}
