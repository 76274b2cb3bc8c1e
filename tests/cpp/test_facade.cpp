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
    std::printf("{\"iterations\": %d, \"converged\": %s, \"final_true_residual\": %.17g, \"recon_error\": %.17g, "
                "\"singular_index\": %d, \"dimension_error\": %s, \"history_len\": %zu}\n",
                rep.iterations, rep.converged ? "true" : "false", rep.final_true_residual,
                relative_error(f, frec), singular_index, dim_error ? "true" : "false", rep.residual_history.size());
    return 0;
}
