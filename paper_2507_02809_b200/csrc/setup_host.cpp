// Host-side setup numerics of the product (problem assembly, not the hot path).
//
// Restatements of numerics.cpp (Lanczos Gamma, L1 weights, time grid), symbol.cpp
// (generating vectors) and system.cpp:228-251 (SplitMix64 noise) of the reference.  The
// multilevel generating tensor uses the reference's rectangle rule with the same sample
// counts (symbol.cpp:122-134); the DFT is evaluated only at the (2n_i - 1) needed
// frequencies, separably, instead of a full FFT (same quadrature, different summation).
#include <cmath>
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace fib {

namespace {
constexpr double kLanczosG = 7.0;
constexpr double kLanczosP[9] = {
    0.99999999999980993,  676.5203681218851,     -1259.1392167224028,
    771.32342877765313,   -176.61502916214059,   12.507343278686905,
    -0.13857109526572012, 9.9843695780195716e-6, 1.5056327351493116e-7,
};
constexpr double kSqrtTwoPi = 2.5066282746310002;
constexpr double kPi = 3.14159265358979323846;

double lanczos(double x) {
    if (x < 0.5) return lanczos(x + 1.0) / x;
    const double z = x - 1.0;
    double s = kLanczosP[0];
    for (int k = 1; k < 9; ++k) s += kLanczosP[k] / (z + k);
    const double t = z + kLanczosG + 0.5;
    if (x < 140.0) return kSqrtTwoPi * std::pow(t, z + 0.5) * std::exp(-t) * s;
    return kSqrtTwoPi * std::exp((z + 0.5) * std::log(t) - t) * s;
}

uint64_t splitmix64_at(uint64_t seed, uint64_t j) {
    uint64_t z = seed + (j + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

double unit_open(uint64_t z) { return (static_cast<double>(z >> 11) + 0.5) * (1.0 / 9007199254740992.0); }
}  // namespace

double gamma_fn(double x) {
    if (!(x > 0.0)) throw Error(FI_E_DOMAIN, "gamma_fn requires x > 0, got " + std::to_string(x));
    return lanczos(x);
}

void l1_weights(double beta, int S, double* b, double* e) {
    if (!(beta > 0.0 && beta < 1.0)) throw Error(FI_E_DOMAIN, "l1_weights requires beta in (0,1)");
    if (S < 1) throw Error(FI_E_DOMAIN, "l1_weights requires S >= 1");
    const double p = 1.0 - beta;
    for (int m = 0; m < S; ++m) b[m] = std::pow(m + 1.0, p) - std::pow(static_cast<double>(m), p);
    e[0] = b[0];
    for (int m = 1; m < S; ++m) e[m] = b[m] - b[m - 1];
}

void time_grid(double beta, int S, double T, double* dt, double* eta) {
    if (!(beta > 0.0 && beta < 1.0)) throw Error(FI_E_DOMAIN, "time_grid requires beta in (0,1)");
    if (S < 1) throw Error(FI_E_DOMAIN, "time_grid requires S >= 1");
    if (!(T > 0.0)) throw Error(FI_E_DOMAIN, "time_grid requires T > 0");
    *dt = T / S;
    *eta = std::pow(*dt, beta) * gamma_fn(2.0 - beta);
}

static void check_omega(double omega) {
    if (!(omega > 0.0 && omega <= 2.0)) throw Error(FI_E_DOMAIN, "symbol coefficients require omega in (0,2]");
}

void symbol_coeffs_1d(double omega, int n, double* coeffs) {
    check_omega(omega);
    if (n < 1) throw Error(FI_E_DOMAIN, "symbol_coeffs_1d requires n >= 1");
    std::vector<double> a((size_t)n);
    const double g1 = gamma_fn(omega / 2.0 + 1.0);
    a[0] = gamma_fn(omega + 1.0) / (g1 * g1);
    for (int l = 0; l + 1 < n; ++l) a[(size_t)l + 1] = (1.0 - (omega + 1.0) / (omega / 2.0 + l + 1.0)) * a[(size_t)l];
    for (int l = -(n - 1); l <= n - 1; ++l) coeffs[l + n - 1] = a[(size_t)std::abs(l)];
}

void symbol_coeffs_md(double omega, int d, const int* n, long long sample_cap, double* coeffs) {
    check_omega(omega);
    if (d < 1 || d > 2) throw Error(FI_E_DOMAIN, "symbol_coeffs_md supports d in {1, 2}");
    int M[2] = {1, 1};
    long long total = 1;
    for (int i = 0; i < d; ++i) {
        if (n[i] < 1) throw Error(FI_E_DOMAIN, "symbol_coeffs_md requires n_i >= 1");
        const int base = d == 1 ? 131072 : 1024;
        M[i] = std::max(4 * n[i], base);
        total *= M[i];
        if (total > sample_cap)
            throw Error(FI_E_RESOURCE, "symbol_coeffs_md: sample tensor of " + std::to_string(total) +
                                           " points exceeds cap " + std::to_string(sample_cap));
    }
    // per-direction 4 sin^2(pi k / M_i) and cos tables (symbol.cpp:142-150)
    std::vector<std::vector<double>> s2(d), ct(d);
    for (int i = 0; i < d; ++i) {
        s2[i].resize((size_t)M[i]);
        ct[i].resize((size_t)M[i]);
        for (int k = 0; k < M[i]; ++k) {
            const double s = std::sin(kPi * k / M[i]);
            s2[i][(size_t)k] = 4.0 * s * s;
            ct[i][(size_t)k] = std::cos(2.0 * kPi * k / M[i]);
        }
    }
    const double half = omega / 2.0;
    const double scale = 1.0 / static_cast<double>(total);
    if (d == 1) {
        const int n0 = n[0];
        std::vector<double> g((size_t)M[0]);
        for (int k = 0; k < M[0]; ++k) g[(size_t)k] = std::pow(s2[0][(size_t)k], half);
        for (int l = 0; l < n0; ++l) {
            double acc = 0.0;
            for (int k = 0; k < M[0]; ++k) acc += g[(size_t)k] * ct[0][(size_t)(((long long)k * l) % M[0])];
            coeffs[l + n0 - 1] = coeffs[-l + n0 - 1] = acc * scale;
        }
        return;
    }
    const int n1 = n[0], n2 = n[1];
    // stage 1: Tk[k1][l2] = sum_k2 g(k1,k2) cos(2 pi k2 l2 / M2), l2 = 0..n2-1
    std::vector<double> Tk((size_t)M[0] * n2);
    std::vector<double> row((size_t)M[1]);
    for (int k1 = 0; k1 < M[0]; ++k1) {
        for (int k2 = 0; k2 < M[1]; ++k2) row[(size_t)k2] = std::pow(s2[0][(size_t)k1] + s2[1][(size_t)k2], half);
        for (int l2 = 0; l2 < n2; ++l2) {
            double acc = 0.0;
            for (int k2 = 0; k2 < M[1]; ++k2) acc += row[(size_t)k2] * ct[1][(size_t)(((long long)k2 * l2) % M[1])];
            Tk[(size_t)k1 * n2 + l2] = acc;
        }
    }
    // stage 2: a[l1][l2] = sum_k1 Tk[k1][l2] cos(2 pi k1 l1 / M1); the symbol is even in each l_i
    const int w2 = 2 * n2 - 1;
    for (int l1 = 0; l1 < n1; ++l1)
        for (int l2 = 0; l2 < n2; ++l2) {
            double acc = 0.0;
            for (int k1 = 0; k1 < M[0]; ++k1)
                acc += Tk[(size_t)k1 * n2 + l2] * ct[0][(size_t)(((long long)k1 * l1) % M[0])];
            const double v = acc * scale;
            for (int sg1 = -1; sg1 <= 1; sg1 += 2)
                for (int sg2 = -1; sg2 <= 1; sg2 += 2)
                    coeffs[(size_t)(sg1 * l1 + n1 - 1) * w2 + (sg2 * l2 + n2 - 1)] = v;
        }
}

void add_noise(const double* mu, long long n, double eps, uint64_t seed, double* out) {
    if (eps < 0.0) throw Error(FI_E_DOMAIN, "add_noise requires eps >= 0");
    for (long long j = 0; j < n; ++j) out[j] = mu[j] + eps * (2.0 * unit_open(splitmix64_at(seed, (uint64_t)j)) - 1.0);
}

void add_gaussian_noise(const double* mu, long long n, double rel_eps, uint64_t seed, double* out) {
    if (rel_eps < 0.0) throw Error(FI_E_DOMAIN, "add_gaussian_noise requires eps >= 0");
    std::vector<double> delta((size_t)n);
    for (long long p = 0; 2 * p < n; ++p) {
        const double u1 = unit_open(splitmix64_at(seed, (uint64_t)(2 * p)));
        const double u2 = unit_open(splitmix64_at(seed, (uint64_t)(2 * p + 1)));
        const double r = std::sqrt(-2.0 * std::log(u1));
        delta[(size_t)(2 * p)] = r * std::cos(2.0 * kPi * u2);
        if (2 * p + 1 < n) delta[(size_t)(2 * p + 1)] = r * std::sin(2.0 * kPi * u2);
    }
    double nmu = 0.0, nd = 0.0;
    for (long long j = 0; j < n; ++j) {
        nmu += mu[j] * mu[j];
        nd += delta[(size_t)j] * delta[(size_t)j];
    }
    const double scale = rel_eps == 0.0 ? 0.0 : rel_eps * std::sqrt(nmu) / std::sqrt(nd);
    for (long long j = 0; j < n; ++j) out[j] = mu[j] + scale * delta[(size_t)j];
}

}  // namespace fib
