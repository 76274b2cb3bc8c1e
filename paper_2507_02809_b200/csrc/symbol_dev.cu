// Setup on the device: the 2D generating tensor of the fractional Laplacian.
//
// Replaces the host's rectangle-rule symbol sums (symbol.cpp:112-191; setup_host.cpp
// symbol_coeffs_md): with M_i = max(4 n_i, 1024) samples per direction,
//   Tk[k1][l2] = sum_k2 g(k1, k2) cos(2 pi k2 l2 / M2),   g = (4 sin^2(pi k1/M1) + 4 sin^2(pi k2/M2))^(w/2)
//   a[l1][l2]  = (sum_k1 Tk[k1][l2] cos(2 pi k1 l1 / M1)) / (M1 M2),   mirrored to +-l1, +-l2.
// The host computes g and the cosine tables with the same expressions as before (g needs 1M pow
// calls; the device's pow may differ from libm's in the last ulp); every sum then runs on the
// device in the host's order, one output per thread, with __dmul_rn/__dadd_rn (no FMA
// contraction), so the tensor is bit-for-bit the host's.  Config 3 / 4
// (255 x 255): 0.33 G multiply-adds, 1.35 s on one host core.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace fib {
namespace {

constexpr double kPiD = 3.14159265358979323846;

// Tk[k1][l2] for one k1 per CTA; the g row and the cosine table in shared memory
__global__ void sym_stage1(const double* __restrict__ G, const double* __restrict__ ct2, int M2, int n2,
                           double* __restrict__ Tk) {
    extern __shared__ double sm[];
    double* row = sm;
    double* ct = sm + M2;
    const int k1 = blockIdx.x;
    for (int k = threadIdx.x; k < M2; k += blockDim.x) {
        row[k] = G[(long long)k1 * M2 + k];
        ct[k] = ct2[k];
    }
    __syncthreads();
    for (int l2 = threadIdx.x; l2 < n2; l2 += blockDim.x) {
        double acc = 0.0;
        for (int k2 = 0; k2 < M2; ++k2) acc = __dadd_rn(acc, __dmul_rn(row[k2], ct[(int)(((long long)k2 * l2) % M2)]));
        Tk[(long long)k1 * n2 + l2] = acc;
    }
}

// a[l1][l2] for one l1 per CTA, mirrored into the (2 n1 - 1) x (2 n2 - 1) tensor
__global__ void sym_stage2(const double* __restrict__ Tk, const double* __restrict__ ct1, int M1, int n1, int n2,
                           double scale, double* __restrict__ coeffs) {
    extern __shared__ double ct[];
    const int l1 = blockIdx.x;
    for (int k = threadIdx.x; k < M1; k += blockDim.x) ct[k] = ct1[k];
    __syncthreads();
    const int w2 = 2 * n2 - 1;
    for (int l2 = threadIdx.x; l2 < n2; l2 += blockDim.x) {
        double acc = 0.0;
#pragma unroll 8
        for (int k1 = 0; k1 < M1; ++k1)
            acc = __dadd_rn(acc, __dmul_rn(__ldg(Tk + (long long)k1 * n2 + l2), ct[(int)(((long long)k1 * l1) % M1)]));
        const double v = __dmul_rn(acc, scale);
        for (int sg1 = -1; sg1 <= 1; sg1 += 2)
            for (int sg2 = -1; sg2 <= 1; sg2 += 2)
                coeffs[(long long)(sg1 * l1 + n1 - 1) * w2 + (sg2 * l2 + n2 - 1)] = v;
    }
}

}  // namespace

// 2D generating tensor on the device of `ctx`; coeffs (host) gets (2 n1 - 1) (2 n2 - 1) entries.
void symbol_coeffs_2d_dev(fi_ctx* ctx, double omega, int n1, int n2, long long sample_cap, double* coeffs) {
    if (!(omega > 0.0 && omega <= 2.0)) throw Error(FI_E_DOMAIN, "symbol coefficients require omega in (0,2]");
    if (n1 < 1 || n2 < 1) throw Error(FI_E_DOMAIN, "symbol_coeffs_md requires n_i >= 1");
    const int M1 = std::max(4 * n1, 1024), M2 = std::max(4 * n2, 1024);
    const long long total = (long long)M1 * M2;
    if (total > sample_cap)
        throw Error(FI_E_RESOURCE, "symbol_coeffs_md: sample tensor of " + std::to_string(total) +
                                       " points exceeds cap " + std::to_string(sample_cap));
    // host tables, the same expressions as setup_host.cpp
    std::vector<double> s2a((size_t)M1), s2b((size_t)M2), ct1((size_t)M1), ct2((size_t)M2);
    for (int k = 0; k < M1; ++k) {
        const double s = std::sin(kPiD * k / M1);
        s2a[(size_t)k] = 4.0 * s * s;
        ct1[(size_t)k] = std::cos(2.0 * kPiD * k / M1);
    }
    for (int k = 0; k < M2; ++k) {
        const double s = std::sin(kPiD * k / M2);
        s2b[(size_t)k] = 4.0 * s * s;
        ct2[(size_t)k] = std::cos(2.0 * kPiD * k / M2);
    }
    const double half = omega / 2.0;
    std::vector<double> G((size_t)total);
    for (int k1 = 0; k1 < M1; ++k1)
        for (int k2 = 0; k2 < M2; ++k2) G[(size_t)k1 * M2 + k2] = std::pow(s2a[(size_t)k1] + s2b[(size_t)k2], half);
    const double scale = 1.0 / static_cast<double>(total);
    const size_t ncoef = (size_t)(2 * n1 - 1) * (2 * n2 - 1);
    DevBuf<double> Gd((size_t)total), c1((size_t)M1), c2((size_t)M2), Tk((size_t)M1 * n2), out(ncoef);
    cudaStream_t s = ctx->stream;
    FI_CUDA(cudaMemcpyAsync(Gd.p, G.data(), G.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    FI_CUDA(cudaMemcpyAsync(c1.p, ct1.data(), ct1.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    FI_CUDA(cudaMemcpyAsync(c2.p, ct2.data(), ct2.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    const size_t sm1 = 2 * (size_t)M2 * sizeof(double), sm2 = (size_t)M1 * sizeof(double);
    if (sm1 > 48 * 1024) FI_CUDA(cudaFuncSetAttribute(sym_stage1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
    if (sm2 > 48 * 1024) FI_CUDA(cudaFuncSetAttribute(sym_stage2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
    const int thr = n2 >= 256 ? 256 : ((n2 + 31) / 32) * 32;
    sym_stage1<<<M1, thr, sm1, s>>>(Gd.p, c2.p, M2, n2, Tk.p);
    FI_LAUNCHED(ctx);
    sym_stage2<<<n1, thr, sm2, s>>>(Tk.p, c1.p, M1, n1, n2, scale, out.p);
    FI_LAUNCHED(ctx);
    FI_CUDA(cudaMemcpyAsync(coeffs, out.p, ncoef * sizeof(double), cudaMemcpyDeviceToHost, s));
    FI_CUDA(cudaStreamSynchronize(s));
}

}  // namespace fib
