// Device-resident all-at-once system (replaces SystemOperator, system.hpp:72-104).
#pragma once

#include "common.cuh"

namespace fib {

// Kernel-side view of the system operator, passed by value to the kernels.
struct OperatorView {
    int n1, n2, ld2, S;
    long long Np;
    int gen_stride;        // row stride of the padded generating tensor (doubles)
    const double* gen;     // (2 n1 - 1) rows x gen_stride: row r holds a[r-(n1-1)][l2] at l2 + ld2
    const double* epad;    // e padded: epad[EOFF + k] = e_k (0 <= k < S), zeros elsewhere
    const double* D1;      // S x Np (pads 0)
    const double* D2;      // S x Np (pads 0)
    const double* q;       // S
    double cs, cr, eta;    // scale_space, scale_reg, eta
};
constexpr int kEOFF = 128;

}  // namespace fib

namespace fib {
class GmresEngine;
}

struct fi_system {
    int refs = 1;
    fi_ctx* ctx = nullptr;
    fib::Layout L;
    double h = 0, eta = 0, cs = 0, cr = 0, omega = 0;
    std::vector<double> gen_h, e_h, b_h, q_h, D1_h, D2_h;  // host copies (reference layout)
    fib::DevBuf<double> gen, epad, D1, D2, q, e, bw;
    fib::DevBuf<double> ubuf, zbuf;  // padded scratch for reference-layout applies
    fib::DevBuf<double> gb, gx, gx0, gio;  // fi_gmres padded b / x / x0 and host-call staging
    fib::DevBuf<double> sp_u, sp_t;        // scratch of the split preconditioned apply
    int split_apply = 1;                   // fi_gmres: P^{-1} A v as v + P^{-1}((A - P) v) (fi_system_set_split_apply)
    int apply_mode = 0;                    // FI_APPLY_AUTO / _DMMA / _FFT (fi_system_set_apply_mode)
    bool fft_ok = false;                   // the FFT apply supports this layout (2D, n_i + 1 a power of two)
    bool fft_ready = false;                // K1f tables and workspace allocated
    fib::DevBuf<double2> fft_tw1, fft_tw2, fft_W;  // K1f: twiddles, half-spectrum workspace (S+1) x n1 x H2
    fib::DevBuf<double> fft_lamB;                  // K1f: L1 x L2 spectrum of the embedded generating tensor
    // AUTO: the transforms where they exist (2D), the dense DMMA contraction (K1) otherwise
    bool use_fft() const { return fft_ok && apply_mode != 1; }
    fib::GmresEngine* engine = nullptr;  // cached Krylov workspace (owned; freed in fi_system_destroy)
    fib::OperatorView view() const {
        fib::OperatorView v;
        v.n1 = L.n1; v.n2 = L.n2; v.ld2 = L.ld2; v.S = L.S; v.Np = L.Np;
        v.gen_stride = 2 * L.ld2 + 8;
        v.gen = gen.p; v.epad = epad.p; v.D1 = D1.p; v.D2 = D2.p; v.q = q.p;
        v.cs = cs; v.cr = cr; v.eta = eta;
        return v;
    }
};

namespace fib {
class GmresEngine;
// Z = A U on padded device vectors (K1: on-the-fly Toeplitz DMMA GEMM + fused epilogue).
// skip: optional device flag; the kernel returns immediately when *skip != 0.
// minus_from != nullptr: Z = minus_from - (A U) (residual form).  precond_matrix: apply P instead of
// A, i.e. drop the -eta q_s f coupling (the block column that P zeroes, spectra.cpp:34-36).
void toeplitz_apply(fi_ctx* ctx, const OperatorView& op, const double* U, double* Z, const int* skip,
                    const double* minus_from = nullptr, bool precond_matrix = false);
// K1 in conv-only mode: the time levels' D1 o (U E^T) - eta q f alone (the f column is not written)
void toeplitz_conv_apply(fi_ctx* ctx, const OperatorView& op, const double* U, double* Z, const int* skip,
                         const double* minus_from, bool precond_matrix, cudaStream_t stream);
// K1f: the same Z with K u_s by batched 2D FFTs (toeplitz_fft.cu); 2D layouts with n_i + 1 a power of two
bool fft_apply_supported(const Layout& L);
void fft_apply_prepare(fi_system* sys);  // tables and workspace (not inside a stream capture)
void toeplitz_apply_fft(fi_ctx* ctx, fi_system* sys, const double* U, double* Z, const int* skip,
                        const double* minus_from = nullptr, bool precond_matrix = false);
// the system's operator apply in its selected realisation (K1f or K1)
void system_apply(fi_ctx* ctx, fi_system* sys, const double* U, double* Z, const int* skip,
                  const double* minus_from = nullptr, bool precond_matrix = false);
}  // namespace fib
