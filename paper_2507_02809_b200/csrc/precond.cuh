// Block lower-triangular preconditioner P (replaces BlockTriangularPreconditioner,
// krylov.hpp:33-50, krylov.cpp:24-70).
#pragma once

#include "system.cuh"

namespace fib {
struct HodlrData;
}

struct fi_precond {
    fi_system* sys = nullptr;
    unsigned long long uid = 0;  // unique per preconditioner built (keys the captured GMRES graph)
    int nb = 0;        // 64-row blocks per level (Np / 64)
    long long T = 0;   // lower-triangular 64x64 tiles per level: nb (nb + 1) / 2
    int G = 0;         // persistent CTAs of the apply kernel
    int levels = 0;    // S + 1
    int refine = 1;    // one iterative-refinement sweep per apply (0 by default once the inverses are polished)
    fib::HodlrData* hodlr = nullptr;  // dense blocks in HODLR form (precond_hodlr.cu), else packed tiles
    double hodlr_check_fwd = 0.0, hodlr_check_bwd = 0.0;  // the build's a-posteriori HODLR check (worst level)
    fib::DevBuf<double> H;      // [level][tile][64*64]: packed symmetric inverses
    fib::DevBuf<float> Hf;      // FP32 copy for the refinement sweep
    fib::DevBuf<double> rbuf, dbuf;  // refinement residual and correction
    fib::DevBuf<double> d2inv;  // S x Np: 1 / D2 (pads 0)
    fib::DevBuf<double> xbuf;   // 2 x Np (pass parity)
    fib::DevBuf<double> pbuf;   // 2 x nb x nb x 64 partial products (pass parity)
    fib::DevBuf<unsigned> counters;  // xready[nb], pdone[nb], grid barrier
    fib::DevBuf<double> zbuf, ybuf;  // padded scratch for reference-layout applies
    // merged refinement sweep (precond_sweep_ir.cu), allocated on first use
    fib::DevBuf<double> ir_xb;        // 3 kinds x 2 parities x Np
    fib::DevBuf<double> ir_pb;        // 3 kinds x 2 parities x nb x nb x 64
    fib::DevBuf<unsigned> ir_counters;  // xready[nb], pdone[3][nb], xready2[nb], pdone1b[nb]

    // ---- mode 1: substituted per-block solve (tau-preconditioned CG, precond_iter.cu)
    int mode = 0;  // 0 = dense packed inverses, 1 = tau-PCG per level
    double it_tol = 1e-14;
    int it_maxit = 200;
    int it_L1 = 0, it_L2 = 0;
    std::vector<double> it_dmean;
    double it_gmax = 0.0;  // largest tau eigenvalue g(theta)
    std::vector<int> it_direct;
    fib::DevBuf<double2> it_tw1, it_tw2, it_X;
    fib::DevBuf<double> it_lamT, it_lamB, it_Rr, it_vec, it_dmean_d, it_hb;
    fib::DevBuf<double2> it_F;                   // fused kernel: Zh, Xp, Yb half-spectrum buffers
    fib::DevBuf<unsigned long long> it_stats;    // CG steps, levels stopped at maxit, max steps, applies
    fib::DevBuf<int> it_direct_d;
    int it_fgrid = 0;                            // fused kernel: cooperative grid size
    int it_cu = 2;                               // fused kernel: B column-pass columns per CTA
    bool it_occ_checked = false;
    fib::DevBuf<double> it_fparts;               // fused kernel: 2 x grid block partials
    fib::DevBuf<unsigned> it_fbar;               // fused kernel: grid-barrier counter
    ~fi_precond();
};

namespace fib {
// sweep dataflow counters are kept one 128-byte L2 line apart (unsigned units)
constexpr int kCounterStride = 32;
// y = P^{-1} z on padded vectors (K2).  levels = S+1 (full P) or S (time levels only:
// the forward solve, system.cpp:192-224).  skip: optional device flag.
void precond_apply(fi_ctx* ctx, fi_precond* P, const double* z, double* y, int levels, const int* skip);
// w = P^{-1} A v = v + P^{-1}((A - P) v) (one sweep, no operator apply); u, t: padded scratch vectors
void precond_times_operator(fi_ctx* ctx, fi_precond* P, const double* v, double* w, double* u, double* t,
                            const int* skip);
// mode 1 (2D blocks above the dense cap): build / apply of the tau-PCG per-level solve
bool iterative_supported(const Layout& L);
void precond_build_iterative(fi_precond* P, double tol, int maxit);
void precond_apply_iterative(fi_ctx* ctx, fi_precond* P, const double* z, double* y, int levels, const int* skip);
// inner-solve counters accumulated on the device since the last reset: [0] CG steps, [1] levels that
// stopped at maxit without reaching the tolerance, [2] most steps of one level, [3] applies (synchronises)
void precond_iterative_stats(fi_precond* P, unsigned long long out[4], bool reset);
void precond_build(fi_precond* P);
// build-time polish of the explicit inverses (precond_polish.cu): W <- W - Q Z^T, a rank-32
// sketch of W - G_x^{-1} D2 from double-double residuals
bool polish_enabled();
size_t polish_work_doubles(long long Np, int nbt);
void polish_inverses(fi_ctx* ctx, const OperatorView& op, double* W, int nbt, int l0, const double* bscale,
                     double* work);
// HODLR form of the dense-block inverses (precond_hodlr.cu)
bool hodlr_supported(const Layout& L, int levels, int sm_count);
HodlrData* hodlr_create(const Layout& L, int levels);
void hodlr_destroy(HodlrData* h);
size_t hodlr_bytes(const HodlrData* h);
size_t hodlr_work_doubles(const Layout& L, int nbt);
void hodlr_compress(fi_ctx* ctx, HodlrData* h, const Layout& L, const double* W, int nbt, int l0, double* work);
double hodlr_check(fi_ctx* ctx, HodlrData* h, const Layout& L, const double* W, int nbt, int l0, double* work,
                   const OperatorView& op, const double* diag, const double* bscale, double* backward);
void hodlr_sweep(fi_ctx* ctx, HodlrData* h, const fi_system* sys, const double* d2inv, const double* z, double* y,
                 int levels, const int* skip);
// merged sweep: forward substitution + one refinement step in one persistent kernel (K2)
bool sweep_ir_available(const fi_precond* P);
void launch_sweep_ir(fi_ctx* ctx, fi_precond* P, const double* z, double* y, int levels, const int* skip);
// cooperative grid size of the sweep kernel for T tiles per level and Np rows
int precond_apply_grid(fi_ctx* ctx, long long T, long long Np);
// z_s = b_{s-1} D1_s o rho + eta q_s f (padded, levels 0..S-1): forward-solve right-hand side.
void forward_rhs(fi_ctx* ctx, const fi_system* sys, const double* rho_pad, const double* f_pad, double* z_pad);
}  // namespace fib
