// K2 setup — per-level symmetric inverses of the block lower-triangular preconditioner.
//
// Reference: BlockTriangularPreconditioner::BlockTriangularPreconditioner (krylov.cpp:24-46)
// assembles G_s = cs D2_s B + e0 D1_s (s = 1..S) and G_f = cr D2_S B and caches their
// PartialPivLU factors.  Here G = D2 M with M = cs B + e0 diag(D1/D2) (resp. cr B) symmetric
// positive definite; the device computes H = M^{-1} by batched blocked Gauss-Jordan (no
// pivoting on an SPD matrix; the 64-wide rank updates run on the FP64 tensor pipe, DMMA) and
// packs the lower triangle of 64x64 tiles in FP64 plus an FP32 copy for the refinement sweep
// (precond_apply.cu).  The reference's pivot test (min|piv| <= 1e-14 max|piv|, krylov.cpp:14-20)
// is applied to the Gauss-Jordan pivots, the LDL^T diagonal of M.
#include <cmath>

#include <cstdlib>

#include "precond.cuh"

namespace fib {
namespace {

constexpr int TB = 64;            // tile edge
constexpr int TILE = TB * TB;     // doubles per tile
// HODLR acceptance: the normwise backward error |M y - x| / (|M| |y| + |x|) of y = H_hodlr x in the block
// matrix itself (an LU solve reaches ~1e-16; the rank-32 truncation is accepted up to this)
constexpr double kHodlrBackwardTol = 1e-13;

__device__ __forceinline__ void tile_coords(long long t, int& bi, int& bj) {
    // lower-triangular row-major order: t = bi (bi + 1) / 2 + bj, bj <= bi
    int r = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while ((long long)(r + 1) * (r + 2) / 2 <= t) ++r;
    while ((long long)r * (r + 1) / 2 > t) --r;
    bi = r;
    bj = (int)(t - (long long)r * (r + 1) / 2);
}

// ------------------------------------------------------------------ setup kernels
struct FillArgs {
    OperatorView op;
    double* W;          // batch x Np x Np
    int level0;         // first level of the batch (0-based; S = f-block)
    const double* diag; // S x Np: e0 * D1 / D2 (pads unused)
    const double* bscale; // per level: coefficient of B (cs, cr, or 0 for a D2 == 0 level)
};

__global__ void gj_fill(FillArgs f) {
    const long long Np = f.op.Np;
    const int b = blockIdx.y;
    const int L = f.level0 + b;
    double* W = f.W + (long long)b * Np * Np;
    const double scale = f.bscale[L];
    const int n1 = f.op.n1, n2 = f.op.n2, ld2 = f.op.ld2;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < Np * Np;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long i = idx / Np, j = idx % Np;
        const int i1 = (int)(i / ld2), i2 = (int)(i % ld2), j1 = (int)(j / ld2), j2 = (int)(j % ld2);
        double v;
        if (i2 >= n2 || j2 >= n2) {
            v = i == j ? 1.0 : 0.0;
        } else {
            v = scale * f.op.gen[(long long)(i1 - j1 + n1 - 1) * f.op.gen_stride + (i2 - j2) + ld2];
            if (i == j && L < f.op.S) v += f.diag[(long long)L * Np + i];
        }
        W[idx] = v;
    }
}

// In-place Gauss-Jordan inversion of the 64x64 pivot block of each matrix; records pivots.
__global__ void gj_diag_inv(double* W, long long Np, int K0, double* Dinv, double* piv) {
    __shared__ double D[TB][TB + 1];
    __shared__ double rowp[TB];
    __shared__ double colp[TB];
    const int b = blockIdx.x;
    const double* Wb = W + (long long)b * Np * Np;
    for (int idx = threadIdx.x; idx < TILE; idx += blockDim.x) {
        const int r = idx / TB, c = idx % TB;
        D[r][c] = Wb[(long long)(K0 + r) * Np + K0 + c];
    }
    __syncthreads();
    double pmin = piv[2 * b], pmax = piv[2 * b + 1];
    for (int p = 0; p < TB; ++p) {
        const double pv = D[p][p];
        if (threadIdx.x < TB) {
            const int c = threadIdx.x;
            rowp[c] = (c == p ? 1.0 : D[p][c]) / pv;
            colp[c] = D[c][p];
        }
        __syncthreads();
        for (int idx = threadIdx.x; idx < TILE; idx += blockDim.x) {
            const int r = idx / TB, c = idx % TB;
            D[r][c] = r == p ? rowp[c] : (c == p ? 0.0 : D[r][c]) - colp[r] * rowp[c];
        }
        __syncthreads();
        pmin = fmin(pmin, pv);
        pmax = fmax(pmax, fabs(pv));
    }
    for (int idx = threadIdx.x; idx < TILE; idx += blockDim.x) {
        const int r = idx / TB, c = idx % TB;
        Dinv[(long long)b * TILE + idx] = D[r][c];
    }
    if (threadIdx.x == 0) {
        piv[2 * b] = pmin;
        piv[2 * b + 1] = pmax;
    }
}

// Ftmp = W[:, K]  (Np x 64);  Rtmp = Dinv W[K, :] with Rtmp[:, K] = Dinv  (64 x Np)
__global__ void gj_panels(const double* W, long long Np, int K0, const double* Dinv, double* Ftmp, double* Rtmp) {
    __shared__ double Ds[TB][TB + 1];
    const int b = blockIdx.y;
    const long long j0 = (long long)blockIdx.x * TB;
    const double* Wb = W + (long long)b * Np * Np;
    const double* Db = Dinv + (long long)b * TILE;
    double* Fb = Ftmp + (long long)b * Np * TB;
    double* Rb = Rtmp + (long long)b * TB * Np;
    for (int idx = threadIdx.x; idx < TILE; idx += blockDim.x) {
        const int r = idx / TB, c = idx % TB;
        Ds[r][c] = Db[idx];
        // column panel rows j0 + r, columns K0 + c
        Fb[(j0 + r) * TB + c] = Wb[(j0 + r) * Np + K0 + c];
    }
    __syncthreads();
    const bool pivot_block = j0 == K0;
    for (int idx = threadIdx.x; idx < TILE; idx += blockDim.x) {
        const int r = idx / TB, c = idx % TB;
        double v;
        if (pivot_block) {
            v = Ds[r][c];
        } else {
            v = 0.0;
            const double* wc = Wb + (long long)K0 * Np + j0 + c;
#pragma unroll 8
            for (int l = 0; l < TB; ++l) v += Ds[r][l] * __ldg(wc + (long long)l * Np);
        }
        Rb[(long long)r * Np + j0 + c] = v;
    }
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// W[i][j] = (i in K) ? Rtmp[i-K0][j] : ((j in K) ? 0 : W[i][j]) - sum_k Ftmp[i][k] Rtmp[k][j]
// 64x64 output tile per CTA, 256 threads, DMMA m8n8k4 (warp tile 32x16).
__global__ void __launch_bounds__(256) gj_update(double* W, long long Np, int K0, const double* Ftmp,
                                                 const double* Rtmp) {
    constexpr int KH = TB / 2;
    __shared__ double Fs[TB][KH + 4];  // [i][k]
    __shared__ double Rs[TB][KH + 4];  // [j][k] (transposed)
    const int b = blockIdx.z;
    const long long i0 = (long long)blockIdx.y * TB, j0 = (long long)blockIdx.x * TB;
    double* Wb = W + (long long)b * Np * Np;
    const double* Rb = Rtmp + (long long)b * TB * Np;
    if (i0 == K0) {
        for (int idx = threadIdx.x; idx < TILE; idx += blockDim.x) {
            const int r = idx / TB, c = idx % TB;
            Wb[(i0 + r) * Np + j0 + c] = Rb[(long long)r * Np + j0 + c];
        }
        return;
    }
    const double* Fb = Ftmp + (long long)b * Np * TB;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm0 = (warp & 1) * 32, wn0 = (warp >> 1) * 16;
    double acc[4][2][2] = {};
    for (int kh = 0; kh < TB; kh += KH) {
        __syncthreads();
        for (int idx = threadIdx.x; idx < TB * KH; idx += blockDim.x) {
            const int r = idx / KH, k = idx % KH;
            Fs[r][k] = Fb[(i0 + r) * TB + kh + k];
            const int k2 = idx / TB, c = idx % TB;
            Rs[c][k2] = Rb[(long long)(kh + k2) * Np + j0 + c];
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < KH / 4; ++kk) {
            double av[4], bv[2];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) av[mi] = Fs[wm0 + 8 * mi + g][4 * kk + t];
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) bv[ni] = Rs[wn0 + 8 * ni + g][4 * kk + t];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni], av[mi], bv[ni]);
        }
    }
    const bool pivot_col = j0 == K0;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const long long i = i0 + wm0 + 8 * mi + g;
                const long long j = j0 + wn0 + 8 * ni + 2 * t + c;
                double* p = Wb + i * Np + j;
                *p = (pivot_col ? 0.0 : *p) - acc[mi][ni][c];
            }
}

// Pack the lower-triangular 64x64 tiles of each inverse, zeroing padded rows/columns.
__global__ void pack_tiles(const double* W, long long Np, int n2, int ld2, long long T, double* Hout, float* Hfout) {
    const int b = blockIdx.y;
    const double* Wb = W + (long long)b * Np * Np;
    double* Hb = Hout + (long long)b * T * TILE;
    float* Hfb = Hfout + (long long)b * T * TILE;
    for (long long t = blockIdx.x; t < T; t += gridDim.x) {
        int bi, bj;
        tile_coords(t, bi, bj);
        for (int idx = threadIdx.x; idx < TILE; idx += blockDim.x) {
            const int r = idx / TB, c = idx % TB;
            const long long i = (long long)bi * TB + r, j = (long long)bj * TB + c;
            const bool pad = (int)(i % ld2) >= n2 || (int)(j % ld2) >= n2;
            const double v = pad ? 0.0 : Wb[i * Np + j];
            Hb[t * TILE + idx] = v;
            Hfb[t * TILE + idx] = (float)v;
        }
    }
}

__global__ void fwd_rhs_kernel(long long Np, int S, const double* D1, const double* b, const double* q, double eta,
                               const double* rho, const double* f, double* z) {
    // z_s = b_{s-1} D1_s o rho + eta q_s f   (system.cpp:209-210), padded layout, levels 0..S-1
    const long long n = (long long)S * Np;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        const int s = (int)(idx / Np);
        const long long i = idx % Np;
        z[idx] = b[s] * (D1[idx] * rho[i]) + eta * q[s] * f[i];
    }
}

}  // namespace

void precond_build(fi_precond* P) {
    fi_system* sys = P->sys;
    fi_ctx* ctx = sys->ctx;
    const Layout& L = sys->L;
    const int S = L.S;
    const long long N = L.N, Np = L.Np;
    const double e0 = sys->e_h[0];

    // --- block admissibility in the reference's level order (krylov.cpp:35-45).  A level whose
    // D2 vanishes identically has G_s = e0 D1 (diagonal); otherwise D2 must be nonzero with
    // D1/D2 >= 0 so that M = cs B + e0 diag(D1/D2) is symmetric positive definite.
    std::vector<double> diag((size_t)S * Np, 0.0), d2inv((size_t)S * Np, 0.0), bscale((size_t)S + 1, sys->cs);
    bscale[(size_t)S] = sys->cr;
    for (int s = 1; s <= S; ++s) {
        bool all_zero = true;
        for (long long j = 0; j < N; ++j) all_zero = all_zero && sys->D2_h[(size_t)(s - 1) * N + j] == 0.0;
        if (all_zero) bscale[(size_t)s - 1] = 0.0;
        for (long long j = 0; j < N; ++j) {
            const long long i1 = j / L.n2, i2 = j % L.n2;
            const long long p = (long long)(s - 1) * Np + i1 * L.ld2 + i2;
            const double d1 = sys->D1_h[(size_t)(s - 1) * N + j], d2 = sys->D2_h[(size_t)(s - 1) * N + j];
            if (all_zero) {
                if (d1 == 0.0 || e0 == 0.0)
                    throw Error(FI_E_SINGULAR, "precond_build: singular block at time level " + std::to_string(s), s);
                diag[p] = e0 * d1;
                d2inv[p] = 1.0;
                continue;
            }
            if (d2 == 0.0) {
                if (d1 == 0.0 || e0 == 0.0)
                    throw Error(FI_E_SINGULAR, "precond_build: singular block at time level " + std::to_string(s), s);
                throw Error(FI_E_DOMAIN, "precond_build: gamma2 vanishes at part of level " + std::to_string(s) +
                                             "; the symmetric block form needs gamma2 != 0 or gamma2 == 0 everywhere");
            }
            if (d1 / d2 < 0.0)
                throw Error(FI_E_DOMAIN, "precond_build: gamma1/gamma2 < 0 at level " + std::to_string(s) +
                                             "; the symmetric block form needs gamma1/gamma2 >= 0");
            diag[p] = e0 * d1 / d2;
            d2inv[p] = 1.0 / d2;
        }
    }
    for (long long j = 0; j < N; ++j)
        if (sys->D2_h[(size_t)(S - 1) * N + j] == 0.0)
            throw Error(FI_E_SINGULAR, "precond_build: singular block at time level " + std::to_string(S + 1), S + 1);

    P->nb = (int)(Np / TB);
    P->T = (long long)P->nb * (P->nb + 1) / 2;
    P->levels = S + 1;
    // dense blocks in HODLR form when the sweep supports the shape (FI_HODLR=0: packed tiles)
    static const bool hodlr_env = [] {
        const char* v = std::getenv("FI_HODLR");
        return v ? std::atoi(v) != 0 : true;
    }();
    bool use_hodlr = hodlr_env && hodlr_supported(L, S + 1, ctx->sm_count);
    P->rbuf.alloc((size_t)L.nI());
    P->dbuf.alloc((size_t)L.nI());
    P->d2inv.alloc((size_t)S * Np);
    P->xbuf.alloc((size_t)2 * Np);
    P->pbuf.alloc((size_t)2 * P->nb * P->nb * TB);
    P->counters.alloc(((size_t)2 * P->nb + 1) * kCounterStride);
    FI_CUDA(cudaMemcpyAsync(P->d2inv.p, d2inv.data(), d2inv.size() * sizeof(double), cudaMemcpyHostToDevice,
                            ctx->stream));
    DevBuf<double> diag_d((size_t)S * Np), bscale_d((size_t)S + 1);
    FI_CUDA(cudaMemcpyAsync(diag_d.p, diag.data(), diag.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    FI_CUDA(cudaMemcpyAsync(bscale_d.p, bscale.data(), bscale.size() * sizeof(double), cudaMemcpyHostToDevice,
                            ctx->stream));

    P->G = precond_apply_grid(ctx, P->T, Np);

    // --- batched Gauss-Jordan inversion of M_L for all levels
    const size_t mat = (size_t)Np * Np;
    size_t free_b = 0, total_b = 0;
    FI_CUDA(cudaMemGetInfo(&free_b, &total_b));
    long long batch = (long long)std::min<size_t>(16, std::max<size_t>(1, (free_b / 4) / (mat * sizeof(double))));
    batch = std::min<long long>(batch, S + 1);
    DevBuf<double> W((size_t)batch * mat), Ftmp((size_t)batch * Np * TB), Rtmp((size_t)batch * TB * Np),
        Dinv((size_t)batch * TILE), piv((size_t)batch * 2);
    std::vector<double> piv_h((size_t)batch * 2);
    const OperatorView op = sys->view();
    // The inverses are polished (precond_polish.cu) to LU-solve accuracy, so one sweep per apply
    // suffices (refinement off by default; FI_POLISH=0 restores the unpolished inverses + refinement).
    const bool polish = polish_enabled();
    P->refine = polish ? 0 : 1;
    // One pass over all levels; the HODLR pass checks every batch a posteriori (probe vector,
    // |H x - H_hodlr x| <= 1e-12 |H x|) and, if the rank does not suffice, the build restarts with
    // packed tiles.
    double check_fwd = 0.0, check_bwd = 0.0;
    auto build_pass = [&](bool hodlr) -> bool {
        DevBuf<double> hwork;
        if (hodlr) {
            P->hodlr = hodlr_create(L, S + 1);
            hwork.alloc(std::max(hodlr_work_doubles(L, (int)batch), (size_t)batch * (2 * 64 * 2 * 32 + 2)));
        } else {
            P->H.alloc((size_t)(S + 1) * P->T * TILE);
            P->Hf.alloc((size_t)(S + 1) * P->T * TILE);
        }
        DevBuf<double> pwork;
        if (polish) pwork.alloc(polish_work_doubles(Np, (int)batch));
        int first_singular = 0;
        for (long long l0 = 0; l0 < S + 1; l0 += batch) {
            const int nbt = (int)std::min<long long>(batch, S + 1 - l0);
            for (int b = 0; b < nbt; ++b) {
                piv_h[2 * b] = INFINITY;
                piv_h[2 * b + 1] = 0.0;
            }
            FI_CUDA(cudaMemcpyAsync(piv.p, piv_h.data(), 2 * nbt * sizeof(double), cudaMemcpyHostToDevice,
                                    ctx->stream));
            FillArgs fa{op, W.p, (int)l0, diag_d.p, bscale_d.p};
            gj_fill<<<dim3((unsigned)std::min<long long>(4096, (Np * Np + 255) / 256), nbt), 256, 0, ctx->stream>>>(fa);
            FI_LAUNCHED(ctx);
            for (int K = 0; K < P->nb; ++K) {
                const int K0 = K * TB;
                gj_diag_inv<<<nbt, 256, 0, ctx->stream>>>(W.p, Np, K0, Dinv.p, piv.p);
                FI_LAUNCHED(ctx);
                gj_panels<<<dim3(P->nb, nbt), 256, 0, ctx->stream>>>(W.p, Np, K0, Dinv.p, Ftmp.p, Rtmp.p);
                FI_LAUNCHED(ctx);
                gj_update<<<dim3(P->nb, P->nb, nbt), 256, 0, ctx->stream>>>(W.p, Np, K0, Ftmp.p, Rtmp.p);
                FI_LAUNCHED(ctx);
            }
            if (polish) polish_inverses(ctx, op, W.p, nbt, (int)l0, bscale_d.p, pwork.p);
            if (hodlr) {
                hodlr_compress(ctx, P->hodlr, L, W.p, nbt, (int)l0, hwork.p);
            } else {
                pack_tiles<<<dim3((unsigned)std::min<long long>(P->T, 4096), nbt), 256, 0, ctx->stream>>>(
                    W.p, Np, L.n2, L.ld2, P->T, P->H.p + (size_t)l0 * P->T * TILE, P->Hf.p + (size_t)l0 * P->T * TILE);
                FI_LAUNCHED(ctx);
            }
            FI_CUDA(cudaMemcpyAsync(piv_h.data(), piv.p, 2 * nbt * sizeof(double), cudaMemcpyDeviceToHost,
                                    ctx->stream));
            FI_CUDA(cudaStreamSynchronize(ctx->stream));
            for (int b = 0; b < nbt && !first_singular; ++b) {
                const double pmin = piv_h[2 * b], pmax = piv_h[2 * b + 1];
                if (!(pmax > 0.0) || !(pmin > 1e-14 * pmax)) first_singular = (int)(l0 + b) + 1;
            }
            if (first_singular)
                throw Error(FI_E_SINGULAR,
                            "precond_build: singular block at time level " + std::to_string(first_singular),
                            first_singular);
            if (hodlr) {
                double bwd = 0.0;
                const double fwd = hodlr_check(ctx, P->hodlr, L, W.p, nbt, (int)l0, hwork.p, op, diag_d.p,
                                               bscale_d.p, &bwd);
                check_fwd = std::max(check_fwd, fwd);
                check_bwd = std::max(check_bwd, bwd);
                if (!(fwd <= 1e-12) || !(bwd <= kHodlrBackwardTol)) {
                    hodlr_destroy(P->hodlr);
                    P->hodlr = nullptr;
                    return false;
                }
            }
        }
        return true;
    };
    if (!(use_hodlr && build_pass(true))) build_pass(false);
    P->hodlr_check_fwd = check_fwd;
    P->hodlr_check_bwd = check_bwd;
}

}  // namespace fib

// forward solve helper (used by abi.cu)
namespace fib {
void forward_rhs(fi_ctx* ctx, const fi_system* sys, const double* rho_pad, const double* f_pad, double* z_pad) {
    fwd_rhs_kernel<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(sys->L.Np, sys->L.S, sys->D1.p, sys->bw.p,
                                                             sys->q.p, sys->eta, rho_pad, f_pad, z_pad);
    FI_LAUNCHED(ctx);
}
}  // namespace fib
