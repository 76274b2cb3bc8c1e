// K1f — the all-at-once operator apply Z = A U with the spatial Toeplitz products by FFT (2D systems).
//
// The reference applies B = K (the multilevel Toeplitz fractional Laplacian) with a circulant embedding
// and two FFTs per call (toeplitz.cpp:68-114), S + 1 times per SystemOperator::apply (system.cpp:144-174).
// K1 (toeplitz_apply.cu) instead forms K U as one dense FP64 DMMA contraction, 2 N^2 (S + 1) FLOP: 1.7e10
// for the 1D config 1, but 4.3e12 for the 2D 255 x 255 grids, where the transforms are ~180x less work.
// K1f keeps K1's fused time convolution (the U E^T DMMA product with E generated from the L1 weights, the
// D1 scaling and the -eta q f coupling; conv-only mode of K1, on the side stream) and does K u_s for all
// S + 1 columns as batched 2D transforms of size L1 x L2 = 2(n1 + 1) x 2(n2 + 1):
//   rows_fwd  (level, row pair): real rows packed two per complex FFT, split into two half spectra -> W
//   cols      (level, 4 adjacent half-spectrum columns): column FFT, x lambda_B, inverse column FFT -> W
//   rows_inv  (level, row pair): the two rows' half spectra packed into one inverse FFT -> K u, and the
//             epilogue Z[:, s] += cs D2_s o K u_s (s < S),  Z[:, S] = u_{S-1} + cr D2_{S-1} o K f
// lambda_B is the real spectrum of the embedded generating tensor, computed at system creation with the
// same transforms as the tau-PCG preconditioner's (precond_iter.cu).  The Stockham FFT groups are shared
// with K5 (fft_dev.cuh).
#include <cmath>
#include <vector>

#include "fft_dev.cuh"
#include "system.cuh"

namespace fib {
namespace {

#ifndef FI_FFTOP_T
#define FI_FFTOP_T 128  // 128: 3.37 ms on config 4, 256: 3.48 ms (occupancy: 41 KB of shared memory per CTA)
#endif
constexpr int FFT_T = FI_FFTOP_T;  // threads per CTA: groups of L/8 threads (FFT_T / 64 groups at L = 512)

struct FftOpArgs {
    int n1, n2, ld2, S, L1, L2, lg1, lg2, H2, nup;
    long long Np;
    const double* U;
    double* Z;
    const double* minus_from;
    const double* D1;
    const double* D2;
    double cs, cr, inv_LL;
    const double2* tw1;   // exp(-2 pi i k / L1), k < L1 (full table)
    const double2* tw2;
    const double* lamB;   // L1 x L2 real spectrum of the embedded generating tensor
    double2* W;           // [(S + 1)][n1][H2] half spectra
    const int* skip;
};

// the stage twiddle table (fft_dev.cuh) of length L = 2^lg from the full table exp(-2 pi i k / L)
__device__ __forceinline__ void load_twiddles(double2* dst, const double2* src, int lg) {
    fft_stage_twiddles(dst, lg, [&](int k) { return src[k]; });
}

// row pairs (2p, 2p + 1) of column (level) l of U, forward FFT along the rows, half spectra -> W
__global__ void __launch_bounds__(FFT_T) fftop_rows_fwd(FftOpArgs a) {
    if (a.skip && *a.skip) return;
    extern __shared__ double2 smf[];
    const int L = a.L2, nt = max(L >> 3, 1), ng = FFT_T / nt, PL = pad8(L) + 1;
    double2* tw = smf;
    double2* gb = smf + L;
    load_twiddles(tw, a.tw2, a.lg2);
    const int tid = threadIdx.x, g = tid / nt, t = tid % nt;
    const long long units = (long long)(a.S + 1) * a.nup;
    const long long u0 = (long long)blockIdx.x * ng;
    // fill: all threads of the CTA, element e = (group, j); pairs (row 2p in .x, row 2p + 1 in .y)
    for (int e = tid; e < ng * L; e += FFT_T) {
        const int gg = e / L, j = e - gg * L;
        const long long u = u0 + gg;
        double2 v = make_double2(0.0, 0.0);
        if (u < units && j < a.n2) {
            const int l = (int)(u / a.nup), p = (int)(u % a.nup);
            const double* src = a.U + (long long)l * a.Np + (long long)(2 * p) * a.ld2 + j;
            v.x = src[0];
            if (2 * p + 1 < a.n1) v.y = src[a.ld2];
        }
        gb[(size_t)gg * 2 * PL + pad8(j)] = v;
    }
    __syncthreads();
    const long long u = u0 + g;
    const bool act = u < units;
    const int w = fft_dispatch(gb + (size_t)g * 2 * PL, gb + (size_t)g * 2 * PL + PL, a.lg2, tw, false, t, act);
    // split the packed spectrum P = X0 + i X1 into the two Hermitian half spectra, k = 0 .. L/2
    for (int e = tid; e < ng * a.H2; e += FFT_T) {
        const int gg = e / a.H2, k = e - gg * a.H2;
        const long long uu = u0 + gg;
        if (uu >= units) continue;
        const int l = (int)(uu / a.nup), p = (int)(uu % a.nup);
        const double2* buf = gb + (size_t)gg * 2 * PL + (size_t)w * PL;
        const double2 P = buf[pad8(k)], Qc = buf[pad8((L - k) & (L - 1))];
        double2* dst = a.W + ((long long)l * a.n1 + 2 * p) * a.H2 + k;
        dst[0] = make_double2(0.5 * (P.x + Qc.x), 0.5 * (P.y - Qc.y));
        if (2 * p + 1 < a.n1) dst[a.H2] = make_double2(0.5 * (P.y + Qc.y), -0.5 * (P.x - Qc.x));
    }
}

// 4 adjacent half-spectrum columns k0.. of level l: column FFT (zero rows beyond n1), x lambda_B, inverse
// column FFT, rows < n1 back into W
__global__ void __launch_bounds__(FFT_T) fftop_cols(FftOpArgs a) {
    if (a.skip && *a.skip) return;
    extern __shared__ double2 smf[];
    const int L = a.L1, nt = max(L >> 3, 1), ng = FFT_T / nt, PL = pad8(L) + 1;
    double2* tw = smf;
    double2* gb = smf + L;
    double* lam = reinterpret_cast<double*>(gb + (size_t)ng * 2 * PL);  // [ng][L]
    load_twiddles(tw, a.tw1, a.lg1);
    const int tid = threadIdx.x, g = tid / nt, t = tid % nt;
    const int cpl = (a.H2 + ng - 1) / ng;  // column groups per level
    const int l = blockIdx.x / cpl, k0 = (blockIdx.x % cpl) * ng;
    const double2* Wl = a.W + (long long)l * a.n1 * a.H2;
    // fill: lane-interleaved over the ng adjacent columns (whole sectors of a row)
    for (int e = tid; e < ng * L; e += FFT_T) {
        const int gg = e % ng, j = e / ng, k = k0 + gg;
        double2 v = make_double2(0.0, 0.0);
        double lm = 0.0;
        if (k < a.H2) {
            if (j < a.n1) v = Wl[(long long)j * a.H2 + k];
            lm = a.lamB[(long long)j * a.L2 + k];
        }
        gb[(size_t)gg * 2 * PL + pad8(j)] = v;
        lam[gg * L + j] = lm;
    }
    __syncthreads();
    const bool act = k0 + g < a.H2;
    const int w = fft_dispatch(gb + (size_t)g * 2 * PL, gb + (size_t)g * 2 * PL + PL, a.lg1, tw, false, t, act);
    for (int e = tid; e < ng * L; e += FFT_T) {
        const int gg = e / L, j = e - gg * L;
        double2* c = gb + (size_t)gg * 2 * PL + (size_t)w * PL + pad8(j);
        const double lm = lam[gg * L + j];
        const double2 v = *c;
        *c = make_double2(v.x * lm, v.y * lm);
    }
    __syncthreads();
    const int w2 = w ^ fft_dispatch(gb + (size_t)g * 2 * PL + (size_t)w * PL, gb + (size_t)g * 2 * PL + (size_t)(1 - w) * PL,
                                    a.lg1, tw, true, t, act);
    double2* Wo = a.W + (long long)l * a.n1 * a.H2;
    for (int e = tid; e < ng * a.n1; e += FFT_T) {
        const int gg = e % ng, j = e / ng, k = k0 + gg;
        if (k < a.H2) Wo[(long long)j * a.H2 + k] = gb[(size_t)gg * 2 * PL + (size_t)w2 * PL + pad8(j)];
    }
}

// row pairs of level l: inverse FFT of the packed half spectra -> K u of rows 2p, 2p + 1; epilogue
__global__ void __launch_bounds__(FFT_T) fftop_rows_inv(FftOpArgs a) {
    if (a.skip && *a.skip) return;
    extern __shared__ double2 smf[];
    const int L = a.L2, nt = max(L >> 3, 1), ng = FFT_T / nt, PL = pad8(L) + 1;
    double2* tw = smf;
    double2* gb = smf + L;
    load_twiddles(tw, a.tw2, a.lg2);
    const int tid = threadIdx.x, g = tid / nt, t = tid % nt;
    const long long units = (long long)(a.S + 1) * a.nup;
    const long long u0 = (long long)blockIdx.x * ng;
    for (int e = tid; e < ng * L; e += FFT_T) {
        const int gg = e / L, k = e - gg * L;
        const long long u = u0 + gg;
        double2 v = make_double2(0.0, 0.0);
        if (u < units) {
            const int l = (int)(u / a.nup), p = (int)(u % a.nup);
            const int kk = k <= L / 2 ? k : L - k;
            const double2* src = a.W + ((long long)l * a.n1 + 2 * p) * a.H2 + kk;
            double2 y0 = src[0];
            double2 y1 = 2 * p + 1 < a.n1 ? src[a.H2] : make_double2(0.0, 0.0);
            if (kk == 0 || kk == L / 2) {
                y0.y = 0.0;
                y1.y = 0.0;
            }
            if (k > L / 2) {
                y0.y = -y0.y;
                y1.y = -y1.y;
            }
            v = make_double2(y0.x - y1.y, y0.y + y1.x);
        }
        gb[(size_t)gg * 2 * PL + pad8(k)] = v;
    }
    __syncthreads();
    const long long u = u0 + g;
    const bool act = u < units;
    const int w = fft_dispatch(gb + (size_t)g * 2 * PL, gb + (size_t)g * 2 * PL + PL, a.lg2, tw, true, t, act);
    // epilogue over the ld2-wide rows (pad columns: 0, or minus_from's value)
    for (int e = tid; e < ng * 2 * a.ld2; e += FFT_T) {
        const int gg = e / (2 * a.ld2), r2 = e - gg * 2 * a.ld2, h = r2 / a.ld2, j = r2 - h * a.ld2;
        const long long uu = u0 + gg;
        if (uu >= units) continue;
        const int l = (int)(uu / a.nup), p = (int)(uu % a.nup), row = 2 * p + h;
        if (row >= a.n1) continue;
        const long long ro = (long long)row * a.ld2 + j, o = (long long)l * a.Np + ro;
        const double2 c = gb[(size_t)gg * 2 * PL + (size_t)w * PL + pad8(j)];
        const double ku = (h ? c.y : c.x) * a.inv_LL;
        if (l < a.S) {
            // Z already holds D1 o conv - eta q f (or minus_from minus that), written by the conv kernel
            if (j < a.n2) {
                const double add = a.cs * a.D2[(long long)l * a.Np + ro] * ku;
                a.Z[o] = a.minus_from ? a.Z[o] - add : a.Z[o] + add;
            }
        } else {
            double out = 0.0;
            if (j < a.n2) {
                const long long dl = (long long)(a.S - 1) * a.Np + ro;
                out = a.U[dl] + a.cr * a.D2[dl] * ku;
            }
            a.Z[o] = a.minus_from ? a.minus_from[o] - out : out;
        }
    }
}

// lambda_B: real spectrum of the circulant embedding of the generating tensor (c[k1][k2] = a[l1][l2],
// l_i = k_i or k_i - L_i), by a plain 2D FFT (setup only)
__global__ void fftop_embed(OperatorView op, int L1, int L2, double2* X) {
    const long long tot = (long long)L1 * L2;
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < tot; q += (long long)gridDim.x * blockDim.x) {
        const int k1 = (int)(q / L2), k2 = (int)(q % L2);
        const int l1 = k1 < op.n1 ? k1 : (k1 > L1 - op.n1 ? k1 - L1 : 1 << 30);
        const int l2 = k2 < op.n2 ? k2 : (k2 > L2 - op.n2 ? k2 - L2 : 1 << 30);
        double v = 0.0;
        if (l1 != (1 << 30) && l2 != (1 << 30)) v = op.gen[(long long)(l1 + op.n1 - 1) * op.gen_stride + l2 + op.ld2];
        X[q] = make_double2(v, 0.0);
    }
}
// one length-L FFT per CTA along rows (stride 1) or columns (stride L2) of X, in place; real part to
// lam when lam != nullptr
__global__ void fftop_plain(double2* X, int L, int lg, long long stride, long long step, const double2* tw,
                            double* lam) {
    extern __shared__ double2 smf[];
    const int nt = max(L >> 3, 1), PL = pad8(L) + 1;
    double2* tws = smf;
    double2* gb = smf + L;
    load_twiddles(tws, tw, lg);
    double2* base = X + (long long)blockIdx.x * step;
    for (int j = threadIdx.x; j < L; j += blockDim.x) gb[pad8(j)] = base[(long long)j * stride];
    __syncthreads();
    const int t = threadIdx.x;
    const int w = fft_dispatch(gb, gb + PL, lg, tws, false, t < nt ? t : 0, t < nt);
    for (int j = threadIdx.x; j < L; j += blockDim.x) {
        const double2 v = gb[(size_t)w * PL + pad8(j)];
        if (lam) lam[(long long)blockIdx.x * step + (long long)j * stride] = v.x;
        else base[(long long)j * stride] = v;
    }
}

int ilog2i(int v) {
    int l = 0;
    while ((1 << l) < v) ++l;
    return l;
}

size_t smem_rows(int L) {
    const int nt = std::max(L >> 3, 1), ng = FFT_T / nt;
    return ((size_t)L + (size_t)ng * 2 * (L + L / 8 + 1)) * sizeof(double2);
}
size_t smem_cols(int L) {
    const int nt = std::max(L >> 3, 1), ng = FFT_T / nt;
    return smem_rows(L) + (size_t)ng * L * sizeof(double);
}

}  // namespace

bool fft_apply_supported(const Layout& L) {
    if (L.d != 2) return false;
    const int a = L.n1 + 1, b = L.n2 + 1;
    return (a & (a - 1)) == 0 && (b & (b - 1)) == 0 && 2 * a >= 8 && 2 * b >= 8 && 2 * a <= 1024 && 2 * b <= 1024;
}

void fft_apply_prepare(fi_system* sys) {
    if (sys->fft_ready) return;
    fi_ctx* ctx = sys->ctx;
    const Layout& L = sys->L;
    const int L1 = 2 * (L.n1 + 1), L2 = 2 * (L.n2 + 1), H2 = L2 / 2 + 1;
    std::vector<double2> t1((size_t)L1), t2((size_t)L2);
    for (int k = 0; k < L1; ++k) t1[(size_t)k] = make_double2(std::cos(2.0 * M_PI * k / L1), -std::sin(2.0 * M_PI * k / L1));
    for (int k = 0; k < L2; ++k) t2[(size_t)k] = make_double2(std::cos(2.0 * M_PI * k / L2), -std::sin(2.0 * M_PI * k / L2));
    sys->fft_tw1.alloc((size_t)L1);
    sys->fft_tw2.alloc((size_t)L2);
    FI_CUDA(cudaMemcpy(sys->fft_tw1.p, t1.data(), t1.size() * sizeof(double2), cudaMemcpyHostToDevice));
    FI_CUDA(cudaMemcpy(sys->fft_tw2.p, t2.data(), t2.size() * sizeof(double2), cudaMemcpyHostToDevice));
    sys->fft_lamB.alloc((size_t)L1 * L2);
    sys->fft_W.alloc((size_t)(L.S + 1) * L.n1 * H2);
    DevBuf<double2> X((size_t)L1 * L2);
    const OperatorView op = sys->view();
    fftop_embed<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(op, L1, L2, X.p);
    FI_LAUNCHED(ctx);
    ensure_smem_attr((const void*)fftop_plain, (size_t)(std::max(L1, L2) + 2 * (std::max(L1, L2) + std::max(L1, L2) / 8 + 1)) * sizeof(double2));
    // rows (stride 1, one row per CTA), then columns (stride L2) with the real part out
    fftop_plain<<<L1, 128, (L2 + 2 * (L2 + L2 / 8 + 1)) * sizeof(double2), ctx->stream>>>(X.p, L2, ilog2i(L2), 1, L2,
                                                                                          sys->fft_tw2.p, nullptr);
    FI_LAUNCHED(ctx);
    fftop_plain<<<L2, 128, (L1 + 2 * (L1 + L1 / 8 + 1)) * sizeof(double2), ctx->stream>>>(X.p, L1, ilog2i(L1), L2, 1,
                                                                                          sys->fft_tw1.p, sys->fft_lamB.p);
    FI_LAUNCHED(ctx);
    FI_CUDA(cudaStreamSynchronize(ctx->stream));
    (void)H2;
    sys->fft_ready = true;
}

void toeplitz_apply_fft(fi_ctx* ctx, fi_system* sys, const double* U, double* Z, const int* skip,
                        const double* minus_from, bool precond_matrix) {
    const Layout& L = sys->L;
    const OperatorView op = sys->view();
    FftOpArgs a{};
    a.n1 = L.n1;
    a.n2 = L.n2;
    a.ld2 = L.ld2;
    a.S = L.S;
    a.L1 = 2 * (L.n1 + 1);
    a.L2 = 2 * (L.n2 + 1);
    a.lg1 = ilog2i(a.L1);
    a.lg2 = ilog2i(a.L2);
    a.H2 = a.L2 / 2 + 1;
    a.nup = (L.n1 + 1) / 2;
    a.Np = L.Np;
    a.U = U;
    a.Z = Z;
    a.minus_from = minus_from;
    a.D1 = op.D1;
    a.D2 = op.D2;
    a.cs = op.cs;
    a.cr = op.cr;
    a.inv_LL = 1.0 / ((double)a.L1 * a.L2);
    a.tw1 = sys->fft_tw1.p;
    a.tw2 = sys->fft_tw2.p;
    a.lamB = sys->fft_lamB.p;
    a.W = sys->fft_W.p;
    a.skip = skip;
    // the time convolution (K1 in conv-only mode, DMMA) on the side stream, overlapping the transforms
    FI_CUDA(cudaEventRecord(ctx->fork, ctx->stream));
    FI_CUDA(cudaStreamWaitEvent(ctx->side, ctx->fork, 0));
    toeplitz_conv_apply(ctx, op, U, Z, skip, minus_from, precond_matrix, ctx->side);
    FI_CUDA(cudaEventRecord(ctx->join, ctx->side));
    const int ngr = FFT_T / std::max(a.L2 >> 3, 1), ngc = FFT_T / std::max(a.L1 >> 3, 1);
    const size_t smr = smem_rows(a.L2), smc = smem_cols(a.L1);
    ensure_smem_attr((const void*)fftop_rows_fwd, smr);
    ensure_smem_attr((const void*)fftop_rows_inv, smr);
    ensure_smem_attr((const void*)fftop_cols, smc);
    const long long units = (long long)(L.S + 1) * a.nup;
    const unsigned gr = (unsigned)((units + ngr - 1) / ngr);
    fftop_rows_fwd<<<gr, FFT_T, smr, ctx->stream>>>(a);
    FI_LAUNCHED(ctx);
    const unsigned gc = (unsigned)((L.S + 1) * ((a.H2 + ngc - 1) / ngc));
    fftop_cols<<<gc, FFT_T, smc, ctx->stream>>>(a);
    FI_LAUNCHED(ctx);
    FI_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->join, 0));
    fftop_rows_inv<<<gr, FFT_T, smr, ctx->stream>>>(a);
    FI_LAUNCHED(ctx);
}

void system_apply(fi_ctx* ctx, fi_system* sys, const double* U, double* Z, const int* skip, const double* minus_from,
                  bool precond_matrix) {
    if (sys->use_fft()) {
        fft_apply_prepare(sys);
        toeplitz_apply_fft(ctx, sys, U, Z, skip, minus_from, precond_matrix);
    } else {
        toeplitz_apply(ctx, sys->view(), U, Z, skip, minus_from, precond_matrix);
    }
}

}  // namespace fib
