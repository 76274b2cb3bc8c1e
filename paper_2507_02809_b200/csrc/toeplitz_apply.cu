// K1 — all-at-once operator apply Z = A U as one FP64 DMMA GEMM with a fused epilogue.
//
// Replaces SystemOperator::apply (system.cpp:144-174), which calls the FFT Toeplitz
// matvec (toeplitz.cpp:75-114) S+1 times and re-sums the L1 history per level.
//
// With U = [y^(1) ... y^(S) f] (Np x (S+1), column s = level s+1, padded layout):
//   acc1 = K U              K = B (multilevel Toeplitz), generated per tile from the
//                           generating tensor in shared memory — never stored N x N
//   acc2 = U E^T            E lower-triangular Toeplitz of the L1 weights e (time conv.)
//   Z[:, s] = D1_s o acc2[:, s] + cs D2_s o acc1[:, s] - eta q_s f      (s < S)
//   Z[:, S] = y^(S) + cr D2_S o acc1[:, S]                               (f-block)
// Both products run on the FP64 tensor pipe (mma.sync m8n8k4 f64 -> DMMA.8x8x4; tcgen05
// has no f64 kind).  Operand tiles are staged by a 4-stage cp.async pipeline; the
// epilogue reads D1/D2/f once per output element, so each Krylov vector makes one HBM
// round trip (north-star (a)+(b)).
#include "system.cuh"

namespace fib {
namespace {

constexpr int BM = 64;       // rows (space i) per CTA tile
constexpr int BN = 64;       // columns (time level s) per CTA tile
constexpr int BK = 32;       // reduction depth per pipeline stage
constexpr int NSTAGE = 4;
constexpr int NTHREADS = 256;  // 8 warps: 2 (m) x 4 (n), warp tile 32 x 16
constexpr int LDJ = BK + 4;    // Us[s][j]  (j fastest), conflict-free B fragments
constexpr int LDI = BM + 4;    // Ut[m][i]  (i fastest), conflict-free A fragments
constexpr int SEG = 96;        // >= BM + BK - 1 and >= BN + BK - 1
constexpr int STAGE_DBL = (BN * LDJ > BK * LDI ? BN * LDJ : BK * LDI) + SEG;
constexpr int LDC = BM + 2;    // epilogue staging
constexpr int SMEM_BYTES =
    (NSTAGE * STAGE_DBL > 2 * BN * LDC ? NSTAGE * STAGE_DBL : 2 * BN * LDC) * (int)sizeof(double);

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, bool valid) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

struct TileCtx {
    int i0, s0;           // tile origin (padded row, column)
    int i1, i2_0;         // i0 = i1*ld2 + i2_0
    int nconv, nmain;     // pipeline stages of each kind
    int nbj2;             // valid BK-blocks per j1 row
};

__device__ __forceinline__ void load_stage(const OperatorView& op, const double* __restrict__ U, const TileCtx& tc,
                                           double* stage, int it) {
    const int tid = threadIdx.x;
    double* seg = stage + (STAGE_DBL - SEG);
    if (it < tc.nconv) {
        // conv stage: Ut[m][i] = U[(m0+m)*Np + i0 + i], eseg[x] = e[s0 - m0 - (BK-1) + x]
        const int m0 = it * BK;
        for (int c = tid; c < BK * BM / 2; c += NTHREADS) {
            const int ml = c / (BM / 2), ip = c % (BM / 2);
            const int m = m0 + ml;
            const bool valid = m < op.S;  // the f column never enters the time convolution
            const double* src = valid ? U + (long long)m * op.Np + tc.i0 + 2 * ip : U;
            cp_async16(stage + ml * LDI + 2 * ip, src, valid);
        }
        if (tid < SEG) cp_async8(seg + tid, op.epad + kEOFF + (tc.s0 - m0 - (BK - 1)) + tid);
    } else {
        // main stage: Us[s][j] = U[(s0+s)*Np + j0 + j], gseg[x] = gen row (i1-j1) at base + x
        const int jb = it - tc.nconv;
        const int j1 = jb / tc.nbj2;
        const int j2_0 = (jb % tc.nbj2) * BK;
        const long long j0 = (long long)j1 * op.ld2 + j2_0;
        for (int c = tid; c < BN * BK / 2; c += NTHREADS) {
            const int sl = c / (BK / 2), jp = c % (BK / 2);
            const int s = tc.s0 + sl;
            const bool valid = s < op.S;
            const double* src = valid ? U + (long long)s * op.Np + j0 + 2 * jp : U;
            cp_async16(stage + sl * LDJ + 2 * jp, src, valid);
        }
        if (tid < SEG) {
            const int row = tc.i1 - j1 + op.n1 - 1;
            const int base = (tc.i2_0 - j2_0) - (BK - 1) + op.ld2;
            cp_async8(seg + tid, op.gen + (long long)row * op.gen_stride + base + tid);
        }
    }
}

__global__ void __launch_bounds__(NTHREADS, 2)
toeplitz_apply_kernel(OperatorView op, const double* __restrict__ U, double* __restrict__ Z, const int* skip,
                      const double* __restrict__ minus_from, int precond_matrix, int conv_only) {
    if (skip && *skip) return;
    extern __shared__ __align__(16) double smem[];

    TileCtx tc;
    tc.i0 = blockIdx.x * BM;
    tc.s0 = blockIdx.y * BN;
    tc.i1 = tc.i0 / op.ld2;
    tc.i2_0 = tc.i0 - tc.i1 * op.ld2;
    tc.nbj2 = (op.n2 + BK - 1) / BK;
    tc.nmain = conv_only ? 0 : op.n1 * tc.nbj2;  // conv-only: the time convolution alone (K1f)
    const int conv_cols = min(tc.s0 + BN, op.S);
    tc.nconv = tc.s0 < op.S ? (conv_cols + BK - 1) / BK : 0;
    const int total = tc.nconv + tc.nmain;

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm0 = (warp & 1) * 32;
    const int wn0 = (warp >> 1) * 16;
    // warps whose 16 columns are all virtual (beyond the last time level) skip the math; the f
    // column is done by fcol_kernel (a 64-wide tile for that one column would cost a full tile)
    const bool active = tc.s0 + wn0 < op.S;

    double acc1[4][2][2], acc2[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            acc1[a][b][0] = acc1[a][b][1] = 0.0;
            acc2[a][b][0] = acc2[a][b][1] = 0.0;
        }

#pragma unroll
    for (int st = 0; st < NSTAGE - 1; ++st) {
        if (st < total) load_stage(op, U, tc, smem + st * STAGE_DBL, st);
        cp_commit();
    }

    for (int it = 0; it < total; ++it) {
        cp_wait<NSTAGE - 2>();
        __syncthreads();
        const int nxt = it + NSTAGE - 1;
        if (nxt < total) load_stage(op, U, tc, smem + (nxt % NSTAGE) * STAGE_DBL, nxt);
        cp_commit();

        const double* stage = smem + (it % NSTAGE) * STAGE_DBL;
        const double* seg = stage + (STAGE_DBL - SEG);
        if (!active) continue;
        if (it < tc.nconv) {
#pragma unroll
            for (int kk = 0; kk < BK / 4; ++kk) {
                double a[4], b[2];
#pragma unroll
                for (int mi = 0; mi < 4; ++mi) a[mi] = stage[(4 * kk + t) * LDI + wm0 + 8 * mi + g];
#pragma unroll
                for (int ni = 0; ni < 2; ++ni) b[ni] = seg[(wn0 + 8 * ni + g) - (4 * kk + t) + BK - 1];
#pragma unroll
                for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                    for (int ni = 0; ni < 2; ++ni) dmma(acc2[mi][ni], a[mi], b[ni]);
            }
        } else {
#pragma unroll
            for (int kk = 0; kk < BK / 4; ++kk) {
                double a[4], b[2];
#pragma unroll
                for (int mi = 0; mi < 4; ++mi) a[mi] = seg[wm0 + 8 * mi + g - 4 * kk - t + BK - 1];
#pragma unroll
                for (int ni = 0; ni < 2; ++ni) b[ni] = stage[(wn0 + 8 * ni + g) * LDJ + 4 * kk + t];
#pragma unroll
                for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                    for (int ni = 0; ni < 2; ++ni) dmma(acc1[mi][ni], a[mi], b[ni]);
            }
        }
    }
    cp_wait<0>();
    __syncthreads();

    // ---- epilogue: stage accumulators as C[s][i] so global traffic is coalesced along i
    double* C1 = smem;
    double* C2 = smem + BN * LDC;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int sl = wn0 + 8 * ni + 2 * t + c;
                const int il = wm0 + 8 * mi + g;
                C1[sl * LDC + il] = acc1[mi][ni][c];
                C2[sl * LDC + il] = acc2[mi][ni][c];
            }
    __syncthreads();

    const long long Np = op.Np;
    const double* fcol = U + (long long)op.S * Np;
    for (int idx = threadIdx.x; idx < BM * BN; idx += NTHREADS) {
        const int sl = idx / BM, il = idx % BM;
        const int s = tc.s0 + sl;
        if (s >= op.S) break;  // idx increases with s
        const long long i = tc.i0 + il;
        const long long o = (long long)s * Np + i;
        double out;
        if (tc.i2_0 + il >= op.n2) {
            out = 0.0;
        } else if (s < op.S) {
            const long long ds = (long long)s * Np + i;
            out = op.D1[ds] * C2[sl * LDC + il] + op.cs * op.D2[ds] * C1[sl * LDC + il];
            if (!precond_matrix) out -= op.eta * op.q[s] * fcol[i];
        } else {
            const long long dl = (long long)(op.S - 1) * Np + i;
            out = U[dl] + op.cr * op.D2[dl] * C1[sl * LDC + il];
        }
        Z[o] = minus_from ? minus_from[o] - out : out;
    }
}

// f column: Z[:, S] = y^(S) + cr D2_S o (K f)   (minus_from: Z = minus_from - that).  K f is one
// matrix-vector product (N^2 FMAs): CUDA cores, one CTA per 64 output rows, the generating-vector
// segment and a chunk of f staged in shared memory; 4 threads per row split each chunk.
constexpr int FC = 256;  // f chunk per stage
__global__ void __launch_bounds__(256) fcol_kernel(OperatorView op, const double* __restrict__ U,
                                                   double* __restrict__ Z, const int* skip,
                                                   const double* __restrict__ minus_from) {
    if (skip && *skip) return;
    __shared__ double fseg[FC];
    __shared__ double gseg[FC + BM];
    __shared__ double red[4][BM];
    const long long Np = op.Np;
    const long long i0 = (long long)blockIdx.x * BM;
    const int i1 = (int)(i0 / op.ld2), i2_0 = (int)(i0 % op.ld2);
    const int r = threadIdx.x & (BM - 1), part = threadIdx.x >> 6;
    const double* f = U + (long long)op.S * Np;
    double acc = 0.0;
    for (int j1 = 0; j1 < op.n1; ++j1) {
        const double* grow = op.gen + (long long)(i1 - j1 + op.n1 - 1) * op.gen_stride + op.ld2;
        for (int j0 = 0; j0 < op.n2; j0 += FC) {
            const int nc = min(FC, op.n2 - j0);
            __syncthreads();
            for (int q = threadIdx.x; q < FC; q += blockDim.x) fseg[q] = q < nc ? f[(long long)j1 * op.ld2 + j0 + q] : 0.0;
            // gseg[x] = a[i2_0 - j0 - (FC - 1) + x]: row r, column c -> gseg[r - c + FC - 1]
            for (int q = threadIdx.x; q < FC + BM; q += blockDim.x) {
                const int l2 = i2_0 - j0 - (FC - 1) + q;
                gseg[q] = (l2 > -op.n2 && l2 < op.n2) ? grow[l2] : 0.0;
            }
            __syncthreads();
            double a4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
            for (int cc = part; cc < FC; cc += 4) a4[cc & 3] += gseg[r - cc + FC - 1] * fseg[cc];
            acc += (a4[0] + a4[1]) + (a4[2] + a4[3]);
        }
    }
    red[part][r] = acc;
    __syncthreads();
    if (threadIdx.x < BM) {
        const double kf = (red[0][r] + red[1][r]) + (red[2][r] + red[3][r]);
        const long long i = i0 + r;
        const long long o = (long long)op.S * Np + i;
        double out = 0.0;
        if (i2_0 + r < op.n2) {
            const long long dl = (long long)(op.S - 1) * Np + i;
            out = U[dl] + op.cr * op.D2[dl] * kf;
        }
        Z[o] = minus_from ? minus_from[o] - out : out;
    }
}

}  // namespace

void toeplitz_apply(fi_ctx* ctx, const OperatorView& op, const double* U, double* Z, const int* skip,
                    const double* minus_from, bool precond_matrix) {
    ensure_smem_attr((const void*)toeplitz_apply_kernel, SMEM_BYTES);
    // the f column (fcol_kernel) on the side stream, overlapping the time-level GEMM
    FI_CUDA(cudaEventRecord(ctx->fork, ctx->stream));
    FI_CUDA(cudaStreamWaitEvent(ctx->side, ctx->fork, 0));
    fcol_kernel<<<(unsigned)(op.Np / BM), 256, 0, ctx->side>>>(op, U, Z, skip, minus_from);
    FI_LAUNCHED(ctx);
    FI_CUDA(cudaEventRecord(ctx->join, ctx->side));
    dim3 grid((unsigned)(op.Np / BM), (unsigned)((op.S + BN - 1) / BN));
    toeplitz_apply_kernel<<<grid, NTHREADS, SMEM_BYTES, ctx->stream>>>(op, U, Z, skip, minus_from,
                                                                         precond_matrix ? 1 : 0, 0);
    FI_LAUNCHED(ctx);
    FI_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->join, 0));
}

void toeplitz_conv_apply(fi_ctx* ctx, const OperatorView& op, const double* U, double* Z, const int* skip,
                         const double* minus_from, bool precond_matrix, cudaStream_t stream) {
    // time levels only: Z[:, s] = D1_s o (U E^T)[:, s] - eta q_s f (s < S); the f column is not written
    ensure_smem_attr((const void*)toeplitz_apply_kernel, SMEM_BYTES);
    dim3 grid((unsigned)(op.Np / BM), (unsigned)((op.S + BN - 1) / BN));
    toeplitz_apply_kernel<<<grid, NTHREADS, SMEM_BYTES, stream>>>(op, U, Z, skip, minus_from, precond_matrix ? 1 : 0, 1);
    FI_LAUNCHED(ctx);
}

}  // namespace fib
