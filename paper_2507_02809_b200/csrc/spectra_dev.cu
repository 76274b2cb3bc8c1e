// Dense realisation of the block matrices on the device (spectra, verification).
//
// Replaces assemble_dense_system (spectra.cpp:14-45): every entry of A (SystemA), of the block
// lower-triangular P (PreconditionerP: A without the f coupling column) or of the forward matrix
// Ahat (ForwardAhat: the S time rows/columns of P) from the operator's own data — the generating
// tensor for B, D1, D2, e, q — with the reference's operation order, so the matrix is bit-for-bit the
// reference realisation.  Row-major dim x dim in device memory; the eigen- and singular-value
// routines that consume it are library calls (paper_2507_02809_b200/spectra.py).
#include "system.cuh"

namespace fib {
namespace {

__global__ void assemble_dense_kernel(OperatorView op, long long N, int n2r, int kind, long long dim, double* M) {
    const long long total = dim * dim;
    const int S = op.S;
    const double e0 = op.epad[kEOFF];
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long r = idx / dim, c = idx - r * dim;
        const int sr = (int)(r / N), sc = (int)(c / N);
        const long long i = r - (long long)sr * N, j = c - (long long)sc * N;
        const int i1 = (int)(i / n2r), i2 = (int)(i % n2r), j1 = (int)(j / n2r), j2 = (int)(j % n2r);
        auto Bij = [&]() {
            return op.gen[(long long)(i1 - j1 + op.n1 - 1) * op.gen_stride + (i2 - j2) + op.ld2];
        };
        double v = 0.0;
        if (sr < S) {
            const long long pi = (long long)sr * op.Np + (long long)i1 * op.ld2 + i2;  // padded (level, row)
            if (sc == sr) {
                v = (op.cs * op.D2[pi]) * Bij();
                if (i == j) v += e0 * op.D1[pi];
            } else if (sc < sr) {
                if (i == j) v = op.epad[kEOFF + (sr - sc)] * op.D1[pi];
            } else if (sc == S && kind == 0) {
                if (i == j) v = -op.eta * op.q[sr];
            }
        } else {  // f row (SystemA, PreconditionerP)
            if (sc == S - 1) {
                v = i == j ? 1.0 : 0.0;
            } else if (sc == S) {
                const long long pi = (long long)(S - 1) * op.Np + (long long)i1 * op.ld2 + i2;
                v = (op.cr * op.D2[pi]) * Bij();
            }
        }
        M[idx] = v;
    }
}

}  // namespace

void assemble_dense(fi_ctx* ctx, const fi_system* sys, int kind, long long cap, double* M) {
    const Layout& L = sys->L;
    if (kind < 0 || kind > 2) throw Error(FI_E_DOMAIN, "assemble_dense_system: kind must be 0 (A), 1 (P) or 2 (Ahat)");
    const long long dim = kind == 2 ? (long long)L.S * L.N : (long long)(L.S + 1) * L.N;
    if (dim > cap)
        throw Error(FI_E_RESOURCE,
                    "assemble_dense_system: dimension " + std::to_string(dim) + " exceeds cap " + std::to_string(cap));
    assemble_dense_kernel<<<ctx->sm_count * 8, 256, 0, ctx->stream>>>(sys->view(), L.N, L.n2, kind, dim, M);
    FI_LAUNCHED(ctx);
}

}  // namespace fib
