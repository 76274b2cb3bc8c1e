/*
 * fracinv_b200.h — C-ABI of the B200-native preconditioned-GMRES path for the
 * all-at-once space-time system of arXiv 2507.02809 (reference library "fracinv").
 *
 * Plain C: opaque handles, plain pointers and sizes, integer status codes.  No C++
 * exceptions and no torch types cross this boundary.  Every entry point names the
 * reference interface it replaces (paths relative to /root/reference/proj).
 *
 * Vector layout at the boundary is the reference's (system.cpp:154-157): a stacked
 * block vector of length (S+1)*N, block s (1-based) at offset (s-1)*N, the source
 * block f last.  Device pointers ("*_dev") are CUDA global-memory pointers on the
 * context's device; host pointers ("*_host") are ordinary host memory.  Internally
 * the library keeps a padded level-major layout.
 *
 * Threading: one CUDA stream per fi_ctx; a context and the objects created from it
 * must not be used from two host threads at once without external locking (the
 * reference's "independent workspaces" rule, toeplitz.hpp:20-22).  Objects are
 * immutable after creation.
 */
#ifndef FRACINV_B200_H
#define FRACINV_B200_H

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. Mapping to the reference's exception taxonomy (errors.hpp:9-43):
 *   FI_E_DIM       DimensionError
 *   FI_E_RESOURCE  ResourceLimitError (block cap, device memory)
 *   FI_E_SINGULAR  SingularBlockError (time index via fi_last_error_time_index)
 *   FI_E_DOMAIN    std::domain_error (invalid parameters)
 *   FI_E_CUDA      CUDA runtime failure / no device
 *   FI_E_NOCONV    a tau-PCG block solve stopped at maxit above its tolerance (fi_precond_apply_host;
 *                  GMRES non-convergence itself is reported in fi_gmres_report, not as an error)
 *   FI_E_CONFIG    ConfigError
 */
enum {
    FI_OK = 0,
    FI_E_DIM = 1,
    FI_E_RESOURCE = 2,
    FI_E_SINGULAR = 3,
    FI_E_DOMAIN = 4,
    FI_E_CUDA = 5,
    FI_E_NOCONV = 6,
    FI_E_CONFIG = 7
};

typedef struct fi_ctx fi_ctx;
typedef struct fi_system fi_system;
typedef struct fi_precond fi_precond;

/* ------------------------------------------------------------------ context / errors */
int fi_ctx_create(int device, fi_ctx** out);
void fi_ctx_destroy(fi_ctx* ctx);
/* cudaStream_t of the context (all work is enqueued on it). */
void* fi_ctx_stream(fi_ctx* ctx);
int fi_ctx_synchronize(fi_ctx* ctx);
/* Message of the last failing call on this host thread. */
const char* fi_last_error(void);
/* SingularBlockError::time_index (errors.hpp:22-30): 1-based level, S+1 = f-block. */
int fi_last_error_time_index(void);
/* Number of this library's kernels launched on `ctx` since creation (launch accounting). */
long long fi_ctx_kernel_launches(fi_ctx* ctx);

/* ------------------------------------------------------------------ host setup numerics
 * Host restatements used to assemble fi_system_desc (setup, not the hot path). */
int fi_gamma(double x, double* out);                                    /* numerics.cpp:57-61 */
int fi_l1_weights(double beta, int S, double* b, double* e);            /* numerics.cpp:63-80 */
int fi_time_grid(double beta, int S, double T, double* dt, double* eta);/* numerics.cpp:82-96 */
/* coeffs: 2n-1 entries, index l+n-1 (symbol.cpp:88-110). */
int fi_symbol_coeffs_1d(double omega, int n, double* coeffs);
/* coeffs: prod(2n_i-1) entries, lexicographic (symbol.cpp:112-191). d in {1,2}. */
int fi_symbol_coeffs_md(double omega, int d, const int* n, long long sample_cap, double* coeffs);
/* The same on the device of ctx (d = 2: the two cosine-sum stages as CUDA kernels, sums in the host's
 * order without FMA contraction: bit-for-bit fi_symbol_coeffs_md; d = 1 falls back to the host).
 * SURVEY 8(f) row 2; coeffs is a host array. */
int fi_symbol_coeffs_md_dev(fi_ctx* ctx, double omega, int d, const int* n, long long sample_cap, double* coeffs);
/* Gaussian relative-L2 noise (EXTENSION for BASELINE.json; SplitMix64-at-index + Box-Muller)
 * and the reference's additive uniform noise (system.cpp:240-251). out may alias mu. */
int fi_add_gaussian_noise(const double* mu, long long n, double rel_eps, unsigned long long seed, double* out);
int fi_add_noise(const double* mu, long long n, double eps, unsigned long long seed, double* out);

/* ------------------------------------------------------------------ system operator
 * Replaces SystemOperator (system.hpp:72-104, system.cpp:121-174).  All arrays are host
 * pointers, copied at creation:
 *   gen : generating tensor of B, prod(2 n_i - 1) entries (SymbolCoefficients::coeffs)
 *   e, b: L1 weights (S entries each), q: q(t_s) (S entries, must be > 0)
 *   D1, D2: S x N, row-major by level (row s-1 = gamma_k(x, t_s), CoefficientDiagonals)
 *   eta = dt^beta Gamma(2-beta); scale_space = eta/h^omega; scale_reg = lambda/h^omega. */
typedef struct {
    int d;          /* 1 or 2 */
    int n[2];       /* interior points per direction (n[1] ignored when d == 1) */
    int S;          /* time steps */
    double h, eta, scale_space, scale_reg;
    const double* gen;
    const double* e;
    const double* b;
    const double* q;
    const double* D1;
    const double* D2;
    double omega;   /* space order (used by the tau preconditioner of 2D blocks; 0 = unknown) */
} fi_system_desc;

int fi_system_create(fi_ctx* ctx, const fi_system_desc* desc, fi_system** out);
void fi_system_destroy(fi_system* sys);
long long fi_system_dim(const fi_system* sys);        /* (S+1)*N   (SystemOperator::dim) */
long long fi_system_space_dim(const fi_system* sys);  /* N         (space_dim) */
/* z = A y on device vectors (SystemOperator::apply, system.cpp:144-174). Async on the stream. */
int fi_system_apply(fi_system* sys, const double* y_dev, double* z_dev);
/* Host-buffer convenience: H2D, apply, D2H, synchronize. */
int fi_system_apply_host(fi_system* sys, const double* y_host, double* z_host);

/* ------------------------------------------------------------------ preconditioner
 * Replaces BlockTriangularPreconditioner (krylov.hpp:33-50, krylov.cpp:24-70).
 * block_cap <= 0 selects the reference default 4096 (kDefaultBlockCap).  N > block_cap returns
 * FI_E_RESOURCE like the reference for 1D; for 2D it selects the substituted tau-PCG block solve
 * (see fi_precond_create_ex), where the reference cannot run at all.  Singular blocks return
 * FI_E_SINGULAR with the 1-based time index (S+1 = regularisation block). */
int fi_precond_create(fi_system* sys, long long block_cap, fi_precond** out);
/* Explicit choice of the per-block solve.  inner = 0: dense (the reference's direct solve, above
 * block_cap -> FI_E_RESOURCE); inner = 1: tau-preconditioned CG per block to relative residual
 * `tol`, or to the rounding floor of a residual evaluated in double, u ||M|| ||x||, where that is
 * larger (at most `maxit` steps) — the substituted solve for 2D blocks beyond the cap (needs
 * n_i + 1 a power of two); inner = -1: what fi_precond_create does (dense up to block_cap, tau-PCG
 * above it for 2D). */
int fi_precond_create_ex(fi_system* sys, long long block_cap, int inner, double tol, int maxit, fi_precond** out);
/* 0 = dense inverses, 1 = tau-PCG per block. */
int fi_precond_inner(const fi_precond* P);
/* Storage of the dense inverses: 0 = packed 64x64 tiles (FP64 + FP32 copy), 1 = tau-PCG (no
 * inverses), 2 = HODLR (64-row leaves, rank-32 off-diagonal blocks). */
int fi_precond_form(const fi_precond* P);
void fi_precond_destroy(fi_precond* P);
/* y = P^{-1} z (forward block substitution), device vectors, async. */
int fi_precond_apply(fi_precond* P, const double* z_dev, double* y_dev);
int fi_precond_apply_host(fi_precond* P, const double* z_host, double* y_host);
/* Inner-solve counters of the tau-PCG block solve (inner = 1), accumulated on the device since the last
 * reset (fi_gmres resets them when it starts): out[0] CG steps, out[1] block solves that stopped at maxit
 * above their tolerance, out[2] most CG steps of one block solve, out[3] preconditioner applies.  All zero
 * for dense blocks.  Synchronises the context's stream; reset != 0 zeroes the counters after reading. */
int fi_precond_stats(fi_precond* P, long long out[4], int reset);
/* The build's a-posteriori check of HODLR-compressed inverses (fi_precond_form == 2), worst over levels and
 * 4 probe vectors x: out[0] forward error |W x - H x| / |W x| against the uncompressed inverse W, out[1]
 * normwise backward error |M y - x| / (|M| |y| + |x|) of y = H x in the block matrix M itself.  A level that
 * fails either bound (1e-12, 1e-13) rebuilds the preconditioner with packed tiles; zeros otherwise. */
int fi_precond_build_check(const fi_precond* P, double out[2]);
/* Device memory held by the preconditioner's per-level inverses (bytes). */
long long fi_precond_bytes(const fi_precond* P);
/* refine == 0 (default for dense blocks): one FP64 sweep over the polished inverses (built to the
 * accuracy of the reference's LU solves: forward parity ~1e-13);
 * refine != 0: each apply adds one iterative-refinement sweep (residual through the operator
 * kernel), which also brings the residual |P y - z| to LU grade.  No effect in tau-PCG mode. */
int fi_precond_set_refine(fi_precond* P, int refine);

/* ------------------------------------------------------------------ problem assembly helpers
 * build_rhs (system.cpp:176-190): z^(s) = b_{s-1} D1^(s) o rho, z^(S+1) = mu_eps. Host pointers. */
int fi_build_rhs(const fi_system* sys, const double* rho_host, const double* mu_eps_host, double* z_host);
/* forward_solve (system.cpp:192-224) on the device through P's cached time-level inverses
 * (P == NULL builds a temporary one).  states_host: S*N (may be NULL); mu_host: N. */
int fi_forward_solve(fi_system* sys, fi_precond* P, const double* rho_host, const double* f_host,
                     double* states_host, double* mu_host);

/* ------------------------------------------------------------------ GMRES
 * Replaces gmres() (krylov.hpp:52-69, krylov.cpp:72-209).  Left-preconditioned, MGS with one
 * conditional re-orthogonalisation, Givens least squares, all on the device: the host
 * synchronises once per restart cycle, never per iteration.
 *   restart = 0 : full GMRES (the reference); restart = m > 0 : GMRES(m) (EXTENSION, see
 *                 DESIGN.md §5 for the exact restart semantics, shared with the oracle).
 *   maxit = 0   : the system dimension (reference default).
 * history_host receives residual_history (history_len = iterations + 1 entries, truncated to
 * history_cap). */
typedef struct {
    double tol;
    int maxit;
    int restart;
} fi_gmres_opts;

typedef struct {
    int iterations;
    int converged;
    int breakdown;
    double wall_time_seconds;
    double final_true_residual;
    int history_len;
    int inner_nonconverged; /* EXTENSION: tau-PCG block solves of this solve that stopped at maxit above
                               their tolerance (0 for dense blocks; see fi_precond_stats) */
} fi_gmres_report;

/* P may be NULL (no preconditioning); x0_dev may be NULL (zero start). */
int fi_gmres(fi_system* sys, fi_precond* P, const double* b_dev, const double* x0_dev, double* x_dev,
             const fi_gmres_opts* opts, fi_gmres_report* report, double* history_host, int history_cap);
/* Host-buffer variant: H2D of b (and x0), solve, D2H of x — the reference-facing call. */
/* Measurement hook (bench roofline of K3): average time of one MGS round (w -= c x; h = y.w, the
 * fused axpy + dot of krylov.cpp:127-132) over device vectors of length n, L2 flushed before each. */
int fi_mgs_round_timed(fi_ctx* ctx, long long n, double* w_dev, const double* x_dev, const double* y_dev, int reps,
                       double* ms_avg);
/* Measurement hook (bench roofline of K3/K4): average time of one Arnoldi step's MGS + Givens kernel
 * (mgs_step_kernel) at step k over pseudo-random vectors of length n, L2 flushed before each; *reorth
 * (may be NULL) tells whether the conditional second pass ran. */
int fi_mgs_step_timed(fi_ctx* ctx, long long n, int k, int reps, double* ms_avg, int* reorth);
/* Dense realisation (spectra.cpp:14-45, verification only): kind 0 = SystemA, 1 = PreconditionerP,
 * 2 = ForwardAhat; row-major dim x dim into device memory M_dev (dim = (S+1)N, or S N for Ahat);
 * FI_E_RESOURCE above cap (<= 0: 4096).  Bit-for-bit the reference's entries. */
int fi_assemble_dense(fi_system* sys, int kind, long long cap, double* M_dev);
/* Arnoldi step of fi_gmres / fi_gmres_host with a system preconditioner: on = 1 (default) computes
 * P^{-1} A v as v + P^{-1}((A - P) v) — A and P differ only in the f column of the time rows,
 * -eta q_s I (spectra.cpp:34-36), so one preconditioner sweep and no operator apply per step (an exact
 * identity, cf. Eisenstat's trick); on = 0: A v by K1, then P^{-1} (the reference's order of
 * operations, krylov.cpp:123-126).  Environment FI_SPLIT_APPLY=0 forces 0. */
int fi_system_set_split_apply(fi_system* sys, int on);
/* Realisation of the operator apply (fi_system_apply*, and A inside fi_gmres): FI_APPLY_DMMA = K1, the
 * dense FP64 DMMA contraction K U with K generated per tile (the 1D default); FI_APPLY_FFT = K1f, the
 * reference's own algorithm (circulant-embedded FFT Toeplitz products, toeplitz.cpp:68-114) as batched
 * 2D transforms with K1's time convolution fused beside them (2D grids with n_i + 1 a power of two);
 * FI_APPLY_AUTO (default) = FFT where supported, else DMMA.  FI_E_DOMAIN for FFT on another layout.
 * Environment FI_APPLY=dmma|fft sets the mode at creation.  get: the realisation in use. */
enum { FI_APPLY_AUTO = 0, FI_APPLY_DMMA = 1, FI_APPLY_FFT = 2 };
int fi_system_set_apply_mode(fi_system* sys, int mode);
int fi_system_get_apply_mode(const fi_system* sys);
int fi_gmres_host(fi_system* sys, fi_precond* P, const double* b_host, const double* x0_host, double* x_host,
                  const fi_gmres_opts* opts, fi_gmres_report* report, double* history_host, int history_cap);

/* Generic LinearOp form (krylov.hpp:52 `LinearOp`): callbacks that enqueue y = op(x) on
 * the context stream for device vectors of length n and return 0 on success.  apply_M may be
 * NULL.  Used for the reference's operator-agnostic GMRES known-answer tests. */
typedef int (*fi_linop_fn)(void* user, const double* x_dev, double* y_dev);
int fi_gmres_op(fi_ctx* ctx, long long n, fi_linop_fn apply_A, void* user_A, fi_linop_fn apply_M, void* user_M,
                const double* b_dev, const double* x0_dev, double* x_dev, const fi_gmres_opts* opts,
                fi_gmres_report* report, double* history_host, int history_cap);

/* ------------------------------------------------------------------ instrumentation
 * Average device time (ms, CUDA events on the context stream) of the last `fi_*_timed`
 * kernel launch sequence; used by bench.py for the roofline.  kind: 0 = operator apply
 * (K1 toeplitz GEMM), 1 = preconditioner apply (K2), 2 = one Arnoldi/MGS step. */
int fi_system_apply_timed(fi_system* sys, const double* y_dev, double* z_dev, int reps, double* ms_avg);
int fi_precond_apply_timed(fi_precond* P, const double* z_dev, double* y_dev, int reps, double* ms_avg);

#ifdef __cplusplus
}
#endif
#endif /* FRACINV_B200_H */
