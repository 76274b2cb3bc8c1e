// Device GMRES engine (K3/K4) shared by fi_gmres and fi_gmres_op.
#pragma once

#include <cstddef>
#include <functional>
#include <vector>

#include "common.cuh"

namespace fib {

// Device-resident Arnoldi/Givens state (one per solve).  The pointer fields come first (the host
// rewrites them alone when the workspace grows during a solve).
struct GmresState {
    double* h;      // current Hessenberg column (capacity + 1)
    double* c;      // second-pass corrections
    double* cs;     // Givens cosines
    double* sn;     // Givens sines
    double* g;      // rotated right-hand side
    double* ycoef;  // back-substitution result
    double* R;      // rotated columns, packed: column k (k + 1 entries) at k (k + 1) / 2
    double bnorm, tol, breakdown_tol;
    double pre_norm2, hnorm2;
    int done, reorth, vnext_ok, iters, kc, converged, breakdown;
    int k;      // device-driven solve: Arnoldi step within the cycle
    int steps;  // device-driven solve: steps of this cycle, min(restart, maxit - iterations)
    int flags;  // device-driven solve: bit 0 zero right-hand side, bit 1 converged at the start
    int ncycles, nresid;  // device-driven solve: executions of the cycle body and of the restart residual
    double beta, bnorm_true, final_rn2;
    double scal[4];  // scratch norms read back by the host
};
constexpr int kStatePointers = 7;

inline double* scal_dev(GmresState* st_dev) {
    return reinterpret_cast<double*>(reinterpret_cast<char*>(st_dev) + offsetof(GmresState, scal));
}

template <class T>
inline T* field_dev(GmresState* st_dev, size_t off) {
    return reinterpret_cast<T*>(reinterpret_cast<char*>(st_dev) + off);
}

// y = op(x) enqueued on the context stream; skip (device flag) lets enqueued work no-op.
using Op = std::function<void(const double* x, double* y, const int* skip)>;

class GmresEngine {
public:
    GmresEngine(fi_ctx* ctx, long long n);
    ~GmresEngine();
    GmresEngine(const GmresEngine&) = delete;
    GmresEngine& operator=(const GmresEngine&) = delete;
    long long n() const { return n_; }
    // optional: w = M^{-1} A v in one operation (used for the Arnoldi step instead of A then M)
    void set_fused(const Op* f) { fused_ = f; }
    // measurement hook (bench roofline): average time of one MGS round w -= c x; h = y.w over
    // device vectors of length n(), L2 flushed (a read larger than L2) before every timed round
    double time_mgs_round(double* w, const double* x, const double* y, int reps);
    // measurement hook (bench roofline of K3/K4): average time of one mgs_step_kernel at Arnoldi step k on
    // pseudo-random vectors, L2 flushed before each; *reorth: whether the second pass ran
    double time_mgs_step(int k, int reps, int* reorth);
    // Reference semantics of gmres() (krylov.cpp:72-209) + restart extension.
    // Host-driven: the host enqueues every Arnoldi step, two steps ahead of the device's convergence
    // flag; the Krylov basis grows on demand (full GMRES allocates as it goes, like the reference).
    void solve(const Op& A, const Op* M, const double* b, const double* x0, double* x, double tol, int maxit,
               int restart, fi_gmres_report* rep, std::vector<double>& history);
    // Device-driven: the whole solve is one CUDA graph (conditional WHILE nodes for the restart cycles
    // and the Arnoldi steps, an IF node for the restart residual); the host launches it and synchronises
    // once.  The operators must be capturable (stream-ordered, no host synchronisation).  Returns false
    // (nothing done) when the cycle's basis does not fit in device memory; use solve() then.
    // key: what the captured graph depends on besides this engine's own buffers (the caller's object ids
    // and settings); a different key re-captures.
    bool solve_device(const Op& A, const Op* M, const double* b, const double* x0, double* x, double tol, int maxit,
                      int restart, const std::vector<long long>& key, fi_gmres_report* rep,
                      std::vector<double>& history);

private:
    void reduce(double* w, const double* x, const double* coef, const double* y, int mode, int slot,
                const int* done);
    double norm2(const double* v, int slot);
    void mgs_step(int k, int maxit, bool graph, unsigned long long cond);
    void reserve(int vectors, bool keep);  // basis and coefficient arrays for `vectors` basis vectors
    void bind_state_pointers();

    template <class T>
    static void ensure(DevBuf<T>& b, size_t count) {
        if (b.n < count) b.alloc(count);
    }

    fi_ctx* ctx_;
    long long n_, ldv_;
    int grid_, mgs_grid_ = 0;
    int cap_ = 0;  // basis capacity (vectors)
    GmresState* st_ = nullptr;
    DevBuf<double> partials_, mparts_;
    DevBuf<unsigned> ticket_, mbar_;
    DevBuf<double> V_, w_, t1_, t2_, vcur_, hist_, h_, c_, cs_, sn_, g_, R_, ycoef_;
    DevBuf<GmresState> st_buf_;
    static constexpr int kLook = 2;  // Arnoldi steps kept queued ahead of the host's convergence check
    const Op* fused_ = nullptr;
    int* done_host_ = nullptr;       // pinned, host-mapped copy of the device `done` flag
    int* done_hmap_ = nullptr;       // its device alias
    cudaEvent_t iter_ev_[kLook] = {};
    // device-driven solve: the captured graph and what it was captured for
    cudaGraphExec_t gexec_ = nullptr;
    cudaGraph_t graph_ = nullptr;
    std::vector<long long> gkey_;
    long long glaunch_[4] = {};  // kernel/memcpy launches captured in the top graph, a cycle, a step, a residual
};

}  // namespace fib
