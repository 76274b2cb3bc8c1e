// Device GMRES engine (K3/K4) shared by fi_gmres and fi_gmres_op.
#pragma once

#include <cstddef>
#include <functional>
#include <vector>

#include "common.cuh"

namespace fib {

// Device-resident Arnoldi/Givens state (one per solve).
struct GmresState {
    double* h;      // current Hessenberg column (cycle + 2)
    double* c;      // second-pass corrections (cycle + 2)
    double* cs;     // Givens cosines
    double* sn;     // Givens sines
    double* g;      // rotated right-hand side
    double* ycoef;  // back-substitution result
    double* R;      // rotated columns, column k at R + k * ldR
    int ldR;
    double bnorm, tol, breakdown_tol;
    double pre_norm2, hnorm2;
    int done, reorth, vnext_ok, iters, kc, converged, breakdown;
    double scal[4];  // scratch norms read back by the host
};

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
    // Reference semantics of gmres() (krylov.cpp:72-209) + restart extension.
    // optional: w = M^{-1} A v in one operation (used for the Arnoldi step instead of A then M)
    void set_fused(const Op* f) { fused_ = f; }
    // measurement hook (bench roofline): average time of one MGS round w -= c x; h = y.w over
    // device vectors of length n(), L2 flushed (a write larger than L2) before every timed round
    double time_mgs_round(double* w, const double* x, const double* y, int reps);
    void solve(const Op& A, const Op* M, const double* b, const double* x0, double* x, double tol, int maxit,
               int restart, fi_gmres_report* rep, std::vector<double>& history);

private:
    void reduce(double* w, const double* x, const double* coef, const double* y, int mode, int k, int slot,
                double* out, const int* gate_on, const int* done);
    double norm2(const double* v, int slot);

    template <class T>
    static void ensure(DevBuf<T>& b, size_t count) {
        if (b.n < count) b.alloc(count);
    }

    fi_ctx* ctx_;
    long long n_;
    int grid_;
    GmresState* st_ = nullptr;
    DevBuf<double> partials_;
    DevBuf<unsigned> ticket_;
    DevBuf<double> V_, w_, t1_, t2_, hist_, arr_, ycoef_;
    DevBuf<GmresState> st_buf_;
    static constexpr int kLook = 2;  // Arnoldi steps kept queued ahead of the host's convergence check
    const Op* fused_ = nullptr;
    int* done_host_ = nullptr;       // pinned, host-mapped copy of the device `done` flag
    int* done_hmap_ = nullptr;       // its device alias
    cudaEvent_t iter_ev_[kLook] = {};
};

}  // namespace fib
