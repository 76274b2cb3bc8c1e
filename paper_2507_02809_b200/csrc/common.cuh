// Internal shared definitions of the fracinv B200 library (not part of the C-ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/fracinv_b200.h"

namespace fib {

// Exception used inside the library; converted to a status code at the C-ABI boundary.
struct Error : std::runtime_error {
    int code;
    int time_index;
    Error(int c, const std::string& m, int ti = 0) : std::runtime_error(m), code(c), time_index(ti) {}
};

#define FI_CUDA(x)                                                                                   \
    do {                                                                                             \
        cudaError_t e_ = (x);                                                                        \
        if (e_ != cudaSuccess)                                                                       \
            throw ::fib::Error(FI_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));          \
    } while (0)

#define FI_LAUNCHED(ctx)                                                                             \
    do {                                                                                             \
        cudaError_t e_ = cudaGetLastError();                                                         \
        if (e_ != cudaSuccess)                                                                       \
            throw ::fib::Error(FI_E_CUDA, std::string("kernel launch (") + __FILE__ + ":" +           \
                                              std::to_string(__LINE__) + "): " + cudaGetErrorString(e_)); \
        (ctx)->launches++;                                                                           \
    } while (0)

inline int poison_mode() {  // FI_POISON: 1 every buffer, 2 only >= 1 MiB, 3 only < 1 MiB (bisecting)
    static const int m = std::getenv("FI_POISON") ? std::atoi(std::getenv("FI_POISON")) : 0;
    return m;
}
inline bool poison_allocs(size_t bytes) {
    const int m = poison_mode();
    return m == 1 || (m == 2 && bytes >= (1u << 20)) || (m == 3 && bytes < (1u << 20));
}

// Owning device buffer (cudaMalloc/cudaFree).
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count) {
        release();
        if (count == 0) return;
        cudaError_t e = cudaMalloc(&p, count * sizeof(T));
        if (e != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            throw Error(FI_E_RESOURCE, "device allocation of " + std::to_string(count * sizeof(T)) +
                                           " bytes failed: " + cudaGetErrorString(e));
        }
        n = count;
        // FI_POISON (diagnostics; the sanitizer is unavailable on this GPU pool): every new device buffer is
        // filled with 0xff bytes (NaN as doubles, ~0 as counters), so a kernel that reads scratch it never
        // wrote, or code that relies on zeroed allocations, shows up as NaN / wrong results in the parity tests
        // (legacy-stream memset + sync: allowed while another stream captures a graph in relaxed mode, as a
        // first apply inside the GMRES capture does; any error is cleared rather than left sticky)
        if (poison_allocs(count * sizeof(T))) {
            if (cudaMemset(p, 0xff, count * sizeof(T)) == cudaSuccess) cudaStreamSynchronize(0);
            cudaGetLastError();
        }
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
};

// Padded level-major layout of a stacked block vector.
//  level s (0-based, S = f-block) occupies [s*Np, (s+1)*Np); within a level the
//  space index is i = i1*ld2 + i2 (i1 < n1, i2 < ld2) and rows with i2 >= n2 are zero.
struct Layout {
    int d = 1;
    int n1 = 1, n2 = 1;  // 1D: n1 = 1, n2 = N
    int ld2 = 64;        // n2 rounded up to a multiple of 64
    long long N = 1;     // n1*n2 (reference block size)
    long long Np = 64;   // n1*ld2 (padded block size)
    int S = 1;
    long long nI() const { return (long long)(S + 1) * Np; }
    long long nRef() const { return (long long)(S + 1) * N; }
};

inline Layout make_layout(int d, const int* n, int S) {
    Layout L;
    L.d = d;
    L.n1 = d == 1 ? 1 : n[0];
    L.n2 = d == 1 ? n[0] : n[1];
    L.ld2 = ((L.n2 + 63) / 64) * 64;
    L.N = (long long)L.n1 * L.n2;
    L.Np = (long long)L.n1 * L.ld2;
    L.S = S;
    return L;
}

}  // namespace fib

// Handles are reference counted so that destruction order is irrelevant (a language
// binding may finalise a preconditioner after its system, or a system after its context).
struct fi_ctx {
    int refs = 1;
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    long long launches = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // side stream for independent work that overlaps a main-stream kernel (fork/join events)
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};

// --------------------------------------------------------------------------- kernels (launchers)
namespace fib {

struct SystemDev;  // defined in system.cuh

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device attribute: raise it to at least `bytes`
// once per (device, kernel).  Thread-safe; the calling thread's current device must be the context's
// (every C-ABI entry binds it, abi.cu).
void ensure_smem_attr(const void* func, size_t bytes);

// Layout conversion: reference (S+1)*N <-> padded (S+1)*Np.
void pack_vector(fi_ctx* ctx, const Layout& L, const double* ref, double* pad);
void unpack_vector(fi_ctx* ctx, const Layout& L, const double* pad, double* ref);

}  // namespace fib
