// Internal shared definitions of libamgr_b200.so (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cstdint>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/amgr.h"

#ifndef GRP_BUF
#define GRP_BUF 256  // contributions per k_rap_grp group buffer (<= 256: 8-bit offsets)
#endif

namespace amgr {

// ---- errors ----------------------------------------------------------------
// Carries the amgr_status and the reference-compatible message.
struct Error : std::runtime_error {
    amgr_status status;
    Error(amgr_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(amgr_status s, const std::string& m) { throw Error(s, m); }
[[noreturn]] inline void invalid(const std::string& m) { throw Error(AMGR_E_INVALID_ARGUMENT, m); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        std::ostringstream os;
        os << "CUDA error in " << what << " (" << file << ":" << line << "): "
           << cudaGetErrorName(e) << ": " << cudaGetErrorString(e);
        throw Error(AMGR_E_CUDA, os.str());
    }
}
#define CK(x) ::amgr::cuda_check((x), #x, __FILE__, __LINE__)

// ---- launch bookkeeping ----------------------------------------------------
// Every kernel launch of the library goes through LAUNCH so that the context
// can (a) count launches and (b) bracket one kernel family with CUDA events
// for the roofline probe (amgr_probe_enable).
struct Probe {
    std::string family;                 // "" = disabled
    int level = -1;                     // >= 0: only launches on this hierarchy level
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;
    std::vector<double> bytes;
};

struct Ctx;
void probe_begin(Ctx& c, const char* family, double bytes);
void probe_end(Ctx& c, const char* family);

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string last_error;
    int64_t launches = 0;
    Probe probe;
    int num_sms = 148;
    int cur_level = -1;  // hierarchy level the orchestration is currently launching for
    // auxiliary stream for independent work inside one call (created lazily,
    // joined back into `stream` before the call returns)
    bool pdl = true;  // AMGR_PDL=0 disables programmatic dependent launch
    // dot-product order of the Krylov solvers: false = deterministic block
    // reduction (fused into the producing kernels), true = strictly sequential
    // left-to-right sums exactly as bicgstab.cpp:11-17 (AMGR_SEQ_DOTS=1 or
    // amgr_ctx_set_dot_order); a parity mode, ~8 cycles per element
    bool seq_dots = false;
    cudaStream_t side = nullptr;
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    cudaStream_t copy = nullptr;  // staged H2D of the next step's values (lazily created)
    // amgr_download_async: device snapshot + D2H on its own stream (lazily created)
    cudaStream_t d2h = nullptr;
    cudaEvent_t snap_ev = nullptr, d2h_done_ev = nullptr;
    double* snap = nullptr;
    int64_t snap_n = 0;
    // timing events of the per-call phase clocks, created once and reused
    // (creating ~30 events per rebuild starved the short small-level kernels)
    std::vector<cudaEvent_t> clock_pool;
    size_t clock_used = 0;
};

// Run fn with c.stream temporarily redirected to the side stream, ordered
// after everything already queued on the main stream; returns with the side
// work NOT yet joined (call join_side).
template <class F>
void on_side(Ctx& c, F&& fn) {
    if (!c.side) {
        // highest priority: the side stream carries the one-CTA coarse
        // factorization, which must not queue behind wide smoother grids
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&c.side, cudaStreamNonBlocking, hi));
        CK(cudaEventCreateWithFlags(&c.fork_ev, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c.join_ev, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(c.fork_ev, c.stream));
    CK(cudaStreamWaitEvent(c.side, c.fork_ev, 0));
    cudaStream_t main = c.stream;
    c.stream = c.side;
    try {
        fn();
    } catch (...) {
        c.stream = main;
        throw;
    }
    c.stream = main;
}

inline void join_side(Ctx& c) {
    if (!c.side) return;
    CK(cudaEventRecord(c.join_ev, c.side));
    CK(cudaStreamWaitEvent(c.stream, c.join_ev, 0));
}

// Programmatic dependent launch for the solve-path kernels: the next kernel
// of the stream may be scheduled while this one drains; every kernel
// launched this way starts with pdl_enter() (griddepcontrol.wait: full
// completion + visibility of the predecessor, then launch_dependents).
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

#define LAUNCH_PDL(ctx, family, bytes, kernel, grid, block, smem, ...)                                  \
    do {                                                                                               \
        ::amgr::probe_begin((ctx), (family), (bytes));                                                 \
        cudaLaunchConfig_t cfg_{};                                                                     \
        cfg_.gridDim = dim3(grid);                                                                     \
        cfg_.blockDim = dim3(block);                                                                   \
        cfg_.dynamicSmemBytes = (smem);                                                                \
        cfg_.stream = (ctx).stream;                                                                    \
        cudaLaunchAttribute at_[1];                                                                    \
        at_[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                                \
        at_[0].val.programmaticStreamSerializationAllowed = 1;                                         \
        cfg_.attrs = at_;                                                                              \
        cfg_.numAttrs = (ctx).pdl ? 1 : 0;                                                             \
        CK(cudaLaunchKernelEx(&cfg_, kernel, __VA_ARGS__));                                           \
        ::amgr::probe_end((ctx), (family));                                                            \
        ++(ctx).launches;                                                                              \
    } while (0)

#define LAUNCH(ctx, family, bytes, kernel, grid, block, smem, ...)                  \
    do {                                                                              \
        ::amgr::probe_begin((ctx), (family), (bytes));                                \
        kernel<<<(grid), (block), (smem), (ctx).stream>>>(__VA_ARGS__);               \
        CK(cudaGetLastError());                                                       \
        ::amgr::probe_end((ctx), (family));                                           \
        ++(ctx).launches;                                                             \
    } while (0)

inline unsigned grid_for(int64_t n, int block, int64_t cap = 1 << 30) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return static_cast<unsigned>(g);
}

// ---- device memory ---------------------------------------------------------
// Stream-ordered allocation (cudaMallocAsync) so per-step allocations of the
// value-semantics API are cheap; freed on the owning stream.
template <class T>
class DevArray {
  public:
    DevArray() = default;
    DevArray(int64_t n, cudaStream_t s) { alloc(n, s); }
    ~DevArray() { release(); }
    DevArray(const DevArray&) = delete;
    DevArray& operator=(const DevArray&) = delete;
    DevArray(DevArray&& o) noexcept { swap(o); }
    DevArray& operator=(DevArray&& o) noexcept {
        if (this != &o) {
            release();
            swap(o);
        }
        return *this;
    }
    void alloc(int64_t n, cudaStream_t s) {
        release();
        stream_ = s;
        n_ = n;
        // +8 elements of slack: TMA bulk copies read 16-byte-rounded ranges
        if (n > 0) {
            static const bool tr = std::getenv("AMGR_TRACE_ALLOC") != nullptr;
            const auto t0 = std::chrono::steady_clock::now();
            CK(cudaMallocAsync(reinterpret_cast<void**>(&p_), sizeof(T) * static_cast<size_t>(n + 8), s));
            if (tr) {
                const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                if (ms > 2.0) std::fprintf(stderr, "[amgr alloc] %.1f MB took %.1f ms\n", sizeof(T) * n / 1e6, ms);
            }
        }
    }
    void release() {
        if (p_) cudaFreeAsync(p_, stream_);
        p_ = nullptr;
        n_ = 0;
    }
    T* get() const { return p_; }
    int64_t size() const { return n_; }
    size_t bytes() const { return sizeof(T) * static_cast<size_t>(n_); }
    void swap(DevArray& o) noexcept {
        std::swap(p_, o.p_);
        std::swap(n_, o.n_);
        std::swap(stream_, o.stream_);
    }

  private:
    T* p_ = nullptr;
    int64_t n_ = 0;
    cudaStream_t stream_ = nullptr;
};

template <class T>
inline void d2h(T* dst, const T* src, int64_t n, cudaStream_t s) {
    if (n > 0) CK(cudaMemcpyAsync(dst, src, sizeof(T) * static_cast<size_t>(n), cudaMemcpyDeviceToHost, s));
}
template <class T>
inline void h2d(T* dst, const T* src, int64_t n, cudaStream_t s) {
    if (n > 0) CK(cudaMemcpyAsync(dst, src, sizeof(T) * static_cast<size_t>(n), cudaMemcpyHostToDevice, s));
}
template <class T>
inline void d2d(T* dst, const T* src, int64_t n, cudaStream_t s) {
    if (n > 0) CK(cudaMemcpyAsync(dst, src, sizeof(T) * static_cast<size_t>(n), cudaMemcpyDeviceToDevice, s));
}
template <class T>
inline T d2h_scalar(const T* src, cudaStream_t s) {
    T v{};
    CK(cudaMemcpyAsync(&v, src, sizeof(T), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return v;
}

// ---- kernel gating ---------------------------------------------------------
// Krylov control flow lives on the device: every kernel of an iteration takes
// a Gate and returns immediately when the solver state says so, so the host
// can enqueue whole iterations without a round trip per decision.
struct Gate {
    const int* flags = nullptr;  // nullptr => always run
    int skip_mask = 0;           // run only if (flags & skip_mask) == 0
    int need_mask = 0;           // ... and (flags & need_mask) == need_mask
};

__device__ __forceinline__ bool gated_off(const Gate& g) {
    if (!g.flags) return false;
    const int f = *reinterpret_cast<const volatile int*>(g.flags);
    return (f & g.skip_mask) != 0 || (f & g.need_mask) != g.need_mask;
}

// Solver state flags.
enum : int {
    KF_DONE = 1,        // solve finished (converged, breakdown or max_iter)
    KF_CONVERGED = 2,
    KF_BREAKDOWN = 4,
    KF_HALF = 8,        // this iteration took the half-step exit test (bicgstab.cpp:91)
    KF_CHECK = 16,      // a true-residual confirmation is pending
    KF_FIRST = 32,      // first iteration (p = r)
};

}  // namespace amgr

// Opaque C-ABI context handle (include/amgr.h): wraps the library context.
struct amgr_ctx {
    amgr::Ctx c;
};
