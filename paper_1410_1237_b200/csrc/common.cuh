// common.cuh -- shared helpers for libplv (B200 / sm_100a parallel Louvain).
//
// Error model: C++ code throws plv::Fail; every extern "C" entry point wraps
// its body in PLV_ENTRY / PLV_EXIT, which converts to a PLV_E* status and
// records a thread-local message for plv_last_error().
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <string>
#include <stdexcept>
#include <utility>

#include "../../include/plv.h"

namespace plv {

struct Fail {
    int code;
};

void set_error(const char *fmt, ...);
void check_device();  // throws PLV_ENODEV unless an sm_100 device is current

#define PLV_CUDA(x)                                                                   \
    do {                                                                              \
        cudaError_t _e = (x);                                                         \
        if (_e != cudaSuccess) {                                                      \
            plv::set_error("%s: %s (%s:%d)", #x, cudaGetErrorString(_e), __FILE__,     \
                           __LINE__);                                                 \
            throw plv::Fail{PLV_ECUDA};                                               \
        }                                                                             \
    } while (0)

// Every kernel launch of this library is followed by PLV_LAUNCH_CHECK, which
// also counts it (plv_launch_count(): evidence of the native path for bench.py).
void count_launch();
#define PLV_LAUNCH_CHECK()                \
    do {                                  \
        plv::count_launch();              \
        PLV_CUDA(cudaGetLastError());     \
    } while (0)

#define PLV_FAIL(code, ...)              \
    do {                                 \
        plv::set_error(__VA_ARGS__);     \
        throw plv::Fail{code};           \
    } while (0)

#define PLV_ENTRY       \
    try {               \
        plv::check_device();

#define PLV_EXIT                                  \
    }                                             \
    catch (plv::Fail & f) {                       \
        return f.code;                            \
    }                                             \
    catch (std::exception & e) {                  \
        plv::set_error("%s", e.what());           \
        return PLV_ECUDA;                         \
    }                                             \
    return PLV_OK;

inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Long-lived device buffers (phase plans, engine state) come from the
// device's default memory pool, which keeps freed memory mapped (release
// threshold raised at first use of a device, api_util.cu): phases allocate
// and free hundreds of MB each, and cudaMalloc / cudaFree of fresh pages
// cost milliseconds and synchronise the device.  pool_free needs the buffer
// idle (callers synchronise first).
void *pool_alloc(size_t bytes);
void pool_free(void *p);
unsigned long long pool_free_failures();  // failed pool_free calls on this thread

// Stream-ordered scratch buffer (cudaMallocAsync pool); freed on scope exit.
template <class T>
struct Buf {
    T *p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    Buf() = default;
    Buf(size_t count, cudaStream_t st) { alloc(count, st); }
    void alloc(size_t count, cudaStream_t st) {
        release();
        s = st;
        n = count;
        if (count) PLV_CUDA(cudaMallocAsync((void **)&p, sizeof(T) * count, st));
    }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    ~Buf() { release(); }
    Buf(const Buf &) = delete;
    Buf &operator=(const Buf &) = delete;
    T *get() const { return p; }
    operator T *() const { return p; }
};

// Programmatic dependent launch (sm_90+).  A kernel launched with
// launch_pdl may be scheduled while its predecessor in the stream is still
// finishing; it must execute pdl_wait() before touching anything the
// predecessor writes (the wait returns at once for ordinary launches).
// pdl_trigger() lets the next PDL kernel start launching early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

// Loads of the local-moving kernels.  CSR rows are immutable during a phase
// and streamed once per sweep: read-only path, no L1 allocation, L2
// evict-first.  The state (assignment, a_tot, sizes) is mutable, so it is read
// coherently at L2 (ld.global.cg), never through the non-coherent path (a
// kernel that decides and applies several stages between cluster / grid
// barriers must not see stale lines).  Measured: L2 evict_last / .nc hints on
// the state gathers changed nothing.
__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ int32_t ld_row(const int32_t *p) {
    int32_t v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
        : "=r"(v) : "l"(p), "l"(pol_first()));
    return v;
}
__device__ __forceinline__ double ld_row(const double *p) {
    double v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
        : "=d"(v) : "l"(p), "l"(pol_first()));
    return v;
}
__device__ __forceinline__ int32_t ld_state(const int32_t *p) { return __ldcg(p); }
__device__ __forceinline__ double ld_state(const double *p) { return __ldcg(p); }
__device__ __forceinline__ uint8_t ld_state(const uint8_t *p) { return __ldcg(p); }

void count_launch();
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    PLV_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
    count_launch();
}

inline unsigned grid_for(int64_t work, int block, int64_t cap = 148 * 64) {
    int64_t g = (work + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

inline int bits_for(int64_t n) {
    int b = 1;
    while (b < 62 && ((int64_t)1 << b) < n) b++;
    return b;
}

template <class T>
T d2h(const T *dev, cudaStream_t s) {
    T v;
    PLV_CUDA(cudaMemcpyAsync(&v, dev, sizeof(T), cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    return v;
}

// ------------------------------------------------------------ fp helpers
// The reference is compiled with -ffp-contract=off (pkg/setup.py:32): every
// product and sum is rounded separately.  We build with --fmad=false and use
// explicit _rn intrinsics on every parity-critical expression.
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// ------------------------------------------------ ordered long folds
// Exact reproduction of a sequential float64 fold needs its additions in
// order: the dependency chain is inherent.  To make the chain the only cost,
// a whole block stages the operands chunk by chunk into shared memory
// (parallel, high-MLP loads, double-buffered) while thread 0 runs the
// dependent additions out of shared memory.  `get(t)` yields operand t.
// Call with every thread of the block; the result is valid in thread 0.
// `sb` must hold 2 * FOLD_CH doubles.
constexpr int FOLD_CH = 1024;

template <class Get>
__device__ double block_fold(Get get, int64_t len, double init, double *sb) {
    double v = init;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int t = tid; t < FOLD_CH; t += nt)
        if (t < len) sb[t] = get(t);
    __syncthreads();
    const int64_t nch = (len + FOLD_CH - 1) / FOLD_CH;
    for (int64_t c = 0; c < nch; c++) {
        const double *cur = sb + (c & 1) * FOLD_CH;
        double *nxt = sb + ((c + 1) & 1) * FOLD_CH;
        if (tid == 0) {
            int64_t m = len - c * FOLD_CH;
            m = m < FOLD_CH ? m : FOLD_CH;
            int64_t t = 0;
            for (; t + 4 <= m; t += 4) {
                double a0 = cur[t], a1 = cur[t + 1], a2 = cur[t + 2], a3 = cur[t + 3];
                v = __dadd_rn(v, a0);
                v = __dadd_rn(v, a1);
                v = __dadd_rn(v, a2);
                v = __dadd_rn(v, a3);
            }
            for (; t < m; t++) v = __dadd_rn(v, cur[t]);
        } else {
            const int64_t base = (c + 1) * FOLD_CH;
            for (int t = tid - 1; t < FOLD_CH; t += nt - 1)
                if (base + t < len) nxt[t] = get(base + t);
        }
        __syncthreads();
    }
    return v;
}

// Two interleaved folds (independent chains) over operand pairs get(t) ->
// (x, y); results valid in thread 0.  `sb` holds 4 * FOLD_CH doubles.
template <class Get>
__device__ void block_fold2(Get get, int64_t len, double &vx, double &vy, double *sb) {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int t = tid; t < FOLD_CH; t += nt)
        if (t < len) get(t, sb[t], sb[2 * FOLD_CH + t]);
    __syncthreads();
    const int64_t nch = (len + FOLD_CH - 1) / FOLD_CH;
    for (int64_t c = 0; c < nch; c++) {
        const int b = (int)(c & 1), nb = (int)((c + 1) & 1);
        if (tid == 0) {
            int64_t m = len - c * FOLD_CH;
            m = m < FOLD_CH ? m : FOLD_CH;
            const double *cx = sb + b * FOLD_CH, *cy = sb + 2 * FOLD_CH + b * FOLD_CH;
            for (int64_t t = 0; t < m; t++) {
                vx = __dadd_rn(vx, cx[t]);
                vy = __dadd_rn(vy, cy[t]);
            }
        } else {
            const int64_t base = (c + 1) * FOLD_CH;
            for (int t = tid - 1; t < FOLD_CH; t += nt - 1)
                if (base + t < len)
                    get(base + t, sb[nb * FOLD_CH + t], sb[2 * FOLD_CH + nb * FOLD_CH + t]);
        }
        __syncthreads();
    }
}

// --------------------------------------------------- counter-based RNG
// SplitMix64 finaliser; u64(key, i) is the i-th SplitMix64 output for state
// `key`.  Mirrored bit-for-bit by paper_1410_1237_b200/synthetic.py.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
constexpr uint64_t GAMMA = 0x9E3779B97F4A7C15ull;
__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t stream) {
    return mix64(seed * 0xD1B54A32D192ED03ull + stream * GAMMA + 1ull);
}
__host__ __device__ __forceinline__ uint64_t rnd64(uint64_t key, uint64_t i) {
    return mix64(key + (i + 1ull) * GAMMA);
}
__host__ __device__ __forceinline__ double rnd01(uint64_t key, uint64_t i) {
    return (double)(rnd64(key, i) >> 11) * (1.0 / 9007199254740992.0);
}

}  // namespace plv
