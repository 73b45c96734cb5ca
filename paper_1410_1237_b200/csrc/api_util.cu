// api_util.cu -- error reporting and device checks for the libplv C ABI.
#include "common.cuh"
#include <cstring>
#include <atomic>

namespace plv {

static thread_local char g_err[1024] = "";
static std::atomic<unsigned long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

static thread_local cudaStream_t g_alloc_stream[64] = {};

static void pool_setup(int dev) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = 64ull << 30;  // keep up to 64 GB mapped between phases
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
}

static cudaStream_t alloc_stream() {
    int dev = 0;
    PLV_CUDA(cudaGetDevice(&dev));
    if (!g_alloc_stream[dev & 63])
        PLV_CUDA(cudaStreamCreateWithFlags(&g_alloc_stream[dev & 63], cudaStreamNonBlocking));
    return g_alloc_stream[dev & 63];
}

void *pool_alloc(size_t bytes) {
    cudaStream_t s = alloc_stream();
    void *p = nullptr;
    PLV_CUDA(cudaMallocAsync(&p, bytes ? bytes : 1, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    return p;
}

static thread_local unsigned long long g_free_fail = 0;

unsigned long long pool_free_failures() { return g_free_fail; }

void pool_free(void *p) {
    if (!p) return;
    cudaError_t e = cudaFreeAsync(p, alloc_stream());
    if (e != cudaSuccess) {
        cudaGetLastError();
        g_free_fail++;
        set_error("cudaFreeAsync failed: %s", cudaGetErrorString(e));
    }
}

void check_device() {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error("no CUDA device: %s (libplv has no CPU fallback)", cudaGetErrorString(e));
        throw Fail{PLV_ENODEV};
    }
    static thread_local int checked_dev = -1;
    if (checked_dev == dev) return;
    int major = 0;
    e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (e != cudaSuccess || major != 10) {
        cudaGetLastError();
        set_error("libplv is built for sm_100a; device %d has compute capability major %d", dev,
                  major);
        throw Fail{PLV_ENODEV};
    }
    static int pooled[64] = {};
    if (!pooled[dev & 63]) {
        pool_setup(dev);
        pooled[dev & 63] = 1;
    }
    checked_dev = dev;
}

}  // namespace plv

extern "C" int plv_abi_version(void) { return 1; }

extern "C" unsigned long long plv_launch_count(void) { return plv::g_launches.load(); }

extern "C" const char *plv_last_error(void) { return plv::g_err; }

extern "C" int plv_device_ok(void) {
    try {
        plv::check_device();
    } catch (plv::Fail &) {
        return 0;
    }
    return 1;
}
