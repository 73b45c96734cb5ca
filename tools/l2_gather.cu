// Effective L2 capacity for random gathers beside a streamed read (B200):
// N threads each gather 4-byte words at uniform random positions of an array
// of S bytes while streaming 12 bytes per gather with an evict-first policy
// (the decide kernels' pattern: rows streamed, assignment / a_tot gathered).
//   nvcc -O3 -arch=sm_100a -o tools/l2_gather tools/l2_gather.cu && tools/l2_gather
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ int ld_first(const int *p) {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    int v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

template <int ES>  // gathered element size in 4-byte words (1: int, 2: double)
__global__ void k_gather(const int *arr, uint64_t nelem, const int *stream, uint64_t nstream,
                         uint64_t per_thread, int with_stream, int *sink) {
    uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
    int acc = 0;
    for (uint64_t r = 0; r < per_thread; r += 8) {
        int v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            uint64_t idx = mix((r + u) * nt + t) % nelem;
            v[u] = __ldcg(arr + idx * ES);
        }
        if (with_stream) {
#pragma unroll
            for (int u = 0; u < 8; u++) {
                uint64_t p = ((r + u) * nt + t) * 3 % nstream;
                acc += ld_first(stream + p) + ld_first(stream + p + 1) + ld_first(stream + p + 2);
            }
        }
#pragma unroll
        for (int u = 0; u < 8; u++) acc += v[u];
    }
    if (acc == 0x7fffffff) *sink = acc;
}

int main() {
    const uint64_t MAXB = 512ull << 20, SB = 2048ull << 20;
    int *arr, *stream, *sink;
    cudaMalloc(&arr, MAXB);
    cudaMalloc(&stream, SB);
    cudaMalloc(&sink, 4);
    cudaMemset(arr, 1, MAXB);
    cudaMemset(stream, 1, SB);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = 148 * 8, threads = 256;
    const uint64_t per_thread = 512;
    const double gathers = (double)blocks * threads * per_thread;
    for (int with_stream = 0; with_stream < 2; with_stream++)
        for (int mb : {16, 32, 48, 64, 80, 96, 112, 128, 160, 192, 256, 384}) {
            uint64_t nelem = ((uint64_t)mb << 20) / 4;
            for (int rep = 0; rep < 3; rep++) {
                cudaEventRecord(e0);
                k_gather<1><<<blocks, threads>>>(arr, nelem, stream, SB / 4 - 4, per_thread, with_stream, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep == 2)
                    printf("stream %d  array %4d MB  %7.3f ms  %6.1f G gathers/s\n", with_stream, mb, ms,
                           gathers / ms / 1e6);
            }
        }
    return 0;
}
