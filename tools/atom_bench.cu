// Latency of the flat-tier accumulate pattern: each thread claims a random
// slot (CAS), then RED f64 + RED s32 into it; FK entries per thread.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned hsh(unsigned x) {
    x ^= x >> 16; x *= 0x85EBCA6Bu; x ^= x >> 13; x *= 0xC2B2AE35u; x ^= x >> 16; return x;
}
template <int MODE, int FK>
__global__ void k(int *keys, double *vals, int *cnt, unsigned mask, unsigned long long *out, int salt) {
    unsigned long long t0 = gt();
    for (int k = 0; k < FK; k++) {
        unsigned id = (blockIdx.x * blockDim.x + threadIdx.x) * FK + k + salt;
        int c = (int)(hsh(id) & 0x3fffffff);
        unsigned s = hsh(c) & mask;
        if (MODE & 1) {
            while (true) {
                int old = atomicCAS(keys + s, -1, c);
                if (old == -1 || old == c) break;
                s = (s + 1) & mask;
            }
        }
        if (MODE & 2) atomicAdd(vals + s, 1.5);
        if (MODE & 4) atomicAdd(cnt + s, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = gt() - t0;
}
int main() {
    const unsigned T = 1 << 22;
    int *keys, *cnt; double *vals; unsigned long long *out, h[1024];
    cudaMalloc(&keys, 4 * T); cudaMalloc(&cnt, 4 * T); cudaMalloc(&vals, 8 * T); cudaMalloc(&out, 8 * 1024);
    cudaMemset(keys, 0xff, 4 * T);
    int nb = 60;
    for (int rep = 0; rep < 2; rep++) {
#define RUN(M) { cudaMemset(keys, 0xff, 4 * T); k<M, 2><<<nb, 256>>>(keys, vals, cnt, T - 1, out, rep * 1000003); \
        cudaMemcpy(h, out, 8 * nb, cudaMemcpyDeviceToHost); double s = 0, mx = 0; \
        for (int i = 0; i < nb; i++) { s += h[i]; if (h[i] > mx) mx = h[i]; } \
        printf("mode %d (cas=%d f64=%d s32=%d): mean %.2f us max %.2f us\n", M, M & 1, (M >> 1) & 1, (M >> 2) & 1, s / nb / 1e3, mx / 1e3); }
        RUN(1) RUN(2) RUN(4) RUN(3) RUN(7)
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
