// Latency probes on one thread (B200): dependent global loads (L2-resident
// and DRAM), atomicCAS / atomicAdd round trips, globaltimer resolution.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_chase(const int *next, int steps, long long *out, int *sink) {
    int p = 0;
    long long c0 = clock64();
    for (int s = 0; s < steps; s++) p = __ldcg(next + p);
    long long c1 = clock64();
    out[0] = (c1 - c0) / steps;
    *sink = p;
}

__global__ void k_cas(int *a, int steps, long long *out) {
    int v = 0;
    long long c0 = clock64();
    for (int s = 0; s < steps; s++) v = atomicCAS(a + (v & 1023) * 32, -1, s) & 7;
    long long c1 = clock64();
    out[0] = (c1 - c0) / steps;
    out[1] = v;
}

__global__ void k_add(int *a, int steps, long long *out) {
    int v = 0;
    long long c0 = clock64();
    for (int s = 0; s < steps; s++) v = atomicAdd(a + (v & 1023) * 32, 1) & 7;
    long long c1 = clock64();
    out[0] = (c1 - c0) / steps;
}

__global__ void k_gt(long long *out) {
    unsigned long long t0 = gt(), t = t0;
    int changes = 0;
    unsigned long long mind = ~0ull;
    for (int s = 0; s < 100000 && changes < 50; s++) {
        unsigned long long u = gt();
        if (u != t) {
            if (u - t < mind) mind = u - t;
            t = u;
            changes++;
        }
    }
    out[0] = mind;
}

int main() {
    const int N = 1 << 26;  // 256 MB of ints for DRAM chase
    int *next, *sink, *a;
    long long *out, h[2];
    cudaMalloc(&next, sizeof(int) * (size_t)N);
    cudaMalloc(&sink, 4);
    cudaMalloc(&a, sizeof(int) * 1024 * 32);
    cudaMalloc(&out, 16);
    cudaMemset(a, 0xff, sizeof(int) * 1024 * 32);
    int *hn = new int[N];
    // random cycle with stride over a span: small span = L2 resident
    for (int span : {1 << 14, 1 << 20, N}) {
        unsigned long long x = 88172645463325252ull;
        for (int i = 0; i < span; i++) hn[i] = i;
        for (int i = span - 1; i > 0; i--) {
            x ^= x << 13; x ^= x >> 7; x ^= x << 17;
            int j = (int)(x % (unsigned long long)(i + 1));
            int t = hn[i]; hn[i] = hn[j]; hn[j] = t;
        }
        // hn is a permutation; use it as a single chase order
        int *nx = new int[span];
        for (int i = 0; i < span; i++) nx[hn[i]] = hn[(i + 1) % span];
        cudaMemcpy(next, nx, sizeof(int) * span, cudaMemcpyHostToDevice);
        delete[] nx;
        k_chase<<<1, 1>>>(next, 2000, out, sink);
        k_chase<<<1, 1>>>(next, 20000, out, sink);
        cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
        printf("chase span %d ints (%d KB): %lld cycles/load\n", span, span / 256, h[0]);
    }
    k_cas<<<1, 1>>>(a, 10000, out);
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("atomicCAS round trip: %lld cycles\n", h[0]);
    k_add<<<1, 1>>>(a, 10000, out);
    cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
    printf("atomicAdd (returning) round trip: %lld cycles\n", h[0]);
    k_gt<<<1, 1>>>(out);
    cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
    printf("globaltimer min increment: %lld ns\n", h[0]);
    printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
