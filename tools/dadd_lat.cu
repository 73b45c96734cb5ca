// Microbenchmark: latency of a dependent float64 add chain (one thread), from
// registers and from shared memory -- the floor of an exact sequential fold.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain_reg(double *out, int n, double w) {
    double v = 0.0, a = w, b = w * 0.5;
    long long t0 = clock64();
    for (int i = 0; i < n; i++) { v = __dadd_rn(v, a); v = __dadd_rn(v, b); }
    long long t1 = clock64();
    out[0] = v; out[1] = (double)(t1 - t0) / (2.0 * n);
}
__global__ void chain_smem(double *out, int n) {
    __shared__ double s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 1.0 + i * 1e-7;
    __syncthreads();
    if (threadIdx.x) return;
    double v = 0.0;
    long long t0 = clock64();
    for (int r = 0; r < n; r++)
        for (int i = 0; i < 4096; i += 4) {
            double a0 = s[i], a1 = s[i + 1], a2 = s[i + 2], a3 = s[i + 3];
            v = __dadd_rn(v, a0); v = __dadd_rn(v, a1); v = __dadd_rn(v, a2); v = __dadd_rn(v, a3);
        }
    long long t1 = clock64();
    out[2] = v; out[3] = (double)(t1 - t0) / (4096.0 * n);
}
int main() {
    double *d, h[4];
    cudaMalloc(&d, 4 * sizeof(double));
    chain_reg<<<1, 1>>>(d, 1 << 16, 1.000001);
    chain_smem<<<1, 256>>>(d, 16);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("dadd chain: %.2f cycles/add (registers), %.2f cycles/add (smem operands)\n", h[1], h[3]);
    return 0;
}
