// gen.cu -- counter-based synthetic graphs for the BASELINE.json configs.
//
// Every random draw is u = rnd01(stream_key(seed, stream), counter) (SplitMix64,
// common.cuh), so the device output is bit-identical to the numpy generators
// in paper_1410_1237_b200/synthetic.py (same draws, same record order, same
// float64 arithmetic without contraction).  Records are emitted in the order
// the numpy version produces them (stable compaction of kept candidates).
#include "common.cuh"
#include "csr.cuh"
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

namespace plv {

// ------------------------------------------------------------------ R-MAT
struct Rmat {
    uint64_t klvl, kw;
    int scale;
    double a, ab, abc, w_lo, span;
    __device__ __forceinline__ void edge(int64_t r, int32_t &u, int32_t &v) const {
        uint32_t s = 0, d = 0;
        for (int l = 0; l < scale; l++) {
            double x = rnd01(klvl, (uint64_t)r * (uint64_t)scale + (uint64_t)l);
            uint32_t ub = x >= ab;
            uint32_t vb = (x >= a && x < ab) || x >= abc;
            s = (s << 1) | ub;
            d = (d << 1) | vb;
        }
        u = (int32_t)s;
        v = (int32_t)d;
    }
    __device__ __forceinline__ bool operator()(int64_t r) const {
        int32_t u, v;
        edge(r, u, v);
        return u != v;
    }
};

__global__ void k_rmat_emit(Rmat g, const int64_t *sel, int64_t cnt, int32_t *u, int32_t *v,
                            double *w) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = sel[t];
        g.edge(r, u[t], v[t]);
        w[t] = dadd(g.w_lo, dmul(g.span, rnd01(g.kw, (uint64_t)r)));
    }
}

template <class Pred>
static int64_t select_if(Pred p, int64_t n, int64_t *out, cudaStream_t s) {
    Buf<int64_t> cnt(1, s);
    thrust::counting_iterator<int64_t> it(0);
    size_t bytes = 0;
    PLV_CUDA(cub::DeviceSelect::If(nullptr, bytes, it, out, cnt.get(), n, p, s));
    Buf<char> tmp(bytes, s);
    PLV_CUDA(cub::DeviceSelect::If(tmp.get(), bytes, it, out, cnt.get(), n, p, s));
    return d2h(cnt.get(), s);
}

// ------------------------------------------------------------------ SBM
struct Sbm {
    uint64_t key;
    int64_t n, block;
    double p_in, p_out;
    __device__ __forceinline__ bool operator()(int64_t p) const {
        int64_t i = p / n, j = p % n;
        if (j <= i) return false;
        double pr = (i / block == j / block) ? p_in : p_out;
        return rnd01(key, (uint64_t)p) < pr;
    }
};

__global__ void k_sbm_emit(int64_t n, const int64_t *sel, int64_t cnt, int32_t *u, int32_t *v,
                           double *w) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = sel[t];
        u[t] = (int32_t)(p / n);
        v[t] = (int32_t)(p % n);
        w[t] = 1.0;
    }
}

// ------------------------------------------------------------------ grid
struct Grid {
    uint64_t kkeep;
    double keep;
    __device__ __forceinline__ bool operator()(int64_t e) const {
        return rnd01(kkeep, (uint64_t)e) < keep;
    }
};

__global__ void k_grid_emit(int64_t side, uint64_t kw, double w_lo, const int64_t *sel,
                            int64_t cnt, int32_t *u, int32_t *v, double *w) {
    int64_t H = side * (side - 1);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t e = sel[t];
        int64_t a, b;
        if (e < H) {
            int64_t r = e / (side - 1), c = e % (side - 1);
            a = r * side + c;
            b = a + 1;
        } else {
            int64_t f = e - H;
            int64_t r = f / side, c = f % side;
            a = r * side + c;
            b = a + side;
        }
        u[t] = (int32_t)a;
        v[t] = (int32_t)b;
        w[t] = dadd(w_lo, rnd01(kw, (uint64_t)e));
    }
}

__global__ void k_pendants(int64_t N, int64_t P, uint64_t kp, uint64_t kpw, double w_lo,
                           int32_t *u, int32_t *v, double *w) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        u[p] = (int32_t)(N + p);
        v[p] = (int32_t)(int64_t)dmul(rnd01(kp, (uint64_t)p), (double)N);
        w[p] = dadd(w_lo, rnd01(kpw, (uint64_t)p));
    }
}

// ------------------------------------------------------------------ Chung-Lu
struct ChungLu {
    uint64_t key;
    const double *cdf;
    int64_t n;
    double total;
    __device__ __forceinline__ int64_t draw(uint64_t ctr) const {
        double x = dmul(rnd01(key, ctr), total);
        // searchsorted(cdf, x, side='right'): first index with cdf[idx] > x
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (cdf[mid] > x)
                hi = mid;
            else
                lo = mid + 1;
        }
        return lo < n ? lo : n - 1;
    }
    __device__ __forceinline__ bool operator()(int64_t r) const {
        return draw(2ull * (uint64_t)r) != draw(2ull * (uint64_t)r + 1ull);
    }
};

__global__ void k_cl_emit(ChungLu g, const int64_t *sel, int64_t cnt, int32_t *u, int32_t *v,
                          double *w) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = sel[t];
        u[t] = (int32_t)g.draw(2ull * (uint64_t)r);
        v[t] = (int32_t)g.draw(2ull * (uint64_t)r + 1ull);
        w[t] = 1.0;
    }
}

}  // namespace plv

using namespace plv;

extern "C" int plv_gen_rmat(uint64_t seed, int scale, int64_t edge_factor, double a, double b,
                            double c, double w_lo, double w_hi, int32_t *u, int32_t *v, double *w,
                            int64_t cap, int64_t *count_h, void *stream) {
    PLV_ENTRY
    cudaStream_t s = S(stream);
    if (scale < 1 || scale > 30) PLV_FAIL(PLV_EINVAL, "rmat scale out of range");
    int64_t R = edge_factor << scale;
    Rmat g{stream_key(seed, 1), stream_key(seed, 2), scale, a, a + b, (a + b) + c, w_lo, w_hi - w_lo};
    Buf<int64_t> sel(R, s);
    int64_t cnt = select_if(g, R, sel, s);
    if (cnt > cap) PLV_FAIL(PLV_EINVAL, "rmat: output capacity %lld < %lld", (long long)cap,
                            (long long)cnt);
    if (cnt) {
        k_rmat_emit<<<grid_for(cnt, 256), 256, 0, s>>>(g, sel, cnt, u, v, w);
        PLV_LAUNCH_CHECK();
    }
    *count_h = cnt;
    PLV_EXIT
}

extern "C" int plv_gen_sbm(uint64_t seed, int64_t n, int64_t block, double p_in, double p_out,
                           int32_t *u, int32_t *v, double *w, int64_t cap, int64_t *count_h,
                           void *stream) {
    PLV_ENTRY
    cudaStream_t s = S(stream);
    Sbm g{stream_key(seed, 3), n, block, p_in, p_out};
    int64_t P = n * n;
    Buf<int64_t> cntb(1, s);
    int64_t cnt = 0;
    const int64_t CH = 1ll << 27;  // chunked selection keeps scratch bounded
    for (int64_t p0 = 0; p0 < P; p0 += CH) {
        int64_t len = P - p0 < CH ? P - p0 : CH;
        Buf<int64_t> sel(len, s);
        thrust::counting_iterator<int64_t> it(p0);
        size_t bytes = 0;
        PLV_CUDA(cub::DeviceSelect::If(nullptr, bytes, it, sel.get(), cntb.get(), len, g, s));
        Buf<char> tmp(bytes, s);
        PLV_CUDA(cub::DeviceSelect::If(tmp.get(), bytes, it, sel.get(), cntb.get(), len, g, s));
        int64_t c = d2h(cntb.get(), s);
        if (cnt + c > cap) PLV_FAIL(PLV_EINVAL, "sbm: output capacity exceeded");
        if (c) {
            k_sbm_emit<<<grid_for(c, 256), 256, 0, s>>>(n, sel, c, u + cnt, v + cnt, w + cnt);
            PLV_LAUNCH_CHECK();
        }
        cnt += c;
    }
    *count_h = cnt;
    PLV_EXIT
}

extern "C" int plv_gen_grid(uint64_t seed, int64_t side, double keep, int64_t pendants,
                            double w_lo, int32_t *u, int32_t *v, double *w, int64_t cap,
                            int64_t *count_h, void *stream) {
    PLV_ENTRY
    cudaStream_t s = S(stream);
    int64_t N = side * side;
    int64_t E = 2 * side * (side - 1);
    Grid g{stream_key(seed, 4), keep};
    Buf<int64_t> sel(E, s);
    int64_t cnt = select_if(g, E, sel, s);
    if (cnt + pendants > cap) PLV_FAIL(PLV_EINVAL, "grid: output capacity exceeded");
    if (cnt) {
        k_grid_emit<<<grid_for(cnt, 256), 256, 0, s>>>(side, stream_key(seed, 5), w_lo, sel, cnt, u,
                                                      v, w);
        PLV_LAUNCH_CHECK();
    }
    if (pendants) {
        k_pendants<<<grid_for(pendants, 256), 256, 0, s>>>(N, pendants, stream_key(seed, 6),
                                                          stream_key(seed, 7), w_lo, u + cnt,
                                                          v + cnt, w + cnt);
        PLV_LAUNCH_CHECK();
    }
    *count_h = cnt + pendants;
    PLV_EXIT
}

extern "C" int plv_gen_chung_lu(uint64_t seed, const double *cdf, int64_t n, int64_t records,
                                int32_t *u, int32_t *v, double *w, int64_t cap, int64_t *count_h,
                                void *stream) {
    PLV_ENTRY
    cudaStream_t s = S(stream);
    double total = d2h(cdf + n - 1, s);
    ChungLu g{stream_key(seed, 8), cdf, n, total};
    Buf<int64_t> sel(records, s);
    int64_t cnt = select_if(g, records, sel, s);
    if (cnt > cap) PLV_FAIL(PLV_EINVAL, "chung-lu: output capacity exceeded");
    if (cnt) {
        k_cl_emit<<<grid_for(cnt, 256), 256, 0, s>>>(g, sel, cnt, u, v, w);
        PLV_LAUNCH_CHECK();
    }
    *count_h = cnt;
    PLV_EXIT
}
