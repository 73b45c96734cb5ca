// csr.cu -- Graph.from_edges on device (PL/graph.py:88-147 + :64-86).
//
// Pipeline (all stream-ordered, one host sync at the end for the sizes):
//   1. validate weights (finite, > 0) and ids (in [0, n))       PL/graph.py:104-110
//   2. key = (min << nb) | max ; stable radix sort (key, w)      np.lexsort((b, a))
//   3. run heads -> segment starts; merged weight per run with
//      numpy's reduceat rule  w[s] + pairwise(w[s+1:e])          PL/graph.py:116-127
//   4. CSR: row i = reversed records (a, i), a < i, ascending a,
//      then forward records (i, b), b >= i, ascending b.  Forward
//      entries are already grouped in the merged order; reversed
//      ones come from a stable 32-bit radix sort by b.           PL/graph.py:131-139
//   5. selfw, k_i = sequential fold of row i + selfw[i] (the
//      weighted np.bincount), m = pairwise(k) / 2                PL/graph.py:73-80
#include "common.cuh"
#include "pairwise.cuh"
#include "csr.cuh"
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

namespace plv {

// ------------------------------------------------------------ CUB wrappers

template <class K, class V>
void sort_pairs(const K *kin, K *kout, const V *vin, V *vout, int64_t n, int begin_bit,
                int end_bit, cudaStream_t s) {
    if (n <= 0) return;
    size_t bytes = 0;
    PLV_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, n, begin_bit,
                                             end_bit, s));
    Buf<char> tmp(bytes, s);
    PLV_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, kin, kout, vin, vout, n, begin_bit,
                                             end_bit, s));
}
template void sort_pairs<uint64_t, double>(const uint64_t *, uint64_t *, const double *, double *,
                                           int64_t, int, int, cudaStream_t);
template void sort_pairs<int32_t, int32_t>(const int32_t *, int32_t *, const int32_t *, int32_t *,
                                           int64_t, int, int, cudaStream_t);
template void sort_pairs<uint32_t, int32_t>(const uint32_t *, uint32_t *, const int32_t *,
                                            int32_t *, int64_t, int, int, cudaStream_t);

// out[j] = index i of every i with flags[i] != 0, in ascending order.
int64_t select_flagged_index(const uint8_t *flags, int64_t n, int64_t *out, cudaStream_t s) {
    if (n <= 0) return 0;
    Buf<int64_t> cnt(1, s);
    thrust::counting_iterator<int64_t> it(0);
    size_t bytes = 0;
    PLV_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, flags, out, cnt.get(), n, s));
    Buf<char> tmp(bytes, s);
    PLV_CUDA(cub::DeviceSelect::Flagged(tmp.get(), bytes, it, flags, out, cnt.get(), n, s));
    return d2h(cnt.get(), s);
}

int64_t select_flagged_index32(const uint8_t *flags, int64_t n, int32_t *out, cudaStream_t s) {
    if (n <= 0) return 0;
    Buf<int64_t> cnt(1, s);
    thrust::counting_iterator<int32_t> it(0);
    size_t bytes = 0;
    PLV_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, flags, out, cnt.get(), n, s));
    Buf<char> tmp(bytes, s);
    PLV_CUDA(cub::DeviceSelect::Flagged(tmp.get(), bytes, it, flags, out, cnt.get(), n, s));
    return d2h(cnt.get(), s);
}

// off[0..n] = exclusive prefix sum of deg[0..n) (int64 output), off[n] = total.
struct ToI64 {
    __host__ __device__ int64_t operator()(int32_t x) const { return (int64_t)x; }
};
void exclusive_offsets(const int32_t *deg, int64_t n, int64_t *off, cudaStream_t s) {
    // deg has n valid entries; scan n+1 items with an implicit trailing 0.
    thrust::transform_iterator<ToI64, const int32_t *, int64_t> it(deg, ToI64{});
    size_t bytes = 0;
    PLV_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, off, n, s));
    Buf<char> tmp(bytes, s);
    if (n > 0) PLV_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, it, off, n, s));
}

__global__ void k_offsets_tail(const int64_t *off, const int32_t *deg, int64_t n, int64_t *tail) {
    tail[0] = n > 0 ? off[n - 1] + deg[n - 1] : 0;
}

void offsets_from_degrees(const int32_t *deg, int64_t n, int64_t *off, cudaStream_t s) {
    if (n > 0) exclusive_offsets(deg, n, off, s);
    k_offsets_tail<<<1, 1, 0, s>>>(off, deg, n, off + n);
    PLV_LAUNCH_CHECK();
}

// rowidx[e] = row owning CSR entry e.
__global__ void k_row_heads(const int64_t *off, int64_t n, int32_t *head) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if (off[i + 1] > off[i]) head[off[i]] = (int32_t)i;
}
struct MaxOp {
    __device__ int32_t operator()(int32_t a, int32_t b) const { return a > b ? a : b; }
};
void row_index(const int64_t *off, int64_t n, int64_t nnz, int32_t *rowidx, cudaStream_t s) {
    if (nnz <= 0) return;
    PLV_CUDA(cudaMemsetAsync(rowidx, 0, sizeof(int32_t) * nnz, s));
    k_row_heads<<<grid_for(n, 256), 256, 0, s>>>(off, n, rowidx);
    PLV_LAUNCH_CHECK();
    size_t bytes = 0;
    PLV_CUDA(cub::DeviceScan::InclusiveScan(nullptr, bytes, rowidx, rowidx, MaxOp{}, nnz, s));
    Buf<char> tmp(bytes, s);
    PLV_CUDA(cub::DeviceScan::InclusiveScan(tmp.get(), bytes, rowidx, rowidx, MaxOp{}, nnz, s));
}

// ---------------------------------------------------------------- kernels

__global__ void k_validate(const int32_t *u, const int32_t *v, const double *w, int64_t R,
                           int64_t n, int *flags) {
    int bad_w = 0, bad_id = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
         r += (int64_t)gridDim.x * blockDim.x) {
        double x = w[r];
        if (!(isfinite(x) && x > 0.0)) bad_w = 1;
        if (u[r] < 0 || v[r] < 0 || u[r] >= n || v[r] >= n) bad_id = 1;
    }
    if (__syncthreads_or(bad_w) && threadIdx.x == 0) atomicOr(flags, 1);
    if (__syncthreads_or(bad_id) && threadIdx.x == 0) atomicOr(flags, 2);
}

__global__ void k_canon_keys(const int32_t *u, const int32_t *v, int64_t R, int nb, uint64_t *key) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
         r += (int64_t)gridDim.x * blockDim.x) {
        uint32_t a = (uint32_t)min(u[r], v[r]), b = (uint32_t)max(u[r], v[r]);
        key[r] = ((uint64_t)a << nb) | (uint64_t)b;
    }
}

__global__ void k_key_heads(const uint64_t *key, int64_t R, uint8_t *head) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
         r += (int64_t)gridDim.x * blockDim.x)
        head[r] = (r == 0 || key[r] != key[r - 1]) ? 1 : 0;
}

__global__ void k_decode_runs(const uint64_t *key, const int64_t *starts, int64_t M, int nb,
                              int32_t *am, int32_t *bm) {
    uint64_t mask = (1ull << nb) - 1ull;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M;
         t += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = key[starts[t]];
        am[t] = (int32_t)(k >> nb);
        bm[t] = (int32_t)(k & mask);
    }
}

// a[] is sorted: a row's forward records are one run, counted once by the
// run's last record (a hub's run would otherwise serialise its atomics on one
// counter); reversed records are counted per record.
__global__ void k_count_rows(const int32_t *a, const int32_t *b, int64_t M, int32_t *deg,
                             int32_t *nrev, uint8_t *nonself, int32_t *fstart) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M;
         t += (int64_t)gridDim.x * blockDim.x) {
        int32_t x = a[t], y = b[t];
        if (t == M - 1 || a[t + 1] != x) {
            int64_t lo = 0, hi = t;  // first record of the run
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (a[mid] < x)
                    lo = mid + 1;
                else
                    hi = mid;
            }
            atomicAdd(deg + x, (int32_t)(t - lo + 1));
            fstart[x] = (int32_t)lo;
        }
        if (x != y) {
            atomicAdd(deg + y, 1);
            atomicAdd(nrev + y, 1);
        }
        nonself[t] = (x != y);
    }
}

__global__ void k_place_forward(const int32_t *a, const int32_t *b, const double *w, int64_t M,
                                const int64_t *off, const int32_t *nrev, const int32_t *fstart,
                                int32_t *nbr, double *wts, double *selfw) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M;
         t += (int64_t)gridDim.x * blockDim.x) {
        int32_t x = a[t], y = b[t];
        int64_t p = off[x] + nrev[x] + (t - fstart[x]);
        nbr[p] = y;
        wts[p] = w[t];
        if (x == y) selfw[x] = w[t];
    }
}

__global__ void k_rev_heads(const int32_t *bkey, int64_t Mn, int32_t *rstart) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < Mn;
         p += (int64_t)gridDim.x * blockDim.x)
        if (p == 0 || bkey[p - 1] != bkey[p]) rstart[bkey[p]] = (int32_t)p;
}

__global__ void k_place_reverse(const int32_t *bkey, const int32_t *tidx, int64_t Mn,
                                const int32_t *a, const double *w, const int64_t *off,
                                const int32_t *rstart, int32_t *nbr, double *wts) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < Mn;
         p += (int64_t)gridDim.x * blockDim.x) {
        int32_t row = bkey[p];
        int32_t t = tidx[p];
        int64_t pos = off[row] + (p - rstart[row]);
        nbr[pos] = a[t];
        wts[pos] = w[t];
    }
}

// k_i = (((0 + w_0) + w_1) + ...) + selfw_i : the weighted np.bincount fold in
// CSR order (PL/graph.py:73-78).  Integral graphs may fold in any order.
constexpr int64_t DEG_LONG = 256;  // longer rows are folded by a whole block

__global__ void k_degrees(const int64_t *off, const double *wts, const double *selfw, int64_t n,
                          double *k, int32_t *longs, unsigned long long *nlong) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t e0 = off[i], e1 = off[i + 1];
        if (e1 - e0 > DEG_LONG) {  // listed for k_degrees_long
            longs[atomicAdd(nlong, 1ull)] = (int32_t)i;
            continue;
        }
        double acc = 0.0;
        for (int64_t e = e0; e < e1; e++) acc = __dadd_rn(acc, wts[e]);
        k[i] = __dadd_rn(acc, selfw[i]);
    }
}

// A long row's fold.  When every weight of the graph is an integer (stats[2]
// == 0, k_integral_check ran first) all partial sums of the row are integers
// below the row total, so a parallel tree is exact -- and equal to the
// sequential fold -- whenever its total is below 2^53 (a total at or above it
// cannot come out below, rounding being monotone); otherwise, and for
// non-integral graphs, the ordered block fold.
__global__ void __launch_bounds__(256) k_degrees_long(const int64_t *off, const double *wts,
                                                     const double *selfw, const int32_t *longs,
                                                     const unsigned long long *nlong, double *k,
                                                     const unsigned long long *stats) {
    __shared__ double sb[2 * FOLD_CH];
    typedef cub::BlockReduce<double, 256> BR;
    __shared__ typename BR::TempStorage red;
    __shared__ double s_tot;
    const bool integral = stats[2] == 0;
    const int64_t nl = (int64_t)*nlong;
    for (int64_t q = blockIdx.x; q < nl; q += gridDim.x) {
        const int64_t i = longs[q];
        const int64_t e0 = off[i], len = off[i + 1] - e0;
        bool done = false;
        if (integral) {
            double part = 0.0;
            for (int64_t t = threadIdx.x; t < len; t += 256) part = __dadd_rn(part, wts[e0 + t]);
            const double tot = BR(red).Sum(part);
            if (threadIdx.x == 0) s_tot = tot;
            __syncthreads();
            done = s_tot < 9007199254740992.0;
            if (done && threadIdx.x == 0) k[i] = __dadd_rn(s_tot, selfw[i]);
            __syncthreads();
        }
        if (!done) {
            double acc = block_fold([=] __device__(int64_t t) { return wts[e0 + t]; }, len, 0.0, sb);
            if (threadIdx.x == 0) k[i] = __dadd_rn(acc, selfw[i]);
            __syncthreads();
        }
    }
}

// stats: [0] num_self, [1] max_degree, [2] non-integral flag
__global__ void k_graph_stats(const int64_t *off, const double *selfw, int64_t n,
                              unsigned long long *stats) {
    unsigned long long ns = 0, md = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        ns += (selfw[i] != 0.0);
        unsigned long long d = (unsigned long long)(off[i + 1] - off[i]);
        md = d > md ? d : md;
    }
    typedef cub::BlockReduce<unsigned long long, 256> BR;
    __shared__ typename BR::TempStorage tmp;
    unsigned long long tns = BR(tmp).Sum(ns);
    __syncthreads();
    unsigned long long tmd = BR(tmp).Reduce(md, cub::Max());
    if (threadIdx.x == 0) {
        if (tns) atomicAdd(stats + 0, tns);
        atomicMax(stats + 1, tmd);
    }
}

__global__ void k_integral_check(const double *w, int64_t M, unsigned long long *stats) {
    int bad = 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M;
         t += (int64_t)gridDim.x * blockDim.x) {
        double x = w[t];
        if (x != floor(x) || x >= 4503599627370496.0) bad = 1;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(stats + 2, 1ull);
}

__global__ void k_half(const double *sum, double *m) { m[0] = __ddiv_rn(sum[0], 2.0); }

// ------------------------------------------------------------- CSR from runs

// Builds the CSR from merged records sorted by (a, b), a <= b, unique.
void csr_from_merged(const int32_t *a, const int32_t *b, const double *w, int64_t M, int64_t n,
                     int64_t merged, int64_t *off, int32_t *nbr, double *wts, double *selfw,
                     double *k, int64_t *info_h, double *m_h, cudaStream_t s) {
    Buf<int32_t> deg(n + 1, s), nrev(n + 1, s), fstart(n + 1, s), rstart(n + 1, s);
    Buf<uint8_t> nonself(M + 1, s);
    PLV_CUDA(cudaMemsetAsync(deg.get(), 0, sizeof(int32_t) * (n + 1), s));
    PLV_CUDA(cudaMemsetAsync(nrev.get(), 0, sizeof(int32_t) * (n + 1), s));
    if (n > 0) PLV_CUDA(cudaMemsetAsync(selfw, 0, sizeof(double) * n, s));
    if (M > 0) {
        k_count_rows<<<grid_for(M, 256), 256, 0, s>>>(a, b, M, deg, nrev, nonself, fstart);
        PLV_LAUNCH_CHECK();
    }
    offsets_from_degrees(deg, n, off, s);
    if (M > 0) {
        k_place_forward<<<grid_for(M, 256), 256, 0, s>>>(a, b, w, M, off, nrev, fstart, nbr, wts,
                                                        selfw);
        PLV_LAUNCH_CHECK();
        Buf<int32_t> tidx(M, s);
        int64_t Mn = select_flagged_index32(nonself, M, tidx, s);
        if (Mn > 0) {
            Buf<int32_t> bkey(Mn, s), bkey_s(Mn, s), tidx_s(Mn, s);
            gather_i32(b, tidx.get(), Mn, bkey.get(), s);  // b of the non-self records
            sort_pairs<int32_t, int32_t>(bkey.get(), bkey_s.get(), tidx.get(), tidx_s.get(), Mn, 0,
                                         bits_for(n), s);
            k_rev_heads<<<grid_for(Mn, 256), 256, 0, s>>>(bkey_s, Mn, rstart);
            PLV_LAUNCH_CHECK();
            k_place_reverse<<<grid_for(Mn, 256), 256, 0, s>>>(bkey_s, tidx_s, Mn, a, w, off, rstart,
                                                             nbr, wts);
            PLV_LAUNCH_CHECK();
        }
    }
    Buf<unsigned long long> stats(3, s);
    PLV_CUDA(cudaMemsetAsync(stats.get(), 0, sizeof(unsigned long long) * 3, s));
    if (M > 0) {
        k_integral_check<<<grid_for(M, 256), 256, 0, s>>>(w, M, stats);
        PLV_LAUNCH_CHECK();
    }
    if (n > 0) {
        // rows longer than DEG_LONG: listed by k_degrees, a block each
        const int64_t lcap = 2 * M / DEG_LONG + 2;  // nnz <= 2M
        Buf<int32_t> longs(lcap, s);
        Buf<unsigned long long> nlong(1, s);
        PLV_CUDA(cudaMemsetAsync(nlong.get(), 0, sizeof(unsigned long long), s));
        k_degrees<<<grid_for(n, 128), 128, 0, s>>>(off, wts, selfw, n, k, longs, nlong);
        PLV_LAUNCH_CHECK();
        k_degrees_long<<<148 * 4, 256, 0, s>>>(off, wts, selfw, longs, nlong, k, stats.get());
        PLV_LAUNCH_CHECK();
        k_graph_stats<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(off, selfw, n, stats);
        PLV_LAUNCH_CHECK();
    }
    Buf<double> msum(2, s);
    pw_sum_async(k, n, msum.get(), s);
    k_half<<<1, 1, 0, s>>>(msum.get(), msum.get() + 1);
    PLV_LAUNCH_CHECK();
    unsigned long long st[3];
    int64_t nnz = 0;
    double m = 0.0;
    PLV_CUDA(cudaMemcpyAsync(st, stats.get(), sizeof(st), cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaMemcpyAsync(&nnz, off + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaMemcpyAsync(&m, msum.get() + 1, sizeof(double), cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    int64_t num_self = (int64_t)st[0];
    info_h[0] = nnz;
    info_h[1] = merged;
    info_h[2] = (nnz + num_self) / 2;
    info_h[3] = (int64_t)st[1];
    info_h[4] = (st[2] == 0 && 2.0 * m < 4503599627370496.0) ? 1 : 0;
    info_h[5] = num_self;
    *m_h = m;
}

__global__ void k_gather_i32(const int32_t *src, const int32_t *idx, int64_t n, int32_t *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = src[idx[i]];
}

__global__ void k_iota_i32(int32_t *p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (int32_t)i;
}

void iota_i32(int32_t *p, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    k_iota_i32<<<grid_for(n, 256), 256, 0, s>>>(p, n);
    PLV_LAUNCH_CHECK();
}

void gather_i32(const int32_t *src, const int32_t *idx, int64_t n, int32_t *out,
                       cudaStream_t s) {
    if (n <= 0) return;
    k_gather_i32<<<grid_for(n, 256), 256, 0, s>>>(src, idx, n, out);
    PLV_LAUNCH_CHECK();
}

void csr_build(const int32_t *u, const int32_t *v, const double *w, int64_t R, int64_t n,
               int64_t *off, int32_t *nbr, double *wts, double *selfw, double *k,
               int64_t *info_h, double *m_h, cudaStream_t s) {
    if (R < 0 || n < 0) PLV_FAIL(PLV_EINVAL, "negative size");
    if (R >= (1ll << 31) - 1 || n >= (1ll << 31) - 1)
        PLV_FAIL(PLV_EINVAL, "plv_csr_build: more than 2^31 records or vertices");
    if (R > 0) {
        Buf<int> flags(1, s);
        PLV_CUDA(cudaMemsetAsync(flags.get(), 0, sizeof(int), s));
        k_validate<<<grid_for(R, 256), 256, 0, s>>>(u, v, w, R, n, flags);
        PLV_LAUNCH_CHECK();
        int f = d2h(flags.get(), s);
        if (f & 1) PLV_FAIL(PLV_EWEIGHT, "non-positive weight in edge records");
        if (f & 2) PLV_FAIL(PLV_ERANGE, "vertex id out of range");
    }
    int nb = bits_for(n > 1 ? n : 2);
    Buf<uint64_t> key(R + 1, s), key_s(R + 1, s);
    Buf<double> w_s(R + 1, s);
    Buf<uint8_t> head(R + 1, s);
    Buf<int64_t> starts(R + 1, s);
    int64_t M = 0;
    if (R > 0) {
        k_canon_keys<<<grid_for(R, 256), 256, 0, s>>>(u, v, R, nb, key);
        PLV_LAUNCH_CHECK();
        sort_pairs<uint64_t, double>(key, key_s, w, w_s, R, 0, 2 * nb, s);
        k_key_heads<<<grid_for(R, 256), 256, 0, s>>>(key_s, R, head);
        PLV_LAUNCH_CHECK();
        M = select_flagged_index(head, R, starts, s);
    }
    Buf<int32_t> am(M + 1, s), bm(M + 1, s);
    Buf<double> wm(M + 1, s);
    if (M > 0) {
        k_decode_runs<<<grid_for(M, 256), 256, 0, s>>>(key_s, starts, M, nb, am, bm);
        PLV_LAUNCH_CHECK();
        reduceat_async(w_s, starts, M, R, wm, s);
    }
    key.release();
    key_s.release();
    csr_from_merged(am, bm, wm, M, n, R - M, off, nbr, wts, selfw, k, info_h, m_h, s);
}

}  // namespace plv

extern "C" int plv_csr_build(const int32_t *u, const int32_t *v, const double *w, int64_t R,
                             int64_t n, int64_t *off, int32_t *nbr, double *wts, double *selfw,
                             double *k, int64_t *info_h, double *m_h, void *stream) {
    PLV_ENTRY
    plv::csr_build(u, v, w, R, n, off, nbr, wts, selfw, k, info_h, m_h, plv::S(stream));
    PLV_EXIT
}

extern "C" int plv_csr_from_sorted(const int32_t *a, const int32_t *b, const double *w, int64_t M,
                                   int64_t n, int64_t *off, int32_t *nbr, double *wts,
                                   double *selfw, double *k, int64_t *info_h, double *m_h,
                                   void *stream) {
    PLV_ENTRY
    plv::csr_from_merged(a, b, w, M, n, 0, off, nbr, wts, selfw, k, info_h, m_h, plv::S(stream));
    PLV_EXIT
}

namespace plv {
__global__ void k_rec_flags(const int64_t *off, const int32_t *nbr, const int32_t *rowidx,
                            int64_t nnz, uint8_t *flag) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x)
        flag[e] = nbr[e] >= rowidx[e];
}
__global__ void k_rec_emit(const int64_t *sel, int64_t cnt, const int32_t *nbr,
                           const double *wts, const int32_t *rowidx, int32_t *ra, int32_t *rb,
                           double *rw) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t e = sel[t];
        ra[t] = rowidx[e];
        rb[t] = nbr[e];
        rw[t] = wts[e];
    }
}

int64_t edge_records(const int64_t *off, const int32_t *nbr, const double *wts, int64_t n,
                     int32_t *ra, int32_t *rb, double *rw, cudaStream_t s) {
    int64_t nnz = n > 0 ? d2h(off + n, s) : 0;
    if (nnz == 0) return 0;
    Buf<int32_t> rowidx(nnz, s);
    row_index(off, n, nnz, rowidx, s);
    Buf<uint8_t> flag(nnz, s);
    k_rec_flags<<<grid_for(nnz, 256), 256, 0, s>>>(off, nbr, rowidx, nnz, flag);
    PLV_LAUNCH_CHECK();
    Buf<int64_t> sel(nnz, s);
    int64_t cnt = select_flagged_index(flag, nnz, sel, s);
    if (cnt > 0) {
        k_rec_emit<<<grid_for(cnt, 256), 256, 0, s>>>(sel, cnt, nbr, wts, rowidx, ra, rb, rw);
        PLV_LAUNCH_CHECK();
    }
    return cnt;
}
}  // namespace plv

extern "C" int plv_edge_records(const int64_t *off, const int32_t *nbr, const double *wts,
                                int64_t n, int32_t *ra, int32_t *rb, double *rw, int64_t *count_h,
                                void *stream) {
    PLV_ENTRY
    *count_h = plv::edge_records(off, nbr, wts, n, ra, rb, rw, plv::S(stream));
    PLV_EXIT
}
