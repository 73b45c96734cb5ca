// part.cu -- the 1D vertex partition of the multi-GPU path.
//
// Rank r of W owns vertices [bounds[r], bounds[r+1]) and holds ONLY their
// rows; the per-vertex state (assignment, a_tot, w_internal, sizes) and the
// per-vertex graph scalars (k, self-loop weight, degree) are replicated.
// These kernels are the per-rank pieces of Graph.from_edges, vf_compact,
// color_graph and rebuild on such a partition; the exchanges between them
// (all-to-all of records, all-reduce of the replicated vectors, all-gather of
// decided slices) are made by the host driver (paper_1410_1237_b200/partition.py)
// over NCCL, or gloo in the tests.  The reference has no distributed mode;
// every result is the single-graph result bit for bit:
//
//  * construction: a record goes to the owner of each endpoint (one or two
//    ranks), senders in rank order and each sender's records in generation
//    order, so every rank's record list is the global list restricted to the
//    records that touch its rows, in global order.  The ordinary CSR build on
//    that list (stable sort, reduceat merge: PL/graph.py:112-139) then yields
//    every owned row exactly as the whole-graph build does; the other rows
//    are dropped (plv_part_own_rows).
//  * k, self loops and degrees of owned rows are exact per rank; an all-reduce
//    of the zero-padded vectors replicates them (x + 0 = x), and m is the
//    pairwise sum of the replicated k, as on one GPU.
#include "common.cuh"
#include "csr.cuh"
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

namespace plv {

__device__ __forceinline__ int owner_of(const int64_t *bounds, int W, int64_t v) {
    int lo = 0, hi = W;  // largest r with bounds[r] <= v
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (bounds[mid] <= v)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

// ------------------------------------------------------------ generation

struct RmatR {
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

__global__ void k_rmat_emit_r(RmatR g, const int64_t *sel, int64_t cnt, int32_t *u, int32_t *v,
                              double *w) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = sel[t];
        g.edge(r, u[t], v[t]);
        w[t] = dadd(g.w_lo, dmul(g.span, rnd01(g.kw, (uint64_t)r)));
    }
}

// ------------------------------------------------------------ routing

// Destinations of record t: owner(min) always, owner(max) when different.
__global__ void k_route_count(const int32_t *u, const int32_t *v, int64_t R,
                              const int64_t *bounds, int W, uint32_t *dkey, int32_t *didx,
                              unsigned long long *hist) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < R;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t a = min(u[t], v[t]), b = max(u[t], v[t]);
        const int da = owner_of(bounds, W, a), db = owner_of(bounds, W, b);
        dkey[2 * t] = (uint32_t)da;
        didx[2 * t] = (int32_t)t;
        dkey[2 * t + 1] = db != da ? (uint32_t)db : (uint32_t)W;  // W: no second copy
        didx[2 * t + 1] = (int32_t)t;
        atomicAdd(hist + da, 1ull);
        if (db != da) atomicAdd(hist + db, 1ull);
    }
}

__global__ void k_route_gather(const int32_t *u, const int32_t *v, const double *w,
                               const int32_t *sidx, int64_t cnt, int32_t *ou, int32_t *ov,
                               double *ow) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = sidx[t];
        ou[t] = u[r];
        ov[t] = v[r];
        ow[t] = w[r];
    }
}

// ------------------------------------------------------------ owned rows

__global__ void k_own_off(const int64_t *off, int64_t n, int64_t lo, int64_t hi, int64_t *out) {
    const int64_t base = off[lo], top = off[hi];
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= n;
         v += (int64_t)gridDim.x * blockDim.x)
        out[v] = v <= lo ? 0 : v >= hi ? top - base : off[v] - base;
}

// info: [0] self loops, [1] unique pairs (entries with nbr >= row),
// [2] max degree, [3] 1 if some weight is not an integer
__global__ void k_own_stats(const int64_t *off, const int32_t *nbr, const double *wts,
                            int64_t lo, int64_t hi, unsigned long long *info) {
    unsigned long long self = 0, pairs = 0, mx = 0, frac = 0;
    for (int64_t v = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < hi;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e0 = off[v], e1 = off[v + 1];
        mx = (unsigned long long)(e1 - e0) > mx ? (unsigned long long)(e1 - e0) : mx;
        for (int64_t e = e0; e < e1; e++) {
            const int32_t j = nbr[e];
            self += j == v;
            pairs += j >= v;
            frac |= wts[e] != floor(wts[e]) || wts[e] >= 4503599627370496.0;
        }
    }
    atomicAdd(info, self);
    atomicAdd(info + 1, pairs);
    atomicMax(info + 2, mx);
    if (frac) atomicOr(info + 3, 1ull);
}

__global__ void k_degrees_own(const int64_t *off, int64_t lo, int64_t hi, int32_t *deg) {
    for (int64_t v = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < hi;
         v += (int64_t)gridDim.x * blockDim.x)
        deg[v] = (int32_t)(off[v + 1] - off[v]);
}

// ------------------------------------------------------- vertex following

// only_p1[v] = the single neighbour + 1 of every owned VF candidate
// (PL/heuristics.py:56-60), 0 elsewhere (all-reduced by the host).
__global__ void k_vf_only(const int64_t *off, const int32_t *nbr, const int32_t *deg,
                          const double *selfw, int64_t lo, int64_t hi, int32_t *only_p1) {
    for (int64_t v = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < hi;
         v += (int64_t)gridDim.x * blockDim.x)
        only_p1[v] = (deg[v] == 1 && selfw[v] == 0.0) ? nbr[off[v]] + 1 : 0;
}

// merged flags (PL/heuristics.py:61-66) from the replicated candidate data
__global__ void k_vf_merged_p(const int32_t *only_p1, int64_t n, uint8_t *merged, int32_t *keep) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        bool m = false;
        const int32_t p = only_p1[v] - 1;
        if (p >= 0) {  // a candidate
            const bool paired = only_p1[p] > 0;
            m = !(paired && v < p);  // the lower id of an isolated pair survives
        }
        merged[v] = m;
        keep[v] = !m;
    }
}

__global__ void k_vf_map_p(const uint8_t *merged, const int32_t *new_id, const int32_t *only_p1,
                           int64_t n, int32_t *vmap) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x)
        vmap[v] = merged[v] ? new_id[only_p1[v] - 1] : new_id[v];
}

// records of the owned rows: kept edge_records (a <= b, neither merged) in
// row-major order, and folded (t, t, w) records of owned merged vertices
__global__ void k_vf_kept_flags(const int64_t *off, const int32_t *nbr, int64_t lo, int64_t hi,
                                const uint8_t *merged, uint8_t *flag) {
    for (int64_t v = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < hi;
         v += (int64_t)gridDim.x * blockDim.x)
        for (int64_t e = off[v]; e < off[v + 1]; e++) {
            const int32_t j = nbr[e];
            flag[e] = j >= v && !merged[v] && !merged[j];
        }
}

__global__ void k_row_of(const int64_t *off, int64_t lo, int64_t hi, int32_t *row) {
    for (int64_t v = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < hi;
         v += (int64_t)gridDim.x * blockDim.x)
        for (int64_t e = off[v]; e < off[v + 1]; e++) row[e] = (int32_t)v;
}

__global__ void k_emit_pairs(const int64_t *sel, int64_t cnt, const int32_t *row,
                             const int32_t *nbr, const double *wts, const int32_t *map_a,
                             const int32_t *map_b, int32_t *ou, int32_t *ov, double *ow) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = sel[t];
        const int32_t a = row[e], b = nbr[e];
        ou[t] = map_a[a];
        ov[t] = map_b[b];
        ow[t] = wts[e];
    }
}

__global__ void k_vf_fold_flags(int64_t lo, int64_t hi, const uint8_t *merged, uint8_t *flag) {
    for (int64_t v = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < hi;
         v += (int64_t)gridDim.x * blockDim.x)
        flag[v - lo] = merged[v];
}

__global__ void k_vf_fold_emit(const int64_t *sel, int64_t cnt, int64_t lo, const int64_t *off,
                               const double *wts, const int32_t *new_id, const int32_t *only_p1,
                               int32_t *ou, int32_t *ov, double *ow) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = lo + sel[t];
        const int32_t tg = new_id[only_p1[v] - 1];
        ou[t] = tg;
        ov[t] = tg;
        ow[t] = wts[off[v]];
    }
}

// ----------------------------------------------------------- colouring aid

__global__ void k_scatter_i32(const int32_t *idx, const int32_t *val, int32_t fill, int64_t cnt,
                              int32_t *out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x)
        out[idx[t]] = val ? val[t] : fill;
}

__global__ void k_keep_to_reject(const uint8_t *keep, int64_t n, uint8_t *rej) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x)
        rej[t] = !keep[t];
}

__global__ void k_gather_sel(const int32_t *src, const int64_t *sel, int64_t cnt, int32_t *out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x)
        out[t] = src[sel[t]];
}

// ------------------------------------------------------------- rebuild

__global__ void k_present(const int32_t *assign, int64_t n, int32_t *pres) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x)
        pres[assign[v]] = 1;
}

__global__ void k_renum(const int32_t *pres, const int32_t *scan, int64_t n, int32_t *ren) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x)
        ren[v] = pres[v] ? scan[v] : -1;
}

__global__ void k_compose_i32(const int32_t *a, const int32_t *b, int64_t n, int32_t *out) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x)
        out[v] = b[a[v]];
}

__global__ void k_rb_flags(const int64_t *off, const int32_t *nbr, int64_t lo, int64_t hi,
                           uint8_t *flag) {
    for (int64_t v = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < hi;
         v += (int64_t)gridDim.x * blockDim.x)
        for (int64_t e = off[v]; e < off[v + 1]; e++) flag[e] = nbr[e] >= v;
}

static int64_t select_flagged64(const uint8_t *flags, int64_t n, int64_t *out, cudaStream_t s) {
    return select_flagged_index(flags, n, out, s);
}

}  // namespace plv

using namespace plv;

extern "C" int plv_gen_rmat_range(uint64_t seed, int scale, int64_t edge_factor, double a,
                                  double b, double c, double w_lo, double w_hi, int64_t r_begin,
                                  int64_t r_end, int32_t *u, int32_t *v, double *w, int64_t cap,
                                  int64_t *count_h, void *stream) {
    PLV_ENTRY
    cudaStream_t s = S(stream);
    if (scale < 1 || scale > 30) PLV_FAIL(PLV_EINVAL, "rmat scale out of range");
    const int64_t R = edge_factor << scale;
    if (r_begin < 0 || r_end > R || r_end < r_begin) PLV_FAIL(PLV_EINVAL, "record range");
    RmatR g{stream_key(seed, 1), stream_key(seed, 2), scale, a, a + b, (a + b) + c, w_lo,
            w_hi - w_lo};
    const int64_t nr = r_end - r_begin;
    Buf<int64_t> sel(nr, s), cnt(1, s);
    thrust::counting_iterator<int64_t> it(r_begin);
    size_t bytes = 0;
    PLV_CUDA(cub::DeviceSelect::If(nullptr, bytes, it, sel.get(), cnt.get(), nr, g, s));
    Buf<char> tmp(bytes, s);
    if (nr) PLV_CUDA(cub::DeviceSelect::If(tmp.get(), bytes, it, sel.get(), cnt.get(), nr, g, s));
    const int64_t k = nr ? d2h(cnt.get(), s) : 0;
    if (k > cap) PLV_FAIL(PLV_EINVAL, "rmat range: capacity %lld < %lld", (long long)cap, (long long)k);
    if (k) {
        k_rmat_emit_r<<<grid_for(k, 256), 256, 0, s>>>(g, sel, k, u, v, w);
        PLV_LAUNCH_CHECK();
    }
    *count_h = k;
    PLV_EXIT
}

extern "C" int plv_route_records(const int32_t *u, const int32_t *v, const double *w, int64_t R,
                                 const int64_t *bounds, int world, int32_t *ou, int32_t *ov,
                                 double *ow, int64_t cap, int64_t *send_counts_h, void *stream) {
    PLV_ENTRY
    cudaStream_t s = S(stream);
    if (world < 1 || world > 1024) PLV_FAIL(PLV_EINVAL, "world size");
    if (R >= (int64_t)1 << 31) PLV_FAIL(PLV_EINVAL, "route: at most 2^31 - 1 records per call");
    Buf<unsigned long long> hist(world + 1, s);
    PLV_CUDA(cudaMemsetAsync(hist.get(), 0, sizeof(unsigned long long) * (world + 1), s));
    std::vector<unsigned long long> h(world + 1, 0);
    if (R) {
        Buf<uint32_t> key(2 * R, s), skey(2 * R, s);
        Buf<int32_t> idx(2 * R, s), sidx(2 * R, s);
        k_route_count<<<grid_for(R, 256), 256, 0, s>>>(u, v, R, bounds, world, key, idx, hist);
        PLV_LAUNCH_CHECK();
        PLV_CUDA(cudaMemcpyAsync(h.data(), hist.get(), sizeof(unsigned long long) * (world + 1),
                                 cudaMemcpyDeviceToHost, s));
        // stable by destination: each destination's records in input order
        sort_pairs<uint32_t, int32_t>(key, skey, idx, sidx, 2 * R, 0, bits_for(world + 2), s);
        PLV_CUDA(cudaStreamSynchronize(s));
        int64_t tot = 0;
        for (int r = 0; r < world; r++) tot += (int64_t)h[r];
        if (tot > cap) PLV_FAIL(PLV_EINVAL, "route: capacity %lld < %lld", (long long)cap, (long long)tot);
        if (tot) {
            k_route_gather<<<grid_for(tot, 256), 256, 0, s>>>(u, v, w, sidx, tot, ou, ov, ow);
            PLV_LAUNCH_CHECK();
        }
    }
    for (int r = 0; r < world; r++) send_counts_h[r] = (int64_t)h[r];
    PLV_EXIT
}

extern "C" int plv_part_own_rows(const int64_t *off, const int32_t *nbr, const double *wts,
                                 int64_t n, int64_t lo, int64_t hi, int64_t *out_off,
                                 int32_t *out_nbr, double *out_wts, int32_t *deg,
                                 int64_t *info_h, void *stream) {
    PLV_ENTRY
    cudaStream_t s = S(stream);
    if (lo < 0 || hi > n || hi < lo) PLV_FAIL(PLV_EINVAL, "owned range");
    int64_t e[2];
    PLV_CUDA(cudaMemcpyAsync(e, off + lo, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaMemcpyAsync(e + 1, off + hi, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    const int64_t cnt = e[1] - e[0];
    if (cnt) {
        PLV_CUDA(cudaMemcpyAsync(out_nbr, nbr + e[0], sizeof(int32_t) * cnt,
                                 cudaMemcpyDeviceToDevice, s));
        PLV_CUDA(cudaMemcpyAsync(out_wts, wts + e[0], sizeof(double) * cnt,
                                 cudaMemcpyDeviceToDevice, s));
    }
    k_own_off<<<grid_for(n + 1, 256), 256, 0, s>>>(off, n, lo, hi, out_off);
    PLV_LAUNCH_CHECK();
    Buf<unsigned long long> info(4, s);
    PLV_CUDA(cudaMemsetAsync(info.get(), 0, sizeof(unsigned long long) * 4, s));
    PLV_CUDA(cudaMemsetAsync(deg, 0, sizeof(int32_t) * n, s));
    if (hi > lo) {
        k_own_stats<<<grid_for(hi - lo, 256), 256, 0, s>>>(out_off, out_nbr, out_wts, lo, hi, info);
        PLV_LAUNCH_CHECK();
        k_degrees_own<<<grid_for(hi - lo, 256), 256, 0, s>>>(out_off, lo, hi, deg);
        PLV_LAUNCH_CHECK();
    }
    unsigned long long hi4[4];
    PLV_CUDA(cudaMemcpyAsync(hi4, info.get(), sizeof(hi4), cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    info_h[0] = cnt;
    for (int t = 0; t < 4; t++) info_h[1 + t] = (int64_t)hi4[t];
    PLV_EXIT
}

extern "C" int plv_part_vf_only(const int64_t *off, const int32_t *nbr, const int32_t *deg,
                                const double *selfw, int64_t n, int64_t lo, int64_t hi,
                                int32_t *only_p1, void *stream) {
    PLV_ENTRY
    cudaStream_t s = S(stream);
    PLV_CUDA(cudaMemsetAsync(only_p1, 0, sizeof(int32_t) * n, s));
    if (hi > lo) {
        k_vf_only<<<grid_for(hi - lo, 256), 256, 0, s>>>(off, nbr, deg, selfw, lo, hi, only_p1);
        PLV_LAUNCH_CHECK();
    }
    PLV_EXIT
}

extern "C" int plv_part_vf_map(const int32_t *only_p1, int64_t n, uint8_t *merged,
                               int32_t *new_id, int32_t *vertex_map, int64_t *info_h,
                               void *stream) {
    PLV_ENTRY
    cudaStream_t s = S(stream);
    Buf<int32_t> keep(n + 1, s);
    if (n) {
        k_vf_merged_p<<<grid_for(n, 256), 256, 0, s>>>(only_p1, n, merged, keep);
        PLV_LAUNCH_CHECK();
    }
    PLV_CUDA(cudaMemsetAsync(keep.get() + n, 0, sizeof(int32_t), s));
    size_t bytes = 0;
    PLV_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, keep.get(), new_id, n + 1, s));
    Buf<char> tmp(bytes, s);
    PLV_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, keep.get(), new_id, n + 1, s));
    if (n) {
        k_vf_map_p<<<grid_for(n, 256), 256, 0, s>>>(merged, new_id, only_p1, n, vertex_map);
        PLV_LAUNCH_CHECK();
    }
    int32_t nn = 0;
    PLV_CUDA(cudaMemcpyAsync(&nn, new_id + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    info_h[0] = nn;
    info_h[1] = n - nn;
    PLV_EXIT
}

extern "C" int plv_part_vf_records(const int64_t *off, const int32_t *nbr, const double *wts,
                                   int64_t n, int64_t lo, int64_t hi, const uint8_t *merged,
                                   const int32_t *new_id, const int32_t *only_p1, int32_t *ku,
                                   int32_t *kv, double *kw, int32_t *fu, int32_t *fv, double *fw,
                                   int64_t *counts_h, void *stream) {
    PLV_ENTRY
    cudaStream_t s = S(stream);
    int64_t e[2];
    PLV_CUDA(cudaMemcpyAsync(e, off + lo, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaMemcpyAsync(e + 1, off + hi, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    const int64_t nnz = e[1];  // owned rows start at entry 0
    counts_h[0] = counts_h[1] = 0;
    if (nnz) {
        Buf<uint8_t> flag(nnz, s);
        Buf<int32_t> row(nnz, s);
        Buf<int64_t> sel(nnz, s);
        k_vf_kept_flags<<<grid_for(hi - lo, 256), 256, 0, s>>>(off, nbr, lo, hi, merged, flag);
        PLV_LAUNCH_CHECK();
        k_row_of<<<grid_for(hi - lo, 256), 256, 0, s>>>(off, lo, hi, row);
        PLV_LAUNCH_CHECK();
        const int64_t k = select_flagged64(flag, nnz, sel, s);
        if (k) {
            k_emit_pairs<<<grid_for(k, 256), 256, 0, s>>>(sel, k, row, nbr, wts, new_id, new_id, ku,
                                                          kv, kw);
            PLV_LAUNCH_CHECK();
        }
        counts_h[0] = k;
    }
    if (hi > lo) {
        Buf<uint8_t> flag(hi - lo, s);
        Buf<int64_t> sel(hi - lo, s);
        k_vf_fold_flags<<<grid_for(hi - lo, 256), 256, 0, s>>>(lo, hi, merged, flag);
        PLV_LAUNCH_CHECK();
        const int64_t k = select_flagged64(flag, hi - lo, sel, s);
        if (k) {
            k_vf_fold_emit<<<grid_for(k, 256), 256, 0, s>>>(sel, k, lo, off, wts, new_id, only_p1,
                                                            fu, fv, fw);
            PLV_LAUNCH_CHECK();
        }
        counts_h[1] = k;
    }
    PLV_EXIT
}

extern "C" int plv_scatter_i32(const int32_t *idx, const int32_t *val, int32_t fill, int64_t cnt,
                               int32_t *out, void *stream) {
    PLV_ENTRY
    cudaStream_t s = S(stream);
    if (cnt) {
        k_scatter_i32<<<grid_for(cnt, 256), 256, 0, s>>>(idx, val, fill, cnt, out);
        PLV_LAUNCH_CHECK();
    }
    PLV_EXIT
}

extern "C" int plv_select_rejected(const int32_t *active, const uint8_t *keep, int64_t na,
                                   int32_t *out, int64_t *count_h, void *stream) {
    PLV_ENTRY
    cudaStream_t s = S(stream);
    *count_h = 0;
    if (na) {
        Buf<uint8_t> rej(na, s);
        Buf<int64_t> sel(na, s);
        k_keep_to_reject<<<grid_for(na, 256), 256, 0, s>>>(keep, na, rej);
        PLV_LAUNCH_CHECK();
        const int64_t k = select_flagged64(rej, na, sel, s);
        if (k) {
            k_gather_sel<<<grid_for(k, 256), 256, 0, s>>>(active, sel, k, out);
            PLV_LAUNCH_CHECK();
        }
        *count_h = k;
    }
    PLV_EXIT
}

extern "C" int plv_renumber(const int32_t *assign, int64_t n, int32_t *renumber, int64_t *n_new_h,
                            void *stream) {
    PLV_ENTRY
    cudaStream_t s = S(stream);
    Buf<int32_t> pres(n + 1, s), scan(n + 1, s);
    PLV_CUDA(cudaMemsetAsync(pres.get(), 0, sizeof(int32_t) * (n + 1), s));
    if (n) {
        k_present<<<grid_for(n, 256), 256, 0, s>>>(assign, n, pres);
        PLV_LAUNCH_CHECK();
    }
    size_t bytes = 0;
    PLV_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, pres.get(), scan.get(), n + 1, s));
    Buf<char> tmp(bytes, s);
    PLV_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, pres.get(), scan.get(), n + 1, s));
    if (n) {
        k_renum<<<grid_for(n, 256), 256, 0, s>>>(pres, scan, n, renumber);
        PLV_LAUNCH_CHECK();
    }
    int32_t nn = 0;
    PLV_CUDA(cudaMemcpyAsync(&nn, scan.get() + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    *n_new_h = nn;
    PLV_EXIT
}

extern "C" int plv_part_rebuild_records(const int64_t *off, const int32_t *nbr, const double *wts,
                                        int64_t n, int64_t lo, int64_t hi, const int32_t *assign,
                                        const int32_t *renumber, int32_t *ou, int32_t *ov,
                                        double *ow, int64_t *count_h, void *stream) {
    PLV_ENTRY
    cudaStream_t s = S(stream);
    int64_t e1 = 0;
    PLV_CUDA(cudaMemcpyAsync(&e1, off + hi, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    *count_h = 0;
    if (e1) {
        Buf<uint8_t> flag(e1, s);
        Buf<int32_t> row(e1, s), comm(n, s);
        Buf<int64_t> sel(e1, s);
        k_rb_flags<<<grid_for(hi - lo, 256), 256, 0, s>>>(off, nbr, lo, hi, flag);
        PLV_LAUNCH_CHECK();
        k_row_of<<<grid_for(hi - lo, 256), 256, 0, s>>>(off, lo, hi, row);
        PLV_LAUNCH_CHECK();
        k_compose_i32<<<grid_for(n, 256), 256, 0, s>>>(assign, renumber, n, comm);
        PLV_LAUNCH_CHECK();
        const int64_t k = select_flagged64(flag, e1, sel, s);
        if (k) {
            k_emit_pairs<<<grid_for(k, 256), 256, 0, s>>>(sel, k, row, nbr, wts, comm, comm, ou, ov,
                                                          ow);
            PLV_LAUNCH_CHECK();
        }
        *count_h = k;
    }
    PLV_EXIT
}
