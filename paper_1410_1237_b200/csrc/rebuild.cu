// rebuild.cu -- graph coarsening (PL/engine.py:229-256) on device.
//
// renumber: community ids present in the assignment, densely ranked in
// ascending id (np.unique), by a flag + exclusive scan.  Records: the a <= b
// half of the CSR in row-major order (Graph.edge_records) mapped to
// (lo, hi) = (min, max) of the renumbered communities, stable radix sort on
// the (lo << nb | hi) key (np.lexsort keeps row-major order among equal keys),
// runs merged with numpy's reduceat rule.  The merged list is sorted and
// unique, so Graph.from_edges on it reduces to plv_csr_from_sorted.
#include "common.cuh"
#include "csr.cuh"
#include "pairwise.cuh"

namespace plv {

__global__ void k_mark_present(const int32_t *assign, int64_t n, int32_t *present) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        present[assign[i]] = 1;
}

__global__ void k_renumber(const int32_t *present, const int64_t *rank, int64_t n, int32_t *ren) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
         c += (int64_t)gridDim.x * blockDim.x)
        ren[c] = present[c] ? (int32_t)rank[c] : -1;
}

__global__ void k_coarse_keys(const int64_t *sel, int64_t cnt, const int32_t *nbr,
                              const double *wts, const int32_t *rowidx, const int32_t *assign,
                              const int32_t *ren, int nb, uint64_t *key, double *w) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t e = sel[t];
        int32_t ca = ren[assign[rowidx[e]]], cb = ren[assign[nbr[e]]];
        uint32_t lo = (uint32_t)min(ca, cb), hi = (uint32_t)max(ca, cb);
        key[t] = ((uint64_t)lo << nb) | hi;
        w[t] = wts[e];
    }
}

__global__ void k_key_heads2(const uint64_t *key, int64_t R, uint8_t *head) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
         r += (int64_t)gridDim.x * blockDim.x)
        head[r] = (r == 0 || key[r] != key[r - 1]) ? 1 : 0;
}

__global__ void k_decode_runs2(const uint64_t *key, const int64_t *starts, int64_t M, int nb,
                               int32_t *am, int32_t *bm) {
    uint64_t mask = (1ull << nb) - 1ull;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M;
         t += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = key[starts[t]];
        am[t] = (int32_t)(k >> nb);
        bm[t] = (int32_t)(k & mask);
    }
}

__global__ void k_rec_flags2(const int32_t *nbr, const int32_t *rowidx, int64_t nnz, uint8_t *flag) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x)
        flag[e] = nbr[e] >= rowidx[e];
}

void rebuild_records(const int64_t *off, const int32_t *nbr, const double *wts, int64_t n,
                     const int32_t *assign, int32_t *ren, int32_t *lo, int32_t *hi, double *w,
                     int64_t *info_h, cudaStream_t s) {
    if (n <= 0) {
        info_h[0] = info_h[1] = 0;
        return;
    }
    Buf<int32_t> present(n, s);
    Buf<int64_t> rank(n + 1, s);
    PLV_CUDA(cudaMemsetAsync(present.get(), 0, sizeof(int32_t) * n, s));
    k_mark_present<<<grid_for(n, 256), 256, 0, s>>>(assign, n, present);
    PLV_LAUNCH_CHECK();
    offsets_from_degrees(present, n, rank, s);
    k_renumber<<<grid_for(n, 256), 256, 0, s>>>(present, rank, n, ren);
    PLV_LAUNCH_CHECK();
    int64_t nc = d2h(rank.get() + n, s);
    int64_t nnz = d2h(off + n, s);
    int64_t M = 0;
    if (nnz > 0) {
        Buf<int32_t> rowidx(nnz, s);
        row_index(off, n, nnz, rowidx, s);
        Buf<uint8_t> flag(nnz, s);
        k_rec_flags2<<<grid_for(nnz, 256), 256, 0, s>>>(nbr, rowidx, nnz, flag);
        PLV_LAUNCH_CHECK();
        Buf<int64_t> sel(nnz, s);
        int64_t R = select_flagged_index(flag, nnz, sel, s);
        flag.release();
        int nb = bits_for(nc > 1 ? nc : 2);
        Buf<uint64_t> key(R, s), key_s(R, s);
        Buf<double> wr(R, s), w_s(R, s);
        k_coarse_keys<<<grid_for(R, 256), 256, 0, s>>>(sel, R, nbr, wts, rowidx, assign, ren, nb,
                                                      key, wr);
        PLV_LAUNCH_CHECK();
        sel.release();
        rowidx.release();
        sort_pairs<uint64_t, double>(key, key_s, wr, w_s, R, 0, 2 * nb, s);
        key.release();
        wr.release();
        Buf<uint8_t> head(R, s);
        k_key_heads2<<<grid_for(R, 256), 256, 0, s>>>(key_s, R, head);
        PLV_LAUNCH_CHECK();
        Buf<int64_t> starts(R, s);
        M = select_flagged_index(head, R, starts, s);
        k_decode_runs2<<<grid_for(M, 256), 256, 0, s>>>(key_s, starts, M, nb, lo, hi);
        PLV_LAUNCH_CHECK();
        reduceat_async(w_s, starts, M, R, w, s);
    }
    info_h[0] = nc;
    info_h[1] = M;
}

__global__ void k_compose(const int32_t *map, const int32_t *assign, const int32_t *ren, int64_t n,
                          int32_t *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t v = map ? map[i] : (int32_t)i;
        out[i] = ren[assign[v]];
    }
}

}  // namespace plv

extern "C" int plv_rebuild_records(const int64_t *off, const int32_t *nbr, const double *wts,
                                   int64_t n, const int32_t *assign, int32_t *renumber,
                                   int32_t *lo, int32_t *hi, double *w, int64_t *info_h,
                                   void *stream) {
    PLV_ENTRY
    plv::rebuild_records(off, nbr, wts, n, assign, renumber, lo, hi, w, info_h, plv::S(stream));
    PLV_EXIT
}

extern "C" int plv_compose(const int32_t *map, const int32_t *assign, const int32_t *renumber,
                           int64_t n, int32_t *out, void *stream) {
    PLV_ENTRY
    if (n > 0) {
        plv::k_compose<<<plv::grid_for(n, 256), 256, 0, plv::S(stream)>>>(map, assign, renumber, n,
                                                                         out);
        PLV_LAUNCH_CHECK();
    }
    PLV_EXIT
}
