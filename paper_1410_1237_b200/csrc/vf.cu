// vf.cu -- vertex following (PL/heuristics.py:46-89) on device.
//
// candidate = one adjacency entry and no self loop; its only neighbour is
// nbr[off[i]].  An isolated candidate pair keeps the lower id.  new_id is the
// exclusive count of surviving vertices; folded vertices map to their
// neighbour's new id.  Records: the kept edge_records (row-major, a <= b,
// both endpoints surviving) followed by one self-loop record (t, t, w) per
// folded vertex in ascending id -- the exact input order of the reference's
// Graph.from_edges call, so its stable sort / reduceat see the same sequence.
#include "common.cuh"
#include "csr.cuh"
#include <cub/cub.cuh>

namespace plv {

__global__ void k_vf_cand(const int64_t *off, const int32_t *nbr, const double *selfw, int64_t n,
                          int32_t *only) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        bool cand = (off[i + 1] - off[i] == 1) && (selfw[i] == 0.0);
        only[i] = cand ? nbr[off[i]] : -1;
    }
}

__global__ void k_vf_merged(const int32_t *only, int64_t n, uint8_t *merged, int32_t *keep_cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t o = only[i];
        bool m = o >= 0;
        if (m && only[o] >= 0 && i < o) m = false;  // isolated pair: lower id survives
        merged[i] = m;
        keep_cnt[i] = !m;
    }
}

__global__ void k_vf_map(const int32_t *only, const uint8_t *merged, const int64_t *new_id,
                         int64_t n, int32_t *vmap) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        vmap[i] = (int32_t)(merged[i] ? new_id[only[i]] : new_id[i]);
}

__global__ void k_vf_rec_flags(const int32_t *nbr, const int32_t *rowidx, const uint8_t *merged,
                               int64_t nnz, uint8_t *flag) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x) {
        int32_t i = rowidx[e], j = nbr[e];
        flag[e] = (j >= i) && !merged[i] && !merged[j];
    }
}

__global__ void k_vf_emit_kept(const int64_t *sel, int64_t cnt, const int32_t *nbr,
                               const double *wts, const int32_t *rowidx, const int64_t *new_id,
                               int32_t *ru, int32_t *rv, double *rw) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t e = sel[t];
        ru[t] = (int32_t)new_id[rowidx[e]];
        rv[t] = (int32_t)new_id[nbr[e]];
        rw[t] = wts[e];
    }
}

__global__ void k_vf_emit_folded(const int64_t *mids, int64_t nm, const int64_t *off,
                                 const double *wts, const int32_t *only, const int64_t *new_id,
                                 int32_t *ru, int32_t *rv, double *rw) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nm;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = mids[t];
        int32_t tg = (int32_t)new_id[only[i]];
        ru[t] = tg;
        rv[t] = tg;
        rw[t] = wts[off[i]];
    }
}

void vf_records(const int64_t *off, const int32_t *nbr, const double *wts, const double *selfw,
                int64_t n, int32_t *vmap, int32_t *ru, int32_t *rv, double *rw, int64_t *info_h,
                cudaStream_t s) {
    if (n <= 0) {
        info_h[0] = info_h[1] = info_h[2] = 0;
        return;
    }
    int64_t nnz = d2h(off + n, s);
    Buf<int32_t> only(n, s), keepc(n, s);
    Buf<uint8_t> merged(n, s);
    Buf<int64_t> new_id(n + 1, s);
    k_vf_cand<<<grid_for(n, 256), 256, 0, s>>>(off, nbr, selfw, n, only);
    PLV_LAUNCH_CHECK();
    k_vf_merged<<<grid_for(n, 256), 256, 0, s>>>(only, n, merged, keepc);
    PLV_LAUNCH_CHECK();
    offsets_from_degrees(keepc, n, new_id, s);  // exclusive count of survivors
    k_vf_map<<<grid_for(n, 256), 256, 0, s>>>(only, merged, new_id, n, vmap);
    PLV_LAUNCH_CHECK();
    int64_t kept = 0;
    if (nnz > 0) {
        Buf<int32_t> rowidx(nnz, s);
        row_index(off, n, nnz, rowidx, s);
        Buf<uint8_t> flag(nnz, s);
        k_vf_rec_flags<<<grid_for(nnz, 256), 256, 0, s>>>(nbr, rowidx, merged, nnz, flag);
        PLV_LAUNCH_CHECK();
        Buf<int64_t> sel(nnz, s);
        kept = select_flagged_index(flag, nnz, sel, s);
        if (kept > 0) {
            k_vf_emit_kept<<<grid_for(kept, 256), 256, 0, s>>>(sel, kept, nbr, wts, rowidx, new_id,
                                                              ru, rv, rw);
            PLV_LAUNCH_CHECK();
        }
    }
    Buf<int64_t> mids(n, s);
    int64_t nm = select_flagged_index(merged, n, mids, s);
    if (nm > 0) {
        k_vf_emit_folded<<<grid_for(nm, 256), 256, 0, s>>>(mids, nm, off, wts, only, new_id,
                                                          ru + kept, rv + kept, rw + kept);
        PLV_LAUNCH_CHECK();
    }
    info_h[0] = n - nm;
    info_h[1] = nm;
    info_h[2] = kept + nm;
}

}  // namespace plv

extern "C" int plv_vf_records(const int64_t *off, const int32_t *nbr, const double *wts,
                              const double *selfw, int64_t n, int32_t *vertex_map, int32_t *rec_u,
                              int32_t *rec_v, double *rec_w, int64_t *info_h, void *stream) {
    PLV_ENTRY
    plv::vf_records(off, nbr, wts, selfw, n, vertex_map, rec_u, rec_v, rec_w, info_h,
                    plv::S(stream));
    PLV_EXIT
}
