// color.cu -- speculative distance-1 colouring (PL/heuristics.py:92-118).
//
// Round r: every active vertex takes the smallest colour not used by an
// already-committed neighbour (color_assign, PL/_kernels.pyx:148-174; active
// vertices carry -1 and impose nothing), the tentative colours are written,
// and a vertex keeps its colour unless a lower-id neighbour holds the same
// one (color_conflicts, PL/_kernels.pyx:177-195).  Rejected vertices are
// uncoloured and form the next active set in ascending order (stable
// compaction, PL/heuristics.py:113-115).
//
// First-fit uses a 64-bit "used" mask per window of 64 colours: thread per
// vertex for low degree, warp per vertex (OR-reduced masks) above 32.
#include "common.cuh"
#include "csr.cuh"
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

namespace plv {

constexpr unsigned FULLC = 0xffffffffu;
constexpr int COLOR_THREAD_MAXD = 32;

__device__ __forceinline__ int first_free_thread(const int64_t *off, const int32_t *nbr,
                                                 const int32_t *colors, int32_t i) {
    int64_t e0 = off[i], e1 = off[i + 1];
    for (int base = 0;; base += 64) {
        uint64_t used = 0;
        for (int64_t e = e0; e < e1; e++) {
            int32_t j = nbr[e];
            if (j == i) continue;
            int32_t cj = colors[j] - base;
            if (cj >= 0 && cj < 64) used |= 1ull << cj;
        }
        if (~used) return base + __ffsll((long long)~used) - 1;
    }
}

__device__ __forceinline__ int first_free_warp(const int64_t *off, const int32_t *nbr,
                                               const int32_t *colors, int32_t i, int lane) {
    int64_t e0 = off[i], e1 = off[i + 1];
    for (int base = 0;; base += 64) {
        uint64_t used = 0;
        for (int64_t e = e0 + lane; e < e1; e += 32) {
            int32_t j = nbr[e];
            if (j == i) continue;
            int32_t cj = colors[j] - base;
            if (cj >= 0 && cj < 64) used |= 1ull << cj;
        }
        unsigned lo = __reduce_or_sync(FULLC, (unsigned)used);
        unsigned hi = __reduce_or_sync(FULLC, (unsigned)(used >> 32));
        uint64_t all = ((uint64_t)hi << 32) | lo;
        if (~all) return base + __ffsll((long long)~all) - 1;
    }
}

// tentative colours for active[0..na) -> out[x]
__global__ void k_color_assign(const int64_t *off, const int32_t *nbr, const int32_t *active,
                               int64_t na, const int32_t *colors, int32_t *out) {
    int lane = threadIdx.x & 31;
    int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // low-degree vertices: one per thread, taken warp-slice by warp-slice
    for (int64_t base = gw * 32; base < na; base += nw * 32) {
        int64_t x = base + lane;
        bool mine = false;
        int32_t i = 0;
        if (x < na) {
            i = active[x];
            mine = (off[i + 1] - off[i]) <= COLOR_THREAD_MAXD;
            if (mine) out[x] = first_free_thread(off, nbr, colors, i);
        }
        unsigned big = __ballot_sync(FULLC, x < na && !mine);
        while (big) {
            int l = __ffs(big) - 1;
            big &= big - 1;
            int32_t ii = __shfl_sync(FULLC, i, l);
            int c = first_free_warp(off, nbr, colors, ii, lane);
            if (lane == 0) out[base + l] = c;
        }
    }
}

// keep[x] = no lower-id neighbour shares colors[active[x]]
__global__ void k_color_conflicts(const int64_t *off, const int32_t *nbr, const int32_t *active,
                                  int64_t na, const int32_t *colors, uint8_t *keep) {
    int lane = threadIdx.x & 31;
    int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = gw * 32; base < na; base += nw * 32) {
        int64_t x = base + lane;
        bool mine = false;
        int32_t i = 0;
        if (x < na) {
            i = active[x];
            int64_t e0 = off[i], e1 = off[i + 1];
            mine = (e1 - e0) <= COLOR_THREAD_MAXD;
            if (mine) {
                int32_t ci = colors[i];
                uint8_t k = 1;
                for (int64_t e = e0; e < e1; e++) {
                    int32_t j = nbr[e];
                    if (j < i && colors[j] == ci) {
                        k = 0;
                        break;
                    }
                }
                keep[x] = k;
            }
        }
        unsigned big = __ballot_sync(FULLC, x < na && !mine);
        while (big) {
            int l = __ffs(big) - 1;
            big &= big - 1;
            int32_t ii = __shfl_sync(FULLC, i, l);
            int32_t ci = colors[ii];
            int64_t e0 = off[ii], e1 = off[ii + 1];
            bool clash = false;
            // neighbour rows are sorted: only the prefix j < i matters
            for (int64_t e = e0 + lane; e < e1; e += 32) {
                int32_t j = nbr[e];
                if (j >= ii) break;
                if (colors[j] == ci) clash = true;
            }
            clash = __any_sync(FULLC, clash);
            if (lane == 0) keep[base + l] = clash ? 0 : 1;
        }
    }
}

__global__ void k_color_init(int32_t *colors, int32_t *active, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        colors[i] = -1;
        active[i] = (int32_t)i;
    }
}

__global__ void k_color_commit(const int32_t *active, int64_t na, const int32_t *tent,
                               int32_t *colors) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < na;
         x += (int64_t)gridDim.x * blockDim.x)
        colors[active[x]] = tent[x];
}

__global__ void k_reject_flags(const uint8_t *keep, int64_t na, uint8_t *rej) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < na;
         x += (int64_t)gridDim.x * blockDim.x)
        rej[x] = !keep[x];
}

__global__ void k_uncolor(const int32_t *rejected, int64_t nr, int32_t *colors) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < nr;
         x += (int64_t)gridDim.x * blockDim.x)
        colors[rejected[x]] = -1;
}

__global__ void k_max_color(const int32_t *colors, int64_t n, int *mx) {
    int m = -1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        m = colors[i] > m ? colors[i] : m;
    typedef cub::BlockReduce<int, 256> BR;
    __shared__ typename BR::TempStorage tmp;
    int b = BR(tmp).Reduce(m, cub::Max());
    if (threadIdx.x == 0) atomicMax(mx, b);
}

static unsigned warp_grid(int64_t items) {
    // one warp handles 32 consecutive active entries per step
    return grid_for((items + 31) / 32 * 32, 256, 148 * 16);
}

void color(const int64_t *off, const int32_t *nbr, int64_t n, int32_t *colors, int64_t *info_h,
           cudaStream_t s) {
    if (n <= 0) {
        info_h[0] = 0;
        info_h[1] = 0;
        return;
    }
    Buf<int32_t> act0(n, s), act1(n, s), tent(n, s);
    Buf<uint8_t> keep(n, s), rej(n, s);
    Buf<int64_t> cnt(1, s);
    k_color_init<<<grid_for(n, 256), 256, 0, s>>>(colors, act0, n);
    PLV_LAUNCH_CHECK();
    int32_t *active = act0.get(), *next = act1.get();
    int64_t na = n, rounds = 0;
    size_t bytes = 0;
    PLV_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, active, rej.get(), next, cnt.get(), n, s));
    Buf<char> tmp(bytes, s);
    while (na > 0) {
        rounds++;
        k_color_assign<<<warp_grid(na), 256, 0, s>>>(off, nbr, active, na, colors, tent);
        PLV_LAUNCH_CHECK();
        k_color_commit<<<grid_for(na, 256), 256, 0, s>>>(active, na, tent, colors);
        PLV_LAUNCH_CHECK();
        k_color_conflicts<<<warp_grid(na), 256, 0, s>>>(off, nbr, active, na, colors, keep);
        PLV_LAUNCH_CHECK();
        k_reject_flags<<<grid_for(na, 256), 256, 0, s>>>(keep, na, rej);
        PLV_LAUNCH_CHECK();
        size_t b2 = bytes;
        PLV_CUDA(cub::DeviceSelect::Flagged(tmp.get(), b2, active, rej.get(), next, cnt.get(), na, s));
        int64_t nr = d2h(cnt.get(), s);
        if (nr > 0) {
            k_uncolor<<<grid_for(nr, 256), 256, 0, s>>>(next, nr, colors);
            PLV_LAUNCH_CHECK();
        }
        int32_t *t = active;
        active = next;
        next = t;
        na = nr;
    }
    Buf<int> mx(1, s);
    PLV_CUDA(cudaMemsetAsync(mx.get(), 0xff, sizeof(int), s));
    k_max_color<<<grid_for(n, 256, 148 * 4), 256, 0, s>>>(colors, n, mx);
    PLV_LAUNCH_CHECK();
    info_h[0] = (int64_t)d2h(mx.get(), s) + 1;
    info_h[1] = rounds;
}

__global__ void k_class_count(const int32_t *colors, int64_t n, int32_t *cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + colors[i], 1);
}

void color_classes(const int32_t *colors, int64_t n, int64_t nc, int64_t *class_off,
                   int32_t *class_vtx, cudaStream_t s) {
    Buf<int32_t> cnt(nc + 1, s);
    PLV_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(int32_t) * (nc + 1), s));
    if (n > 0) {
        k_class_count<<<grid_for(n, 256), 256, 0, s>>>(colors, n, cnt);
        PLV_LAUNCH_CHECK();
    }
    offsets_from_degrees(cnt, nc, class_off, s);
    if (n <= 0) return;
    Buf<int32_t> idx(n, s);
    Buf<uint32_t> ks(n, s);
    // vertex ids ascending in, stable sort by colour
    iota_i32(idx, n, s);
    sort_pairs<uint32_t, int32_t>(reinterpret_cast<const uint32_t *>(colors), ks, idx, class_vtx, n,
                                  0, bits_for(nc > 1 ? nc : 2), s);
}

}  // namespace plv

extern "C" int plv_color(const int64_t *off, const int32_t *nbr, int64_t n, int64_t max_degree,
                         int32_t *colors, int64_t *info_h, void *stream) {
    PLV_ENTRY
    (void)max_degree;
    plv::color(off, nbr, n, colors, info_h, plv::S(stream));
    PLV_EXIT
}

extern "C" int plv_color_assign(const int64_t *off, const int32_t *nbr, const int32_t *active,
                                int64_t na, const int32_t *colors, int32_t *out_colors,
                                void *stream) {
    PLV_ENTRY
    if (na > 0) {
        plv::k_color_assign<<<plv::warp_grid(na), 256, 0, plv::S(stream)>>>(off, nbr, active, na,
                                                                           colors, out_colors);
        PLV_LAUNCH_CHECK();
    }
    PLV_EXIT
}

extern "C" int plv_color_conflicts(const int64_t *off, const int32_t *nbr, const int32_t *active,
                                   int64_t na, const int32_t *colors, uint8_t *out_keep,
                                   void *stream) {
    PLV_ENTRY
    if (na > 0) {
        plv::k_color_conflicts<<<plv::warp_grid(na), 256, 0, plv::S(stream)>>>(off, nbr, active, na,
                                                                              colors, out_keep);
        PLV_LAUNCH_CHECK();
    }
    PLV_EXIT
}

extern "C" int plv_color_classes(const int32_t *colors, int64_t n, int64_t num_colors,
                                 int64_t *class_off, int32_t *class_vtx, void *stream) {
    PLV_ENTRY
    plv::color_classes(colors, n, num_colors, class_off, class_vtx, plv::S(stream));
    PLV_EXIT
}
