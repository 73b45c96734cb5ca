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
// Low-degree vertices (<= 32 entries) are one thread each with a 64-bit
// "used" mask per window of 64 colours.  Higher-degree vertices are pushed to
// a worklist and handled one block each: the block marks the colours of the
// row in a shared-memory bitmap (windows of 4096 colours) and finds the first
// free bit, or scans the lower-id prefix of the row for a clash.  The round
// loop runs on the device (a CUDA graph WHILE node, see color()): no host
// synchronisation until the colouring is complete.
#include "common.cuh"
#include "csr.cuh"
#include <cub/cub.cuh>

namespace plv {

constexpr int COLOR_THREAD_MAXD = 32;
constexpr int CB = 256;             // threads per block, big-vertex kernels
constexpr int CWIN = 4096;          // colours per bitmap window
constexpr int CBIG_GRID = 148 * 4;  // blocks of the big-vertex kernels

// The active list of a round: a host-driven call passes (a0, na); the device
// loop passes both ping-pong buffers and its control words (ctl[0] = active
// count, ctl[1] = rounds done: round r reads buffer r & 1, writes the other).
struct ActiveRef {
    const int32_t *a0, *a1;
    const int64_t *ctl;
    int64_t na;
    __device__ __forceinline__ const int32_t *act() const {
        return ctl ? ((ctl[1] & 1) ? a1 : a0) : a0;
    }
    __device__ __forceinline__ int32_t *next() const {
        return const_cast<int32_t *>((ctl[1] & 1) ? a0 : a1);
    }
    __device__ __forceinline__ int64_t count() const { return ctl ? ctl[0] : na; }
};

inline ActiveRef host_active(const int32_t *a, int64_t na) { return ActiveRef{a, nullptr, nullptr, na}; }

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

// Tentative colours of low-degree active vertices; the others go to `big`
// (one block each) or, above CPEND entries, to `huge` (split over blocks).
constexpr int64_t CHUGE = 2048;  // entries per huge-row chunk (1024, 2048, 4096 measured)
constexpr int64_t CPEND = 4096;  // rows above this keep pending lists across rounds (512, 1024 measured slower)
constexpr int64_t CMID_MAXD = 512;  // warp per vertex up to here, then a block

__global__ void k_color_assign_small(const int64_t *off, const int32_t *nbr, ActiveRef R,
                                     const int32_t *colors, int32_t *out, int32_t *big,
                                     unsigned long long *nbig, int32_t *huge,
                                     unsigned long long *nhuge, int32_t *mid = nullptr,
                                     unsigned long long *nmid = nullptr) {
    const int32_t *active = R.act();
    const int64_t na = R.count();
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < na;
         x += (int64_t)gridDim.x * blockDim.x) {
        int32_t i = active[x];
        int64_t d = off[i + 1] - off[i];
        if (d <= COLOR_THREAD_MAXD)
            out[x] = first_free_thread(off, nbr, colors, i);
        else if (d <= CMID_MAXD || !mid)
            big[atomicAdd(nbig, 1ull)] = (int32_t)x;
        else if (d <= CPEND || !huge)
            mid[atomicAdd(nmid, 1ull)] = (int32_t)x;
        else
            huge[atomicAdd(nhuge, 1ull)] = (int32_t)x;
    }
}

constexpr int HPT = CHUGE / CB;  // entries per thread per chunk

// Huge rows (> CPEND entries) keep state across the rounds of a colouring,
// per slot (hslot[i]): the bitmap of the colours of their committed
// neighbours (first window of CWIN colours) and, per chunk of CHUGE row
// entries, the sorted list of the chunk's neighbours still uncoloured at the
// last assignment ("pending").  A neighbour that has a colour at an
// assignment is committed -- active vertices carry -1 and committed colours
// never change -- so the bitmap only grows, and round r reads the pending
// lists of round r - 1 (round 0: the row) instead of the whole row.  After
// round r's assignment the pending lists are exactly the neighbours active in
// round r: the only ones a clash can come from.
struct HugeState {
    const int32_t *hslot;  // [n] slot of a huge vertex (only those entries are read)
    const int64_t *hoff;   // [slots] first entry of the slot's region (its degree long)
    const int64_t *hcb;    // [slots] first chunk index of the slot
    const int32_t *cown;   // [chunks] the chunk's slot
    int32_t *pend;         // [entries] pending lists, CHUGE entries per chunk
    int32_t *pc;           // [chunks] pending count per chunk
    uint32_t *bits;        // [slots * CWIN / 32] colours of committed neighbours
    const int32_t *hvid;   // [slots] the slot's vertex
    int32_t *xof;          // [slots] its position in this round's active list
    int64_t *wl[2];        // chunks with pending entries, (slot << 32) | chunk, by round parity
    unsigned long long *wc;  // [2] their counts
};

__device__ __forceinline__ unsigned lanes_below() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Block (q, chunk): the chunk's pending entries (round 0: its row entries).
// Coloured neighbours go into the slot's bitmap (shared-memory
// pre-aggregation, then the non-zero words); the uncoloured ones are
// compacted in place, in order.  A chunk where nothing was committed is left
// as it is.
__global__ void __launch_bounds__(CB) k_color_assign_huge(const int64_t *off, const int32_t *nbr,
                                                          ActiveRef R,
                                                          const int32_t *colors,
                                                          const int32_t *huge,
                                                          const unsigned long long *nhuge,
                                                          HugeState H, int64_t nchunks) {
    constexpr int NWC = CB / 32;
    __shared__ uint32_t sb[CWIN / 32];
    __shared__ int wofs[HPT * NWC];  // pending per (u, warp), then their offsets
    __shared__ int s_tot;
    const int32_t *active = R.act();
    const int64_t r = R.ctl[1];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int cur = (int)(r & 1), nxt = cur ^ 1;
    // round 0: every chunk of every huge row.  color() seeds all n vertices as
    // active, so every huge row is active in round 0; a row that is already
    // coloured (a caller starting from a subset) is skipped below instead of
    // getting pending lists.  Later rounds: the chunks left with pending
    // entries (those of committed vertices are skipped).
    (void)active;
    (void)huge;
    (void)nhuge;
    const int64_t cnt = r == 0 ? nchunks : (int64_t)H.wc[cur];
    for (int64_t w0 = blockIdx.x; w0 < cnt; w0 += gridDim.x) {
        int32_t i, sl;
        int64_t ch, r0 = 0;
        if (r == 0) {
            sl = H.cown[w0];
            ch = w0 - H.hcb[sl];
            i = H.hvid[sl];
            r0 = off[i] + ch * CHUGE;
            if (colors[i] >= 0) continue;  // not active (see above)
        } else {
            const int64_t e = H.wl[cur][w0];
            sl = (int32_t)(e >> 32);
            ch = e & 0xffffffffll;
            i = H.hvid[sl];
            if (colors[i] >= 0) continue;  // committed
        }
        const int64_t deg = off[i + 1] - off[i];
        const int64_t rb = H.hoff[sl] + ch * CHUGE;
        int32_t *reg = H.pend + rb;
        int32_t *pcnt = H.pc + H.hcb[sl] + ch;
        const int32_t *src = r == 0 ? nbr + r0 : reg;
        const int64_t len = r == 0 ? (deg - ch * CHUGE < CHUGE ? deg - ch * CHUGE : CHUGE) : *pcnt;
        if (len == 0) continue;
        for (int w = threadIdx.x; w < CWIN / 32; w += CB) sb[w] = 0u;
        __syncthreads();
        int32_t jj[HPT], cc[HPT];
#pragma unroll
        for (int u = 0; u < HPT; u++) {
            const int64_t e = threadIdx.x + u * CB;
            jj[u] = e < len ? src[e] : i;
        }
#pragma unroll
        for (int u = 0; u < HPT; u++) cc[u] = jj[u] != i ? colors[jj[u]] : 0x7fffffff;
        unsigned m[HPT];
        bool done = false;
#pragma unroll
        for (int u = 0; u < HPT; u++) {
            m[u] = __ballot_sync(0xffffffffu, cc[u] < 0);
            if (lane == 0) wofs[u * NWC + wid] = __popc(m[u]);
            if (cc[u] >= 0 && cc[u] != 0x7fffffff) {
                done = true;
                if (cc[u] < CWIN) atomicOr(sb + (cc[u] >> 5), 1u << (cc[u] & 31));
            }
        }
        int left = (int)len;
        if (__syncthreads_or(done) || r == 0) {
            if (wid == 0) {  // exclusive scan of the (u, warp) counts, in entry order
                constexpr int PER = HPT * NWC / 32;
                int v[PER], t = 0;
#pragma unroll
                for (int k = 0; k < PER; k++) {
                    v[k] = wofs[lane * PER + k];
                    t += v[k];
                }
                int incl = t;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                int base = incl - t;
#pragma unroll
                for (int k = 0; k < PER; k++) {
                    wofs[lane * PER + k] = base;
                    base += v[k];
                }
                if (lane == 31) s_tot = incl;
            }
            __syncthreads();
            const unsigned lt = lanes_below();
#pragma unroll
            for (int u = 0; u < HPT; u++)
                if (cc[u] < 0) reg[wofs[u * NWC + wid] + __popc(m[u] & lt)] = jj[u];
            if (threadIdx.x == 0) *pcnt = s_tot;
            left = s_tot;  // read before the barrier below
        }
        if (threadIdx.x == 0 && left > 0)
            H.wl[nxt][atomicAdd(H.wc + nxt, 1ull)] = ((int64_t)sl << 32) | ch;
        __syncthreads();
        uint32_t *bits = H.bits + (int64_t)sl * (CWIN / 32);
        for (int w = threadIdx.x; w < CWIN / 32; w += CB)
            if (sb[w]) atomicOr(bits + w, sb[w]);
        __syncthreads();
    }
}

// First free colour of every huge item from its slot's bitmap (block per
// item); a row whose first CWIN colours are all taken falls back to windowed
// scans of the row.
__global__ void __launch_bounds__(CB) k_color_huge_final(const int64_t *off, const int32_t *nbr,
                                                         ActiveRef R,
                                                         const int32_t *colors,
                                                         const int32_t *huge,
                                                         const unsigned long long *nhuge,
                                                         HugeState H, int32_t *out,
                                                         uint8_t *keep) {
    const int32_t *active = R.act();
    __shared__ uint32_t bits[CWIN / 32];
    __shared__ int s_found;
    const int tid = threadIdx.x;
    const int64_t cnt = (int64_t)*nhuge;
    if (blockIdx.x == 0 && tid == 0) H.wc[R.ctl[1] & 1] = 0ull;  // read by the assignment only
    for (int64_t q = blockIdx.x; q < cnt; q += gridDim.x) {
        int64_t x = huge[q];
        int32_t i = active[x];
        const int32_t sl = H.hslot[i];
        if (tid == 0) {
            s_found = INT32_MAX;
            H.xof[sl] = (int32_t)x;
        }
        __syncthreads();
        for (int w = tid; w < CWIN / 32; w += CB) {
            uint32_t free = ~H.bits[(int64_t)sl * (CWIN / 32) + w];
            if (free) atomicMin(&s_found, w * 32 + __ffs(free) - 1);
        }
        __syncthreads();
        int f = s_found;
        int64_t e0 = off[i], e1 = off[i + 1];
        for (int base = CWIN; f == INT32_MAX; base += CWIN) {
            __syncthreads();
            for (int w = tid; w < CWIN / 32; w += CB) bits[w] = 0u;
            __syncthreads();
            for (int64_t e = e0 + tid; e < e1; e += CB) {
                int32_t j = nbr[e];
                if (j == i) continue;
                int32_t cj = colors[j] - base;
                if (cj >= 0 && cj < CWIN) atomicOr(bits + (cj >> 5), 1u << (cj & 31));
            }
            __syncthreads();
            for (int w = tid; w < CWIN / 32; w += CB) {
                uint32_t free = ~bits[w];
                if (free) atomicMin(&s_found, base + w * 32 + __ffs(free) - 1);
            }
            __syncthreads();
            f = s_found;
        }
        if (tid == 0) {
            out[x] = f;
            keep[x] = 1;  // k_color_conflicts_huge clears it on a clash
        }
        __syncthreads();
    }
}

// Huge rows: block per chunk with pending entries after this round's
// assignment (the worklist it wrote) scans them -- the neighbours active this
// round, sorted: the j < i prefix ends the scan -- for a lower id with the
// same tentative colour.
__global__ void __launch_bounds__(CB) k_color_conflicts_huge(ActiveRef R,
                                                             const int32_t *colors,
                                                             HugeState H, uint8_t *keep) {
    const int nxt = (int)((R.ctl[1] + 1) & 1);
    const int64_t cnt = (int64_t)H.wc[nxt];
    for (int64_t w = blockIdx.x; w < cnt; w += gridDim.x) {
        const int64_t e = H.wl[nxt][w];
        const int32_t sl = (int32_t)(e >> 32);
        const int64_t ch = e & 0xffffffffll;
        const int32_t i = H.hvid[sl];
        const int64_t rb = H.hoff[sl] + ch * CHUGE;
        const int32_t *src = H.pend + rb;
        const int64_t len = H.pc[H.hcb[sl] + ch];
        if (src[0] >= i) continue;  // block-uniform
        const int32_t ci = colors[i];
        int32_t jj[HPT];
#pragma unroll
        for (int u = 0; u < HPT; u++) {
            const int64_t t = threadIdx.x + u * CB;
            jj[u] = t < len ? src[t] : i;
        }
        bool clash = false;
#pragma unroll
        for (int u = 0; u < HPT; u++)
            if (jj[u] < i && colors[jj[u]] == ci) clash = true;
        if (clash) keep[H.xof[sl]] = 0;
    }
}

// One warp per active vertex of COLOR_THREAD_MAXD < degree <= CMID_MAXD: a 1024-colour bitmap per warp in shared memory, windows of 1024
// colours until one has a free bit.
constexpr int WWIN = 1024;

__global__ void __launch_bounds__(CB) k_color_assign_big(const int64_t *off, const int32_t *nbr,
                                                         ActiveRef R, const int32_t *colors,
                                                         int32_t *out, const int32_t *big,
                                                         const unsigned long long *nbig) {
    __shared__ uint32_t bits[CB / 32][WWIN / 32];
    const int32_t *active = R.act();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t *wb = bits[wid];
    const int64_t cnt = (int64_t)*nbig;
    for (int64_t q = blockIdx.x * (int64_t)(CB / 32) + wid; q < cnt;
         q += (int64_t)gridDim.x * (CB / 32)) {
        const int64_t x = big[q];
        const int32_t i = active[x];
        const int64_t e0 = off[i], e1 = off[i + 1];
        for (int base = 0;; base += WWIN) {
            wb[lane] = 0u;
            __syncwarp();
            for (int64_t e = e0 + lane; e < e1; e += 32) {
                const int32_t j = nbr[e];
                if (j == i) continue;
                const int32_t cj = colors[j] - base;
                if (cj >= 0 && cj < WWIN) atomicOr(wb + (cj >> 5), 1u << (cj & 31));
            }
            __syncwarp();
            const uint32_t fr = ~wb[lane];  // lane l owns colours [32 l, 32 l + 32)
            const unsigned any = __ballot_sync(0xffffffffu, fr != 0u);
            __syncwarp();
            if (any) {
                const int l = __ffs(any) - 1;
                const uint32_t frl = __shfl_sync(0xffffffffu, fr, l);
                if (lane == 0) out[x] = base + l * 32 + __ffs(frl) - 1;
                break;
            }
        }
    }
}

// One block per active vertex of CMID_MAXD < degree <= CPEND: bitmap of
// neighbour colours in shared memory.
__global__ void __launch_bounds__(CB) k_color_assign_mid(const int64_t *off, const int32_t *nbr,
                                                         ActiveRef R, const int32_t *colors,
                                                         int32_t *out, const int32_t *big,
                                                         const unsigned long long *nbig) {
    const int32_t *active = R.act();
    __shared__ uint32_t bits[CWIN / 32];
    __shared__ int s_found;
    const int tid = threadIdx.x;
    const int64_t cnt = (int64_t)*nbig;
    for (int64_t q = blockIdx.x; q < cnt; q += gridDim.x) {
        int64_t x = big[q];
        int32_t i = active[x];
        int64_t e0 = off[i], e1 = off[i + 1];
        for (int base = 0;; base += CWIN) {
            for (int w = tid; w < CWIN / 32; w += CB) bits[w] = 0u;
            if (tid == 0) s_found = INT32_MAX;
            __syncthreads();
            for (int64_t e = e0 + tid; e < e1; e += CB) {
                int32_t j = nbr[e];
                if (j == i) continue;
                int32_t cj = colors[j] - base;
                if (cj >= 0 && cj < CWIN) atomicOr(bits + (cj >> 5), 1u << (cj & 31));
            }
            __syncthreads();
            for (int w = tid; w < CWIN / 32; w += CB) {
                uint32_t free = ~bits[w];
                if (free) atomicMin(&s_found, w * 32 + __ffs(free) - 1);
            }
            __syncthreads();
            int f = s_found;
            __syncthreads();
            if (f != INT32_MAX) {
                if (tid == 0) out[x] = base + f;
                break;
            }
        }
    }
}

// keep[x] = no lower-id neighbour shares colors[active[x]] (low degree).
__global__ void k_color_conflicts_small(const int64_t *off, const int32_t *nbr, ActiveRef R,
                                        const int32_t *colors, uint8_t *keep) {
    const int32_t *active = R.act();
    const int64_t na = R.count();
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < na;
         x += (int64_t)gridDim.x * blockDim.x) {
        int32_t i = active[x];
        int64_t e0 = off[i], e1 = off[i + 1];
        if (e1 - e0 > COLOR_THREAD_MAXD) continue;
        int32_t ci = colors[i];
        uint8_t k = 1;
        for (int64_t e = e0; e < e1; e++) {
            int32_t j = nbr[e];
            if (j >= i) break;  // rows are sorted: only the prefix j < i matters
            if (colors[j] == ci) {
                k = 0;
                break;
            }
        }
        keep[x] = k;
    }
}

__global__ void __launch_bounds__(CB) k_color_conflicts_big(const int64_t *off, const int32_t *nbr,
                                                            ActiveRef R,
                                                            const int32_t *colors, uint8_t *keep,
                                                            const int32_t *big,
                                                            const unsigned long long *nbig) {
    const int32_t *active = R.act();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t cnt = (int64_t)*nbig;
    for (int64_t q = blockIdx.x * (int64_t)(CB / 32) + wid; q < cnt;
         q += (int64_t)gridDim.x * (CB / 32)) {
        const int64_t x = big[q];
        const int32_t i = active[x];
        const int32_t ci = colors[i];
        const int64_t e0 = off[i], e1 = off[i + 1];
        bool clash = false;
        for (int64_t c0 = e0; c0 < e1; c0 += 32) {
            const int64_t e = c0 + lane;
            bool past = true;
            if (e < e1) {
                const int32_t j = nbr[e];
                past = j >= i;  // rows are sorted: only the prefix j < i matters
                if (!past && colors[j] == ci) clash = true;
            }
            if (__any_sync(0xffffffffu, clash || past)) break;
        }
        clash = __any_sync(0xffffffffu, clash);
        if (lane == 0) keep[x] = clash ? 0 : 1;
    }
}

__global__ void __launch_bounds__(CB) k_color_conflicts_mid(const int64_t *off, const int32_t *nbr,
                                                            ActiveRef R,
                                                            const int32_t *colors, uint8_t *keep,
                                                            const int32_t *big,
                                                            const unsigned long long *nbig) {
    const int32_t *active = R.act();
    const int tid = threadIdx.x;
    const int64_t cnt = (int64_t)*nbig;
    for (int64_t q = blockIdx.x; q < cnt; q += gridDim.x) {
        int64_t x = big[q];
        int32_t i = active[x];
        int32_t ci = colors[i];
        int64_t e0 = off[i], e1 = off[i + 1];
        bool clash = false;
        for (int64_t c0 = e0; c0 < e1; c0 += CB) {
            int64_t e = c0 + tid;
            bool past = true;
            if (e < e1) {
                int32_t j = nbr[e];
                past = j >= i;
                if (!past && colors[j] == ci) clash = true;
            }
            // stop once the whole chunk is past the j < i prefix or a clash is seen
            int stop = __syncthreads_or(clash || past);
            if (stop) break;
        }
        clash = __syncthreads_or(clash);
        if (tid == 0) keep[x] = clash ? 0 : 1;
    }
}

__global__ void k_big_list(const int64_t *off, const int32_t *active, int64_t na, int32_t *big,
                           unsigned long long *nbig) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < na;
         x += (int64_t)gridDim.x * blockDim.x) {
        int32_t i = active[x];
        if (off[i + 1] - off[i] > COLOR_THREAD_MAXD) big[atomicAdd(nbig, 1ull)] = (int32_t)x;
    }
}

__global__ void k_color_init(int32_t *colors, int32_t *active, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        colors[i] = -1;
        active[i] = (int32_t)i;
    }
}

__global__ void k_color_commit(ActiveRef R, const int32_t *tent, int32_t *colors) {
    const int32_t *active = R.act();
    const int64_t na = R.count();
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < na;
         x += (int64_t)gridDim.x * blockDim.x)
        colors[active[x]] = tent[x];
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

// One speculative round over the active list: tentative colours, commit, keep flags.
struct ColorScratch {
    int32_t *big, *huge, *mid;
    unsigned long long *cnt;  // [0] big, [1] huge, [2] mid (zero at the start of a round)
    HugeState H;              // huge rows' state across rounds
    int64_t nhuge_max;
    int64_t huge_chunks;      // chunks of the rows above CPEND
};

// Side streams of a captured round: the big / mid / huge kernels of the
// assignment and of the conflict test touch disjoint vertices, so each group
// runs as parallel graph branches (fork / join events).
struct RoundStreams {
    cudaStream_t side[2] = {nullptr, nullptr};
    cudaEvent_t fork = nullptr, join[2] = {nullptr, nullptr};
    void create() {
        for (int t = 0; t < 2; t++) {
            PLV_CUDA(cudaStreamCreateWithFlags(&side[t], cudaStreamNonBlocking));
            PLV_CUDA(cudaEventCreateWithFlags(&join[t], cudaEventDisableTiming));
        }
        PLV_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    }
    void destroy() {
        for (int t = 0; t < 2; t++) {
            if (side[t]) cudaStreamDestroy(side[t]);
            if (join[t]) cudaEventDestroy(join[t]);
        }
        if (fork) cudaEventDestroy(fork);
    }
    void split(cudaStream_t s) {
        PLV_CUDA(cudaEventRecord(fork, s));
        for (int t = 0; t < 2; t++) PLV_CUDA(cudaStreamWaitEvent(side[t], fork, 0));
    }
    void merge(cudaStream_t s) {
        for (int t = 0; t < 2; t++) {
            PLV_CUDA(cudaEventRecord(join[t], side[t]));
            PLV_CUDA(cudaStreamWaitEvent(s, join[t], 0));
        }
    }
};

// Grid of the huge-row kernels: grid-stride loops over the pairs / chunks;
// after round 0 only a few chunks have work, so no more than a wave or two.
constexpr unsigned HUGE_GRID_MAX = 148 * 3;  // 3, 8, 16 measured
static unsigned huge_grid(int64_t chunks) {
    return chunks < (int64_t)HUGE_GRID_MAX ? (unsigned)(chunks > 0 ? chunks : 1) : HUGE_GRID_MAX;
}

static void color_round(const int64_t *off, const int32_t *nbr, ActiveRef R, int64_t na_max,
                        int32_t *colors, int32_t *tent, uint8_t *keep, const ColorScratch &C,
                        cudaStream_t s, RoundStreams *rs = nullptr) {
    bool huge = C.nhuge_max > 0;
    const unsigned g = grid_for(na_max, 256, 148 * 8);
    cudaStream_t s1 = rs ? rs->side[0] : s, s2 = rs ? rs->side[1] : s;
    k_color_assign_small<<<g, 256, 0, s>>>(off, nbr, R, colors, tent, C.big, C.cnt,
                                           huge ? C.huge : nullptr, C.cnt + 1, C.mid, C.cnt + 2);
    PLV_LAUNCH_CHECK();
    if (rs) rs->split(s);
    k_color_assign_big<<<CBIG_GRID, CB, 0, s1>>>(off, nbr, R, colors, tent, C.big, C.cnt);
    PLV_LAUNCH_CHECK();
    k_color_assign_mid<<<CBIG_GRID, CB, 0, s2>>>(off, nbr, R, colors, tent, C.mid, C.cnt + 2);
    PLV_LAUNCH_CHECK();
    if (huge) {
        k_color_assign_huge<<<huge_grid(C.huge_chunks), CB, 0, s>>>(off, nbr, R, colors, C.huge,
                                                                    C.cnt + 1, C.H, C.huge_chunks);
        PLV_LAUNCH_CHECK();
        k_color_huge_final<<<148 * 4, CB, 0, s>>>(off, nbr, R, colors, C.huge, C.cnt + 1, C.H,
                                              tent, keep);
        PLV_LAUNCH_CHECK();
    }
    if (rs) rs->merge(s);
    k_color_commit<<<g, 256, 0, s>>>(R, tent, colors);
    PLV_LAUNCH_CHECK();
    if (rs) rs->split(s);
    k_color_conflicts_small<<<g, 256, 0, s>>>(off, nbr, R, colors, keep);
    PLV_LAUNCH_CHECK();
    k_color_conflicts_big<<<CBIG_GRID, CB, 0, s1>>>(off, nbr, R, colors, keep, C.big, C.cnt);
    PLV_LAUNCH_CHECK();
    k_color_conflicts_mid<<<CBIG_GRID, CB, 0, s2>>>(off, nbr, R, colors, keep, C.mid, C.cnt + 2);
    PLV_LAUNCH_CHECK();
    if (huge) {
        k_color_conflicts_huge<<<huge_grid(C.huge_chunks), CB, 0, s>>>(R, colors, C.H, keep);
        PLV_LAUNCH_CHECK();
    }
    if (rs) rs->merge(s);
}

// Stable compaction of the rejected (keep == 0) active vertices into the
// other buffer, which they leave uncoloured (PL/heuristics.py:113-115):
// per-tile counts, one-block scan of the tile counts, ordered scatter.
constexpr int RT = 256, RI = 4, RTILE = RT * RI;

// Per-tile rejected counts; the last block to finish (ticket ctl[3]) turns
// them into exclusive tile offsets and the total ctl[2].
__global__ void __launch_bounds__(RT) k_rej_tiles(ActiveRef R, const uint8_t *keep,
                                                  int64_t *tsum, int64_t *ctl) {
    typedef cub::BlockReduce<int, RT> BR;
    typedef cub::BlockScan<int64_t, RT> Scan;
    __shared__ union {
        typename BR::TempStorage red;
        typename Scan::TempStorage scan;
    } tmp;
    __shared__ bool s_last;
    const int64_t na = R.count(), nt = (na + RTILE - 1) / RTILE;
    for (int64_t t = blockIdx.x; t < nt; t += gridDim.x) {
        int c = 0;
#pragma unroll
        for (int u = 0; u < RI; u++) {
            const int64_t x = t * RTILE + threadIdx.x * RI + u;
            c += (x < na && !keep[x]) ? 1 : 0;
        }
        const int tot = BR(tmp.red).Sum(c);
        if (threadIdx.x == 0) tsum[t] = tot;
        __syncthreads();
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0)
        s_last = atomicAdd((unsigned long long *)(ctl + 3), 1ull) == (unsigned long long)gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int64_t per = (nt + RT - 1) / RT, t0 = threadIdx.x * per;
    int64_t loc = 0;
    for (int64_t t = t0; t < t0 + per && t < nt; t++) loc += __ldcg(tsum + t);
    int64_t base, total;
    Scan(tmp.scan).ExclusiveSum(loc, base, total);
    for (int64_t t = t0; t < t0 + per && t < nt; t++) {
        const int64_t v = __ldcg(tsum + t);
        tsum[t] = base;
        base += v;
    }
    if (threadIdx.x == 0) {
        ctl[2] = total;
        ctl[3] = 0;
    }
}

// Ordered scatter of the rejected into the other buffer (uncoloured); the
// last block (ticket ctl[4]) ends the round: the rejected become the active
// list, the worklist counters reset, and the loop continues while any.
__global__ void __launch_bounds__(RT) k_rej_scatter(ActiveRef R, const uint8_t *keep,
                                                    const int64_t *tsum, int32_t *colors,
                                                    int64_t *ctl, unsigned long long *cnt,
                                                    cudaGraphConditionalHandle h) {
    typedef cub::BlockScan<int, RT> Scan;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ bool s_last;
    const int32_t *A = R.act();
    int32_t *N = R.next();
    const int64_t na = R.count(), nt = (na + RTILE - 1) / RTILE;
    for (int64_t t = blockIdx.x; t < nt; t += gridDim.x) {
        int f[RI], c = 0;
#pragma unroll
        for (int u = 0; u < RI; u++) {
            const int64_t x = t * RTILE + threadIdx.x * RI + u;
            f[u] = (x < na && !keep[x]) ? 1 : 0;
            c += f[u];
        }
        int pos;
        Scan(tmp).ExclusiveSum(c, pos);
        int64_t o = tsum[t] + pos;
#pragma unroll
        for (int u = 0; u < RI; u++) {
            if (!f[u]) continue;
            const int32_t i = A[t * RTILE + threadIdx.x * RI + u];
            N[o++] = i;
            colors[i] = -1;
        }
        __syncthreads();
    }
    __syncthreads();
    if (threadIdx.x == 0)
        s_last = atomicAdd((unsigned long long *)(ctl + 4), 1ull) == (unsigned long long)gridDim.x - 1;
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        const int64_t nr = ctl[2];
        ctl[0] = nr;
        ctl[1] += 1;
        ctl[4] = 0;
        cnt[0] = cnt[1] = cnt[2] = 0ull;
        cudaGraphSetConditional(h, nr > 0 ? 1u : 0u);
    }
}

// ctl: [0] active count, [1] rounds done, [2] rejected count, [3] / [4]
// tickets of the compaction kernels' last blocks.
__global__ void k_color_init_ctl(int64_t *ctl, int64_t n, unsigned long long *cnt) {
    ctl[0] = n;
    ctl[1] = 0;
    ctl[2] = 0;
    ctl[3] = 0;
    ctl[4] = 0;
    cnt[0] = cnt[1] = cnt[2] = 0ull;
}

// cnt[0] rows above CPEND, cnt[1] max degree, cnt[2] their entries, cnt[3] their chunks.
__global__ void k_count_huge(const int64_t *off, int64_t n, unsigned long long *cnt) {
    unsigned long long c = 0, md = 0, te = 0, tk = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long d = (unsigned long long)(off[i + 1] - off[i]);
        c += d > (unsigned long long)CPEND;
        te += d > (unsigned long long)CPEND ? d : 0ull;
        tk += d > (unsigned long long)CPEND ? (d + CHUGE - 1) / CHUGE : 0ull;
        md = d > md ? d : md;
    }
    typedef cub::BlockReduce<unsigned long long, 256> BR;
    __shared__ typename BR::TempStorage t1;
    unsigned long long tc = BR(t1).Sum(c);
    __syncthreads();
    unsigned long long tt = BR(t1).Sum(te);
    __syncthreads();
    unsigned long long tkk = BR(t1).Sum(tk);
    __syncthreads();
    unsigned long long tm = BR(t1).Reduce(md, cub::Max());
    if (threadIdx.x == 0) {
        if (tc) atomicAdd(cnt, tc);
        if (tt) atomicAdd(cnt + 2, tt);
        if (tkk) atomicAdd(cnt + 3, tkk);
        atomicMax(cnt + 1, tm);
    }
}

// Slots of the huge rows (any order) and their pending-list offsets.
__global__ void k_huge_slots(const int64_t *off, int64_t n, int32_t *hslot, int64_t *hoff,
                             int64_t *hcb, int32_t *cown, int32_t *hvid,
                             unsigned long long *ctr) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long d = (unsigned long long)(off[i + 1] - off[i]);
        if (d <= (unsigned long long)CPEND) continue;
        const int32_t sl = (int32_t)atomicAdd(ctr, 1ull);
        hslot[i] = sl;
        hvid[sl] = (int32_t)i;
        hoff[sl] = (int64_t)atomicAdd(ctr + 1, d);
        const unsigned long long nc = (d + CHUGE - 1) / CHUGE;
        const int64_t cb = (int64_t)atomicAdd(ctr + 2, nc);
        hcb[sl] = cb;
        for (unsigned long long c = 0; c < nc; c++) cown[cb + c] = sl;
    }
}

// The whole colouring as one CUDA graph: init, then WHILE (active) { round;
// compaction; step }.  Rounds repeat until no vertex is rejected, exactly as
// the host loop of PL/heuristics.py:100-116, with no host round trip per round.
void color(const int64_t *off, const int32_t *nbr, int64_t n, int32_t *colors, int64_t *info_h,
           cudaStream_t s) {
    if (n <= 0) {
        info_h[0] = 0;
        info_h[1] = 0;
        return;
    }
    Buf<int32_t> act0(n, s), act1(n, s), tent(n, s), big(n, s), mid(n, s);
    Buf<uint8_t> keep(n, s);
    Buf<int64_t> ctl(6, s), tsum((n + RTILE - 1) / RTILE + 1, s);
    Buf<unsigned long long> cnts(8, s);
    PLV_CUDA(cudaMemsetAsync(cnts.get(), 0, 8 * sizeof(unsigned long long), s));
    k_count_huge<<<grid_for(n, 256, 148 * 4), 256, 0, s>>>(off, n, cnts.get() + 4);
    PLV_LAUNCH_CHECK();
    unsigned long long hc[4];
    PLV_CUDA(cudaMemcpyAsync(hc, cnts.get() + 4, sizeof(hc), cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    const int64_t nh = (int64_t)hc[0], nh1 = nh ? nh : 1, ne1 = hc[2] ? (int64_t)hc[2] : 1,
                  nk1 = hc[3] ? (int64_t)hc[3] : 1;
    Buf<int32_t> huge(nh1, s), hslot(nh ? n : 1, s), pend(ne1, s), hpc(nk1, s), cown(nk1, s),
        hvid(nh1, s), xof(nh1, s);
    Buf<int64_t> hoff(nh1, s), hcb(nh1, s), wl0(nk1, s), wl1(nk1, s);
    Buf<unsigned long long> hctr(6, s);
    Buf<uint32_t> hbits(nh1 * (CWIN / 32), s);
    if (nh) {
        PLV_CUDA(cudaMemsetAsync(hctr.get(), 0, sizeof(unsigned long long) * 6, s));
        PLV_CUDA(cudaMemsetAsync(hbits.get(), 0, sizeof(uint32_t) * nh1 * (CWIN / 32), s));
        k_huge_slots<<<grid_for(n, 256, 148 * 4), 256, 0, s>>>(off, n, hslot, hoff, hcb, cown, hvid,
                                                               hctr);
        PLV_LAUNCH_CHECK();
    }
    HugeState H{hslot.get(), hoff.get(), hcb.get(), cown.get(), pend.get(), hpc.get(), hbits.get(),
                hvid.get(), xof.get(), {wl0.get(), wl1.get()}, hctr.get() + 4};
    ColorScratch C{big.get(), huge.get(), mid.get(), cnts.get(), H, nh, (int64_t)hc[3]};
    k_color_init<<<grid_for(n, 256), 256, 0, s>>>(colors, act0, n);
    PLV_LAUNCH_CHECK();
    k_color_init_ctl<<<1, 1, 0, s>>>(ctl, n, cnts);
    PLV_LAUNCH_CHECK();
    PLV_CUDA(cudaStreamSynchronize(s));
    ActiveRef R{act0.get(), act1.get(), ctl.get(), 0};
    cudaGraph_t graph = nullptr, body = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaStream_t cs = nullptr;
    RoundStreams rs;
    try {
        PLV_CUDA(cudaGraphCreate(&graph, 0));
        cudaGraphConditionalHandle h;
        PLV_CUDA(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t loop;
        PLV_CUDA(cudaGraphAddNode(&loop, graph, nullptr, 0, &cp));
        body = cp.conditional.phGraph_out[0];
        PLV_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        rs.create();
        PLV_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0,
                                               cudaStreamCaptureModeThreadLocal));
        try {
            color_round(off, nbr, R, n, colors, tent, keep, C, cs, &rs);
            const unsigned gt = grid_for((n + RTILE - 1) / RTILE, 1, 148 * 8);
            k_rej_tiles<<<gt, RT, 0, cs>>>(R, keep, tsum, ctl);
            PLV_LAUNCH_CHECK();
            k_rej_scatter<<<gt, RT, 0, cs>>>(R, keep, tsum, colors, ctl, cnts, h);
            PLV_LAUNCH_CHECK();
        } catch (...) {
            cudaGraph_t g2 = nullptr;
            cudaStreamEndCapture(cs, &g2);
            throw;
        }
        cudaGraph_t got = nullptr;
        PLV_CUDA(cudaStreamEndCapture(cs, &got));
        PLV_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        PLV_CUDA(cudaGraphLaunch(exec, s));
        PLV_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        if (cs) cudaStreamDestroy(cs);
        rs.destroy();
        throw;
    }
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    cudaStreamDestroy(cs);
    rs.destroy();
    int64_t c[2];
    PLV_CUDA(cudaMemcpyAsync(c, ctl.get(), sizeof(c), cudaMemcpyDeviceToHost, s));
    Buf<int> mx(1, s);
    PLV_CUDA(cudaMemsetAsync(mx.get(), 0xff, sizeof(int), s));
    k_max_color<<<grid_for(n, 256, 148 * 4), 256, 0, s>>>(colors, n, mx);
    PLV_LAUNCH_CHECK();
    info_h[0] = (int64_t)d2h(mx.get(), s) + 1;
    info_h[1] = c[1];
}

__global__ void k_class_count(const int32_t *colors, int64_t n, int32_t *cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
    {
        // one atomic per (warp, colour): colour 0 holds most vertices
        const int32_t c = colors[i];
        const unsigned grp = __match_any_sync(__activemask(), c);
        if ((threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(cnt + c, __popc(grp));
    }
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
    iota_i32(idx, n, s);  // vertex ids ascending in, stable sort by colour
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
        cudaStream_t s = plv::S(stream);
        plv::Buf<int32_t> big(na, s);
        plv::Buf<unsigned long long> nbig(1, s);
        PLV_CUDA(cudaMemsetAsync(nbig.get(), 0, sizeof(unsigned long long), s));
        plv::k_color_assign_small<<<plv::grid_for(na, 256), 256, 0, s>>>(
            off, nbr, plv::host_active(active, na), colors, out_colors, big, nbig, nullptr, nullptr);
        PLV_LAUNCH_CHECK();
        plv::k_color_assign_big<<<plv::CBIG_GRID, plv::CB, 0, s>>>(
            off, nbr, plv::host_active(active, na), colors, out_colors, big, nbig);
        PLV_LAUNCH_CHECK();
        PLV_CUDA(cudaStreamSynchronize(s));
    }
    PLV_EXIT
}

extern "C" int plv_color_conflicts(const int64_t *off, const int32_t *nbr, const int32_t *active,
                                   int64_t na, const int32_t *colors, uint8_t *out_keep,
                                   void *stream) {
    PLV_ENTRY
    if (na > 0) {
        cudaStream_t s = plv::S(stream);
        plv::Buf<int32_t> big(na, s);
        plv::Buf<unsigned long long> nbig(1, s);
        PLV_CUDA(cudaMemsetAsync(nbig.get(), 0, sizeof(unsigned long long), s));
        plv::k_color_conflicts_small<<<plv::grid_for(na, 256), 256, 0, s>>>(
            off, nbr, plv::host_active(active, na), colors, out_keep);
        PLV_LAUNCH_CHECK();
        plv::k_big_list<<<plv::grid_for(na, 256), 256, 0, s>>>(off, active, na, big, nbig);
        PLV_LAUNCH_CHECK();
        plv::k_color_conflicts_big<<<plv::CBIG_GRID, plv::CB, 0, s>>>(
            off, nbr, plv::host_active(active, na), colors, out_keep, big, nbig);
        PLV_LAUNCH_CHECK();
        PLV_CUDA(cudaStreamSynchronize(s));
    }
    PLV_EXIT
}

extern "C" int plv_color_classes(const int32_t *colors, int64_t n, int64_t num_colors,
                                 int64_t *class_off, int32_t *class_vtx, void *stream) {
    PLV_ENTRY
    plv::color_classes(colors, n, num_colors, class_off, class_vtx, plv::S(stream));
    PLV_EXIT
}
