// decide.cu -- decide_moves (PL/_kernels.pyx:21-101) on device.
//
// Vertices of a stage are degree-binned once per plan:
//   tier 0  deg <= 8      thread per vertex, candidate list in registers
//   tier 1  deg <= 128    warp per vertex, hash table in shared memory
//   tier 2  deg <= 2048   block per vertex, hash table in shared memory
//   tier 3  larger (hubs) sort-based: every hub entry becomes a
//           (hub, community) key; one stable radix sort over all hubs of the
//           stage groups each community's entries in adjacency order, and a
//           block per hub folds the runs in parallel (runs of different
//           communities are independent; each run is the reference's
//           sequential left fold, so the critical path is the longest run,
//           not the row).
// Tiers 1-2 fold a 32-entry chunk at a time: lanes with the same community
// are grouped with __match_any_sync and the group leader adds their weights
// in lane (= adjacency) order; chunks are processed in order.  Integral graphs
// (every weight an integer, 2m < 2^52) may fold in any order and use atomics.
#include "localmove.cuh"
#include "csr.cuh"
#include <cub/cub.cuh>

namespace plv {

__device__ __forceinline__ int64_t LBL(const int32_t *labels, int32_t c) {
    return labels ? (int64_t)labels[c] : (int64_t)c;
}

// (gain, label) lexicographic order of PL/_kernels.pyx:88.
__device__ __forceinline__ bool better(double g1, int64_t l1, double g2, int64_t l2) {
    return g1 > g2 || (g1 == g2 && l1 < l2);
}

// Eq. 4 gain, PL/_kernels.pyx:86-87, evaluated with one rounding per op.
__device__ __forceinline__ double gain_of(double e_c, double e_old, double m, double ki,
                                          double a_old_excl, double atot_c, double four_m_sq) {
    double t2 = ddiv(dsub(e_c, e_old), m);
    double tk = dmul(2.0, ki);
    double t5 = dsub(dmul(tk, a_old_excl), dmul(tk, atot_c));
    return dadd(t2, ddiv(t5, four_m_sq));
}

__device__ __forceinline__ uint32_t hslot(int32_t c, uint32_t mask) {
    return ((uint32_t)c * 0x9E3779B1u) & mask;
}

// Find-or-insert c; tables start cleared to key -1 / value 0.0.
__device__ __forceinline__ uint32_t probe_insert(int32_t *keys, int32_t c, uint32_t mask) {
    uint32_t s = hslot(c, mask);
    while (true) {
        int32_t k = keys[s];
        if (k == c) return s;
        if (k == -1) {
            int32_t old = atomicCAS(keys + s, -1, c);
            if (old == -1 || old == c) return s;
        }
        s = (s + 1) & mask;
    }
}

__device__ __forceinline__ int probe_find(const int32_t *keys, int32_t c, uint32_t mask) {
    uint32_t s = hslot(c, mask);
    while (true) {
        int32_t k = keys[s];
        if (k == c) return (int)s;
        if (k == -1) return -1;
        s = (s + 1) & mask;
    }
}

// Final decision of PL/_kernels.pyx:92-98.
__device__ __forceinline__ void finish_vertex(const DecideArgs &A, int64_t x, int32_t c_old,
                                              double e_old, double bg, int32_t bc, double be) {
    bool moved = bg > 0.0 && bc != c_old;
    if (moved && A.sizes[c_old] == 1 && A.sizes[bc] == 1 &&
        LBL(A.labels, bc) > LBL(A.labels, c_old))
        moved = false;  // singleton-pair guard
    A.out_target[x] = moved ? bc : c_old;
    A.out_moved[x] = moved ? 1 : 0;
    A.out_e_old[x] = e_old;
    A.out_e_best[x] = moved ? be : e_old;
}

// Warp-level argmax reduction under `better`; result valid in every lane.
__device__ __forceinline__ void warp_best(double &bg, int64_t &bl, int32_t &bc, double &be) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double g2 = __shfl_xor_sync(FULL, bg, o);
        int64_t l2 = __shfl_xor_sync(FULL, bl, o);
        int32_t c2 = __shfl_xor_sync(FULL, bc, o);
        double e2 = __shfl_xor_sync(FULL, be, o);
        if (better(g2, l2, bg, bl)) {
            bg = g2;
            bl = l2;
            bc = c2;
            be = e2;
        }
    }
}

struct BestSmem {
    double g[BLK / 32];
    int64_t l[BLK / 32];
    int32_t c[BLK / 32];
    double e[BLK / 32];
};

// Block-level argmax (BLK threads); the result is valid in thread 0.
__device__ __forceinline__ void block_best(BestSmem &S, double &bg, int64_t &bl, int32_t &bc,
                                           double &be, int64_t l0, int32_t c0) {
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    warp_best(bg, bl, bc, be);
    if (lane == 0) {
        S.g[wid] = bg;
        S.l[wid] = bl;
        S.c[wid] = bc;
        S.e[wid] = be;
    }
    __syncthreads();
    if (wid == 0) {
        if (lane < BLK / 32) {
            bg = S.g[lane];
            bl = S.l[lane];
            bc = S.c[lane];
            be = S.e[lane];
        } else {
            bg = 0.0;
            bl = l0;
            bc = c0;
            be = 0.0;
        }
        warp_best(bg, bl, bc, be);
    }
}

// ------------------------------------------------------------ tier 0

__global__ void __launch_bounds__(256) k_decide_t0(DecideArgs A, const int32_t *list, int64_t cnt) {
    unsigned long long my_cand = 0;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < cnt;
         q += (int64_t)gridDim.x * blockDim.x) {
        int64_t x = list[q];
        int32_t i = A.subset[x];
        int32_t c_old = A.assign[i];
        int64_t e0 = A.off[i];
        int deg = (int)(A.off[i + 1] - e0);
        int32_t keys[T0_MAXD];
        double vals[T0_MAXD];
        int nc = 0;
#pragma unroll
        for (int t = 0; t < T0_MAXD; t++) {
            if (t < deg) {
                int32_t j = A.nbr[e0 + t];
                if (j != i) {
                    int32_t c = A.assign[j];
                    double w = A.wts[e0 + t];
                    bool found = false;
#pragma unroll
                    for (int s = 0; s < T0_MAXD; s++) {
                        if (s < nc && keys[s] == c) {
                            vals[s] = dadd(vals[s], w);
                            found = true;
                        }
                    }
                    if (!found) {
#pragma unroll
                        for (int s = 0; s < T0_MAXD; s++)
                            if (s == nc) {
                                keys[s] = c;
                                vals[s] = w;  // 0.0 + w
                            }
                        nc++;
                    }
                }
            }
        }
        my_cand += nc;
        double e_old = 0.0;
#pragma unroll
        for (int s = 0; s < T0_MAXD; s++)
            if (s < nc && keys[s] == c_old) e_old = vals[s];
        double ki = A.k[i];
        double a_old_excl = dsub(A.a_tot[c_old], ki);
        double bg = 0.0, be = 0.0;
        int32_t bc = c_old;
        int64_t bl = LBL(A.labels, c_old);
#pragma unroll
        for (int s = 0; s < T0_MAXD; s++) {
            if (s < nc && keys[s] != c_old) {
                int32_t c = keys[s];
                double g = gain_of(vals[s], e_old, A.m, ki, a_old_excl, A.a_tot[c], A.four_m_sq);
                int64_t l = LBL(A.labels, c);
                if (better(g, l, bg, bl)) {
                    bg = g;
                    bl = l;
                    bc = c;
                    be = vals[s];
                }
            }
        }
        finish_vertex(A, x, c_old, e_old, bg, bc, be);
    }
    if (A.cand) {
        typedef cub::BlockReduce<unsigned long long, 256> BR;
        __shared__ typename BR::TempStorage tmp;
        unsigned long long tot = BR(tmp).Sum(my_cand);
        if (threadIdx.x == 0 && tot) atomicAdd(A.cand, tot);
    }
}

// Fold one 32-entry chunk (c, w per lane; c = -1 for none) into a table in
// adjacency order.  wb: the chunk's 32 weights staged in lane order.
__device__ __forceinline__ void fold_chunk(int32_t *keys, double *vals, uint32_t mask, int32_t c,
                                           const double *wb, int lane, int integral) {
    unsigned grp = __match_any_sync(FULL, c);
    if (c >= 0 && lane == __ffs(grp) - 1) {
        uint32_t s = probe_insert(keys, c, mask);
        if (integral) {
            double v = 0.0;
            for (unsigned g = grp; g; g &= g - 1) v = dadd(v, wb[__ffs(g) - 1]);
            atomicAdd(vals + s, v);  // any order is exact for integral weights
        } else {
            double v = vals[s];  // 0.0 when fresh
            for (unsigned g = grp; g; g &= g - 1) v = dadd(v, wb[__ffs(g) - 1]);
            vals[s] = v;
        }
    }
}

// ------------------------------------------------------------ tier 1

__global__ void __launch_bounds__(T1_WARPS * 32) k_decide_t1(DecideArgs A, const int32_t *list,
                                                              int64_t cnt) {
    __shared__ int32_t skeys[T1_WARPS][T1_TS];
    __shared__ double svals[T1_WARPS][T1_TS];
    __shared__ double swb[T1_WARPS][32];
    int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int32_t *keys = skeys[wid];
    double *vals = svals[wid];
    double *wb = swb[wid];
    unsigned long long my_cand = 0;
    for (int64_t q = blockIdx.x * (int64_t)T1_WARPS + wid; q < cnt;
         q += (int64_t)gridDim.x * T1_WARPS) {
        int64_t x = list[q];
        int32_t i = A.subset[x];
        int32_t c_old = A.assign[i];
        int64_t e0 = A.off[i], e1 = A.off[i + 1];
        int deg = (int)(e1 - e0);
        uint32_t ts = 32;
        while (ts < (uint32_t)(deg + deg / 2 + 2)) ts <<= 1;
        uint32_t mask = ts - 1;
        for (uint32_t s = lane; s < ts; s += 32) {
            keys[s] = -1;
            vals[s] = 0.0;
        }
        __syncwarp();
        for (int64_t base = e0; base < e1; base += 32) {
            int64_t e = base + lane;
            int32_t c = -1;
            double w = 0.0;
            if (e < e1) {
                int32_t j = A.nbr[e];
                if (j != i) {
                    c = A.assign[j];
                    w = A.wts[e];
                }
            }
            wb[lane] = w;
            __syncwarp();
            fold_chunk(keys, vals, mask, c, wb, lane, A.integral);
            __syncwarp();
        }
        double e_old = 0.0;
        if (lane == 0) {
            int s = probe_find(keys, c_old, mask);
            e_old = s >= 0 ? vals[s] : 0.0;
        }
        e_old = __shfl_sync(FULL, e_old, 0);
        double ki = A.k[i];
        double a_old_excl = dsub(A.a_tot[c_old], ki);
        double bg = 0.0, be = 0.0;
        int32_t bc = c_old;
        int64_t bl = LBL(A.labels, c_old);
        int nc = 0;
        for (uint32_t s = lane; s < ts; s += 32) {
            int32_t c = keys[s];
            if (c < 0) continue;
            nc++;
            if (c == c_old) continue;
            double g = gain_of(vals[s], e_old, A.m, ki, a_old_excl, A.a_tot[c], A.four_m_sq);
            int64_t l = LBL(A.labels, c);
            if (better(g, l, bg, bl)) {
                bg = g;
                bl = l;
                bc = c;
                be = vals[s];
            }
        }
        warp_best(bg, bl, bc, be);
        my_cand += nc;
        if (lane == 0) finish_vertex(A, x, c_old, e_old, bg, bc, be);
        __syncwarp();
    }
    if (A.cand) {
        for (int o = 16; o > 0; o >>= 1) my_cand += __shfl_xor_sync(FULL, my_cand, o);
        if (lane == 0 && my_cand) atomicAdd(A.cand, my_cand);
    }
}

// ------------------------------------------------------------ tier 2

__global__ void __launch_bounds__(BLK) k_decide_t2(DecideArgs A, const int32_t *list, int64_t cnt) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ int32_t cbuf[BLK];
    __shared__ double wbuf[BLK];
    __shared__ BestSmem bs;
    __shared__ double s_e_old;
    int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    double *vals = reinterpret_cast<double *>(dsm);
    int32_t *keys = reinterpret_cast<int32_t *>(dsm + sizeof(double) * T2_TS);
    unsigned long long my_cand = 0;
    for (int64_t q = blockIdx.x; q < cnt; q += gridDim.x) {
        int64_t x = list[q];
        int32_t i = A.subset[x];
        int32_t c_old = A.assign[i];
        int64_t e0 = A.off[i], e1 = A.off[i + 1];
        int64_t deg = e1 - e0;
        uint32_t ts = 64;
        while (ts < (uint64_t)(deg + deg / 2 + 2)) ts <<= 1;
        uint32_t mask = ts - 1;
        for (uint32_t s = tid; s < ts; s += BLK) {
            keys[s] = -1;
            vals[s] = 0.0;
        }
        __syncthreads();
        for (int64_t base = e0; base < e1; base += BLK) {
            int64_t e = base + tid;
            int32_t c = -1;
            double w = 0.0;
            if (e < e1) {
                int32_t j = A.nbr[e];
                if (j != i) {
                    c = A.assign[j];
                    w = A.wts[e];
                }
            }
            cbuf[tid] = c;
            wbuf[tid] = w;
            __syncthreads();
            if (A.integral) {
                // every warp folds its own sub-chunk; order is irrelevant
                fold_chunk(keys, vals, mask, c, wbuf + wid * 32, lane, 1);
            } else {
                // communities are partitioned over the warps; each warp walks
                // the sub-chunks in order and folds only its own communities,
                // so every community still sees a single in-order left fold
                int nsub = (int)((e1 - base + 31) / 32);
                if (nsub > BLK / 32) nsub = BLK / 32;
                for (int sc = 0; sc < nsub; sc++) {
                    int32_t cc = cbuf[sc * 32 + lane];
                    bool mine = cc >= 0 && (int)(((uint32_t)cc * 0x85EBCA6Bu) >> 29) == wid;
                    if (__any_sync(FULL, mine))
                        fold_chunk(keys, vals, mask, mine ? cc : -1, wbuf + sc * 32, lane, 0);
                    __syncwarp();
                }
            }
            __syncthreads();
        }
        if (tid == 0) {
            int s = probe_find(keys, c_old, mask);
            s_e_old = s >= 0 ? vals[s] : 0.0;
        }
        __syncthreads();
        double e_old = s_e_old;
        double ki = A.k[i];
        double a_old_excl = dsub(A.a_tot[c_old], ki);
        int64_t l_old = LBL(A.labels, c_old);
        double bg = 0.0, be = 0.0;
        int32_t bc = c_old;
        int64_t bl = l_old;
        int nc = 0;
        for (uint32_t s = tid; s < ts; s += BLK) {
            int32_t c = keys[s];
            if (c < 0) continue;
            nc++;
            if (c == c_old) continue;
            double g = gain_of(vals[s], e_old, A.m, ki, a_old_excl, A.a_tot[c], A.four_m_sq);
            int64_t l = LBL(A.labels, c);
            if (better(g, l, bg, bl)) {
                bg = g;
                bl = l;
                bc = c;
                be = vals[s];
            }
        }
        my_cand += nc;
        block_best(bs, bg, bl, bc, be, l_old, c_old);
        if (tid == 0) finish_vertex(A, x, c_old, e_old, bg, bc, be);
        __syncthreads();
    }
    if (A.cand) {
        typedef cub::BlockReduce<unsigned long long, BLK> BR;
        __shared__ typename BR::TempStorage tmp;
        unsigned long long tot = BR(tmp).Sum(my_cand);
        if (threadIdx.x == 0 && tot) atomicAdd(A.cand, tot);
    }
}

// ------------------------------------------------------------ tier 3 (hubs)

// key = (hub << cb) | community, val = entry index within the hub row.  A
// self-loop entry gets the community id `nskip` (>= n) and is ignored.
__global__ void k_hub_keys(DecideArgs A, const int32_t *list, const int64_t *eoff, int64_t nh,
                           int64_t E, int cb, int32_t nskip, uint64_t *key, int32_t *val) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < E;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = nh;  // largest q with eoff[q] <= t
        while (hi - lo > 1) {
            int64_t mid = (lo + hi) >> 1;
            if (eoff[mid] <= t)
                lo = mid;
            else
                hi = mid;
        }
        int32_t i = A.subset[list[lo]];
        int64_t loc = t - eoff[lo];
        int32_t j = A.nbr[A.off[i] + loc];
        int32_t c = (j == i) ? nskip : A.assign[j];
        key[t] = ((uint64_t)lo << cb) | (uint32_t)c;
        val[t] = (int32_t)loc;
    }
}

// Sequential fold of the run starting at sorted position p: every entry of
// one community of the hub row starting at e0, in adjacency order.  Loads are
// batched eight at a time so only the additions form the dependency chain.
__device__ __forceinline__ double fold_hub_run(const uint64_t *key, const int32_t *val,
                                               const double *wts, int64_t e0, int64_t p,
                                               int64_t hi) {
    const uint64_t k0 = key[p];
    double v = 0.0;
    while (true) {
        double w[8];
        bool ok[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            int64_t q = p + u;
            ok[u] = q < hi && key[q] == k0;
            w[u] = ok[u] ? wts[e0 + val[q]] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
            if (!ok[u]) return v;
            v = dadd(v, w[u]);
        }
        p += 8;
    }
}

// Largest hub q with eoff[q] <= t.
__device__ __forceinline__ int64_t hub_of(const int64_t *eoff, int64_t nh, int64_t t) {
    int64_t lo = 0, hi = nh;
    while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if (eoff[mid] <= t)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

// Sorted range [a, b) of hub q's entries with key `want`.
__device__ __forceinline__ void key_range(const uint64_t *key, int64_t lo, int64_t hi,
                                          uint64_t want, int64_t *a_out, int64_t *b_out) {
    int64_t a = lo, b = hi;
    while (a < b) {
        int64_t mid = (a + b) >> 1;
        if (key[mid] < want)
            a = mid + 1;
        else
            b = mid;
    }
    int64_t c = a, d = hi;
    while (c < d) {
        int64_t mid = (c + d) >> 1;
        if (key[mid] <= want)
            c = mid + 1;
        else
            d = mid;
    }
    *a_out = a;
    *b_out = c;
}

constexpr int SHORT_RUN = 32;  // longer runs are folded by a whole block

// e_{i->c_old} of every hub: its c_old run, one block per hub.
__global__ void __launch_bounds__(BLK) k_hub_eold(DecideArgs A, const int32_t *list,
                                                 const int64_t *eoff, const uint64_t *key,
                                                 const int32_t *val, int cb, double *eold) {
    __shared__ double sb[2 * FOLD_CH];
    __shared__ int64_t s_a, s_b;
    const int64_t q = blockIdx.x;
    const int32_t i = A.subset[list[q]];
    const int32_t c_old = A.assign[i];
    if (threadIdx.x == 0) {
        int64_t a, b;
        key_range(key, eoff[q], eoff[q + 1], ((uint64_t)q << cb) | (uint32_t)c_old, &a, &b);
        s_a = a;
        s_b = b;
    }
    __syncthreads();
    const int64_t a = s_a, len = s_b - s_a, e0 = A.off[i];
    const double *wts = A.wts;
    double v = block_fold([=] __device__(int64_t t) { return wts[e0 + val[a + t]]; }, len, 0.0,
                          sb);
    if (threadIdx.x == 0) eold[q] = v;
}

// One thread per sorted position: heads of short runs fold their community
// and compute its gain (all hubs of the stage at once); heads of long runs go
// to a worklist for k_hub_long; every other position is marked -inf.
__global__ void k_hub_runs(DecideArgs A, const int32_t *list, const int64_t *eoff, int64_t nh,
                           int64_t E, const uint64_t *key, const int32_t *val, int cb,
                           int32_t nskip, const double *eold, double *rgain, int32_t *rc,
                           double *rv, int64_t *lrun, unsigned long long *lcnt) {
    const uint64_t cmask = (1ull << cb) - 1ull;
    unsigned long long nc = 0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < E;
         p += (int64_t)gridDim.x * blockDim.x) {
        uint64_t kk = key[p];
        int64_t q = (int64_t)(kk >> cb);
        int32_t c = (int32_t)(kk & cmask);
        double g = -INFINITY;
        bool head = (p == eoff[q]) || key[p - 1] != kk;
        if (head && c != nskip) {
            nc++;
            int32_t i = A.subset[list[q]];
            int32_t c_old = A.assign[i];
            int64_t hi = eoff[q + 1];
            if (c != c_old) {
                if (p + SHORT_RUN < hi && key[p + SHORT_RUN] == kk) {
                    lrun[atomicAdd(lcnt, 1ull)] = p;
                } else {
                    double v = fold_hub_run(key, val, A.wts, A.off[i], p, hi);
                    double ki = A.k[i];
                    g = gain_of(v, eold[q], A.m, ki, dsub(A.a_tot[c_old], ki), A.a_tot[c],
                                A.four_m_sq);
                    rv[p] = v;
                }
            }
        }
        rgain[p] = g;
        rc[p] = c;
    }
    if (A.cand) {
        typedef cub::BlockReduce<unsigned long long, 256> BR;
        __shared__ typename BR::TempStorage tmp;
        unsigned long long tot = BR(tmp).Sum(nc);
        if (threadIdx.x == 0 && tot) atomicAdd(A.cand, tot);
    }
}

// Long runs: one block each (block-staged ordered fold), then the gain.
__global__ void __launch_bounds__(BLK) k_hub_long(DecideArgs A, const int32_t *list,
                                                 const int64_t *eoff, const uint64_t *key,
                                                 const int32_t *val, int cb, const double *eold,
                                                 const int64_t *lrun,
                                                 const unsigned long long *lcnt, double *rgain,
                                                 double *rv) {
    __shared__ double sb[2 * FOLD_CH];
    __shared__ int64_t s_b;
    const int64_t cnt = (int64_t)*lcnt;
    const uint64_t cmask = (1ull << cb) - 1ull;
    for (int64_t w = blockIdx.x; w < cnt; w += gridDim.x) {
        const int64_t p = lrun[w];
        const uint64_t kk = key[p];
        const int64_t q = (int64_t)(kk >> cb);
        const int32_t c = (int32_t)(kk & cmask);
        const int32_t i = A.subset[list[q]];
        if (threadIdx.x == 0) {
            int64_t a, b;
            key_range(key, p, eoff[q + 1], kk, &a, &b);
            s_b = b;
        }
        __syncthreads();
        const int64_t len = s_b - p, e0 = A.off[i];
        const double *wts = A.wts;
        double v = block_fold([=] __device__(int64_t t) { return wts[e0 + val[p + t]]; }, len,
                              0.0, sb);
        if (threadIdx.x == 0) {
            int32_t c_old = A.assign[i];
            double ki = A.k[i];
            rgain[p] = gain_of(v, eold[q], A.m, ki, dsub(A.a_tot[c_old], ki), A.a_tot[c],
                               A.four_m_sq);
            rv[p] = v;
        }
        __syncthreads();
    }
}

// Block per hub: argmax over its run candidates, then the decision.
__global__ void __launch_bounds__(BLK) k_hub_final(DecideArgs A, const int32_t *list,
                                                  const int64_t *eoff, const double *eold,
                                                  const double *rgain, const int32_t *rc,
                                                  const double *rv) {
    __shared__ BestSmem bs;
    const int64_t q = blockIdx.x;
    const int64_t x = list[q];
    const int32_t c_old = A.assign[A.subset[x]];
    const int64_t l_old = LBL(A.labels, c_old);
    double bg = 0.0, be = 0.0;
    int32_t bc = c_old;
    int64_t bl = l_old;
    for (int64_t p = eoff[q] + threadIdx.x; p < eoff[q + 1]; p += BLK) {
        double g = rgain[p];
        if (g == -INFINITY) continue;
        int32_t c = rc[p];
        int64_t l = LBL(A.labels, c);
        if (better(g, l, bg, bl)) {
            bg = g;
            bl = l;
            bc = c;
            be = rv[p];
        }
    }
    block_best(bs, bg, bl, bc, be, l_old, c_old);
    if (threadIdx.x == 0) finish_vertex(A, x, c_old, eold[q], bg, bc, be);
}

// ================================================================ planning

__global__ void k_tier_keys(const int64_t *off, const int32_t *vtx, const int64_t *stage_off,
                            int64_t nst, int64_t total, uint32_t *key, unsigned long long *hist) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        int64_t a = 0, b = nst;  // stage: largest s with stage_off[s] <= g
        while (b - a > 1) {
            int64_t mid = (a + b) >> 1;
            if (stage_off[mid] <= g)
                a = mid;
            else
                b = mid;
        }
        int32_t i = vtx[g];
        int64_t d = off[i + 1] - off[i];
        uint32_t t = d <= T0_MAXD ? 0 : d <= T1_MAXD ? 1 : d <= T2_MAXD ? 2 : 3;
        uint32_t kk = (uint32_t)(a * 4 + t);
        key[g] = kk;
        atomicAdd(hist + kk, 1ull);
    }
}

__global__ void k_tier_local(const uint32_t *skey, const int32_t *sidx, const int64_t *stage_off,
                             int64_t total, int32_t *local) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < total;
         p += (int64_t)gridDim.x * blockDim.x)
        local[p] = (int32_t)(sidx[p] - stage_off[skey[p] >> 2]);
}

__global__ void k_hub_degrees(const int64_t *off, const int32_t *vtx, const int64_t *stage_off,
                              const int32_t *local, const int64_t *hub_pos, const int64_t *hub_stage,
                              int64_t nh, int64_t *deg) {
    for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < nh;
         h += (int64_t)gridDim.x * blockDim.x) {
        int32_t i = vtx[stage_off[hub_stage[h]] + local[hub_pos[h]]];
        deg[h] = off[i + 1] - off[i];
    }
}

void Plan::release() {
    void *ps[] = {tier_list, hub_eoff, hkey, hkey2, hval, hval2, htmp, heold, rgain, rc, rv,
                  lrun, lcnt};
    for (void *p : ps)
        if (p) cudaFree(p);
    heold = rgain = rv = nullptr;
    lrun = nullptr;
    lcnt = nullptr;
    rc = nullptr;
    tier_list = nullptr;
    hub_eoff = nullptr;
    hkey = hkey2 = nullptr;
    hval = hval2 = nullptr;
    htmp = nullptr;
}

void plan_build(Plan &P, const int64_t *off, const int32_t *vtx, const int64_t *stage_off_h,
                int64_t nst, int64_t n, cudaStream_t s) {
    int64_t total = stage_off_h[nst];
    P.st.assign(nst, StagePlan{});
    for (int64_t a = 0; a < nst; a++) {
        P.st[a].off = stage_off_h[a];
        P.st[a].ns = stage_off_h[a + 1] - stage_off_h[a];
    }
    P.cb = bits_for(n + 2);
    P.nskip = (int32_t)n;
    P.tier_list = dalloc<int32_t>(total);
    if (total == 0) return;
    Buf<int64_t> d_soff(nst + 1, s);
    PLV_CUDA(cudaMemcpyAsync(d_soff.get(), stage_off_h, sizeof(int64_t) * (nst + 1),
                             cudaMemcpyHostToDevice, s));
    Buf<uint32_t> key(total, s), skey(total, s);
    Buf<int32_t> gidx(total, s), sidx(total, s);
    Buf<unsigned long long> hist(4 * nst, s);
    PLV_CUDA(cudaMemsetAsync(hist.get(), 0, sizeof(unsigned long long) * 4 * nst, s));
    k_tier_keys<<<grid_for(total, 256), 256, 0, s>>>(off, vtx, d_soff, nst, total, key, hist);
    PLV_LAUNCH_CHECK();
    iota_i32(gidx, total, s);
    sort_pairs<uint32_t, int32_t>(key, skey, gidx, sidx, total, 0, bits_for(4 * nst + 4), s);
    k_tier_local<<<grid_for(total, 256), 256, 0, s>>>(skey, sidx, d_soff, total, P.tier_list);
    PLV_LAUNCH_CHECK();
    std::vector<unsigned long long> h(4 * nst);
    PLV_CUDA(cudaMemcpyAsync(h.data(), hist.get(), sizeof(unsigned long long) * 4 * nst,
                             cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    int64_t pos = 0;
    std::vector<int64_t> hub_pos, hub_stage;
    for (int64_t a = 0; a < nst; a++)
        for (int t = 0; t < 4; t++) {
            P.st[a].tstart[t] = pos;
            P.st[a].tcount[t] = (int64_t)h[4 * a + t];
            if (t == 3)
                for (int64_t z = 0; z < P.st[a].tcount[3]; z++) {
                    hub_pos.push_back(pos + z);
                    hub_stage.push_back(a);
                }
            pos += (int64_t)h[4 * a + t];
        }
    int64_t nh = (int64_t)hub_pos.size();
    if (nh == 0) return;
    Buf<int64_t> d_hpos(nh, s), d_hst(nh, s), d_deg(nh, s);
    PLV_CUDA(cudaMemcpyAsync(d_hpos.get(), hub_pos.data(), sizeof(int64_t) * nh,
                             cudaMemcpyHostToDevice, s));
    PLV_CUDA(cudaMemcpyAsync(d_hst.get(), hub_stage.data(), sizeof(int64_t) * nh,
                             cudaMemcpyHostToDevice, s));
    k_hub_degrees<<<grid_for(nh, 256), 256, 0, s>>>(off, vtx, d_soff, P.tier_list, d_hpos, d_hst,
                                                   nh, d_deg);
    PLV_LAUNCH_CHECK();
    std::vector<int64_t> deg(nh);
    PLV_CUDA(cudaMemcpyAsync(deg.data(), d_deg.get(), sizeof(int64_t) * nh, cudaMemcpyDeviceToHost,
                             s));
    PLV_CUDA(cudaStreamSynchronize(s));
    std::vector<int64_t> eoff;
    int64_t h0 = 0;
    for (int64_t a = 0; a < nst; a++) {
        StagePlan &sp = P.st[a];
        sp.hub_base = (int64_t)eoff.size();
        int64_t acc = 0;
        eoff.push_back(0);
        for (int64_t z = 0; z < sp.tcount[3]; z++) {
            acc += deg[h0 + z];
            eoff.push_back(acc);
        }
        h0 += sp.tcount[3];
        sp.hub_entries = acc;
        P.max_hub_entries = acc > P.max_hub_entries ? acc : P.max_hub_entries;
        P.max_hubs = sp.tcount[3] > P.max_hubs ? sp.tcount[3] : P.max_hubs;
    }
    P.hub_eoff = dalloc<int64_t>(eoff.size());
    PLV_CUDA(cudaMemcpyAsync(P.hub_eoff, eoff.data(), sizeof(int64_t) * eoff.size(),
                             cudaMemcpyHostToDevice, s));
    P.qb = bits_for(P.max_hubs + 1);
    int64_t E = P.max_hub_entries;
    P.hkey = dalloc<uint64_t>(E);
    P.hkey2 = dalloc<uint64_t>(E);
    P.hval = dalloc<int32_t>(E);
    P.hval2 = dalloc<int32_t>(E);
    P.heold = dalloc<double>(P.max_hubs);
    P.rgain = dalloc<double>(E);
    P.rc = dalloc<int32_t>(E);
    P.rv = dalloc<double>(E);
    P.lrun = dalloc<int64_t>(E);
    P.lcnt = dalloc<unsigned long long>(1);
    PLV_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, P.hbytes, P.hkey, P.hkey2, P.hval, P.hval2,
                                             E, 0, P.cb + P.qb, s));
    PLV_CUDA(cudaMalloc(&P.htmp, P.hbytes ? P.hbytes : 1));
    PLV_CUDA(cudaStreamSynchronize(s));
}

void ensure_decide_attrs() {
    static int dev_done = -1;
    int dev;
    PLV_CUDA(cudaGetDevice(&dev));
    if (dev_done == dev) return;
    PLV_CUDA(cudaFuncSetAttribute(k_decide_t2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)T2_SMEM));
    dev_done = dev;
}

void launch_decide(const Plan &P, int64_t a, DecideArgs A, cudaStream_t st) {
    const StagePlan &sp = P.st[a];
    if (sp.tcount[0]) {
        k_decide_t0<<<grid_for(sp.tcount[0], 256), 256, 0, st>>>(A, P.tier_list + sp.tstart[0],
                                                                 sp.tcount[0]);
        PLV_LAUNCH_CHECK();
    }
    if (sp.tcount[1]) {
        k_decide_t1<<<grid_for(sp.tcount[1], T1_WARPS), T1_WARPS * 32, 0, st>>>(
            A, P.tier_list + sp.tstart[1], sp.tcount[1]);
        PLV_LAUNCH_CHECK();
    }
    if (sp.tcount[2]) {
        k_decide_t2<<<grid_for(sp.tcount[2], 1, 148 * 8), BLK, T2_SMEM, st>>>(
            A, P.tier_list + sp.tstart[2], sp.tcount[2]);
        PLV_LAUNCH_CHECK();
    }
    if (sp.tcount[3]) {
        const int32_t *list = P.tier_list + sp.tstart[3];
        const int64_t *eoff = P.hub_eoff + sp.hub_base;
        int64_t E = sp.hub_entries;
        k_hub_keys<<<grid_for(E, 256), 256, 0, st>>>(A, list, eoff, sp.tcount[3], E, P.cb, P.nskip,
                                                     P.hkey, P.hval);
        PLV_LAUNCH_CHECK();
        size_t bytes = P.hbytes;
        PLV_CUDA(cub::DeviceRadixSort::SortPairs(P.htmp, bytes, P.hkey, P.hkey2, P.hval, P.hval2, E,
                                                 0, P.cb + P.qb, st));
        int64_t nh = sp.tcount[3];
        k_hub_eold<<<(unsigned)nh, BLK, 0, st>>>(A, list, eoff, P.hkey2, P.hval2, P.cb, P.heold);
        PLV_LAUNCH_CHECK();
        PLV_CUDA(cudaMemsetAsync(P.lcnt, 0, sizeof(unsigned long long), st));
        k_hub_runs<<<grid_for(E, 256), 256, 0, st>>>(A, list, eoff, nh, E, P.hkey2, P.hval2, P.cb,
                                                     P.nskip, P.heold, P.rgain, P.rc, P.rv, P.lrun,
                                                     P.lcnt);
        PLV_LAUNCH_CHECK();
        k_hub_long<<<148 * 2, BLK, 0, st>>>(A, list, eoff, P.hkey2, P.hval2, P.cb, P.heold, P.lrun,
                                            P.lcnt, P.rgain, P.rv);
        PLV_LAUNCH_CHECK();
        k_hub_final<<<(unsigned)nh, BLK, 0, st>>>(A, list, eoff, P.heold, P.rgain, P.rc, P.rv);
        PLV_LAUNCH_CHECK();
    }
}

DecideArgs make_decide_args(const int64_t *off, const int32_t *nbr, const double *wts,
                            const double *k, const int32_t *labels, const int32_t *subset,
                            const int32_t *assign, const double *a_tot, const int32_t *sizes,
                            double m, int integral, int32_t *out_target, uint8_t *out_moved,
                            double *out_e_old, double *out_e_best, unsigned long long *cand) {
    DecideArgs A;
    A.off = off;
    A.nbr = nbr;
    A.wts = wts;
    A.k = k;
    A.labels = labels;
    A.subset = subset;
    A.assign = assign;
    A.a_tot = a_tot;
    A.sizes = sizes;
    A.m = m;
    A.four_m_sq = (2.0 * m) * (2.0 * m);
    A.integral = integral;
    A.out_target = out_target;
    A.out_moved = out_moved;
    A.out_e_old = out_e_old;
    A.out_e_best = out_e_best;
    A.cand = cand;
    return A;
}

// One-off decide over `subset` (plans a single stage, then synchronises).
static void decide_once(const int64_t *off, const int32_t *nbr, const double *wts,
                        const double *k, const int32_t *labels, const int32_t *subset, int64_t ns,
                        const int32_t *assign, const double *a_tot, const int32_t *sizes,
                        double m, int integral, int32_t *out_target, uint8_t *out_moved,
                        double *out_e_old, double *out_e_best, int64_t *cand_h, cudaStream_t s) {
    if (cand_h) *cand_h = 0;
    if (ns <= 0) return;
    ensure_decide_attrs();
    // community ids are vertex ids of the graph: < 2^31 - 2 is enough for the
    // hub keys' community field
    const int64_t n_bound = (int64_t)INT32_MAX - 2;
    Plan P;
    int64_t soff[2] = {0, ns};
    Buf<unsigned long long> cand(1, s);
    PLV_CUDA(cudaMemsetAsync(cand.get(), 0, sizeof(unsigned long long), s));
    try {
        plan_build(P, off, subset, soff, 1, n_bound, s);
        DecideArgs A = make_decide_args(off, nbr, wts, k, labels, subset, assign, a_tot, sizes, m,
                                        integral, out_target, out_moved, out_e_old, out_e_best,
                                        cand.get());
        launch_decide(P, 0, A, s);
        if (cand_h) *cand_h = (int64_t)d2h(cand.get(), s);
        PLV_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
        cudaStreamSynchronize(s);
        P.release();
        throw;
    }
    P.release();
}

}  // namespace plv

extern "C" int plv_decide(const int64_t *off, const int32_t *nbr, const double *wts,
                          const double *k, const int32_t *labels, const int32_t *subset,
                          int64_t ns, const int32_t *assign, const double *a_tot,
                          const int32_t *sizes, double m, int32_t *out_target, uint8_t *out_moved,
                          double *out_e_old, double *out_e_best, int64_t *cand_h, void *stream) {
    PLV_ENTRY
    if (!(m > 0.0)) PLV_FAIL(PLV_EINVAL, "modularity undefined for edgeless graph");
    plv::decide_once(off, nbr, wts, k, labels, subset, ns, assign, a_tot, sizes, m, 0, out_target,
                     out_moved, out_e_old, out_e_best, cand_h, plv::S(stream));
    PLV_EXIT
}

extern "C" int plv_decide_ex(const int64_t *off, const int32_t *nbr, const double *wts,
                             const double *k, const int32_t *labels, const int32_t *subset,
                             int64_t ns, const int32_t *assign, const double *a_tot,
                             const int32_t *sizes, double m, int flags, int32_t *out_target,
                             uint8_t *out_moved, double *out_e_old, double *out_e_best,
                             int64_t *cand_h, void *stream) {
    PLV_ENTRY
    if (!(m > 0.0)) PLV_FAIL(PLV_EINVAL, "modularity undefined for edgeless graph");
    plv::decide_once(off, nbr, wts, k, labels, subset, ns, assign, a_tot, sizes, m,
                     (flags & PLV_F_INTEGRAL) ? 1 : 0, out_target, out_moved, out_e_old,
                     out_e_best, cand_h, plv::S(stream));
    PLV_EXIT
}
