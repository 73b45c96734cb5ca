// localmove.cu -- the local-moving hot kernel: decide_moves + apply_moves.
//
// decide (PL/_kernels.pyx:21-101): every subset vertex i aggregates
// e_{i->C} over its neighbours j != i by snapshot community, summed in
// adjacency order per community (fp64, bit-exact with the reference's hash
// accumulation), then takes the argmax of the Eq. 4 gain under (gain desc,
// label asc) with the singleton-pair guard.  Vertices are degree-binned:
//   tier 0  deg <= 8      thread per vertex, candidate list in registers
//   tier 1  deg <= 128    warp per vertex, hash table in shared memory
//   tier 2  deg <= 2048   block per vertex, hash table in shared memory
//   tier 3  larger        block per vertex, hash table in a global slab
// Within a 32-entry chunk, lanes with the same community are grouped with
// __match_any_sync and the group leader folds their weights in lane order
// (= adjacency order); chunks are processed in order, so every community's
// sum is the sequential left fold of the reference.  Integral graphs (every
// weight an integer, total < 2^52) may fold in any order and use atomics.
//
// apply (PL/_kernels.pyx:104-145) is restated in parallel, bit-exactly:
// e_a / e_b of a moved vertex use the *live* assignment, i.e. the target of
// an earlier-moved subset vertex or else the snapshot; the per-community
// updates of a_tot / w_internal are then folded in subset order by one thread
// per community after a stable sort of the (community, subset position)
// events.  sizes are integers (atomics), the assignment is scattered.
#include "common.cuh"
#include "csr.cuh"
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <vector>

namespace plv {

constexpr unsigned FULL = 0xffffffffu;
constexpr int T0_MAXD = 8;
constexpr int T1_MAXD = 128;
constexpr int T2_MAXD = 2048;
constexpr int T1_WARPS = 8;        // warps per block in tier 1
constexpr int T1_TS = 256;         // slots per warp table (>= 1.5 * (128 + 1))
constexpr int BLK = 256;           // threads per block in tiers 2/3
constexpr int T2_TS = 4096;        // smem slots for tier 2 (>= 1.5 * (2048 + 1))

struct DecideArgs {
    const int64_t *off;
    const int32_t *nbr;
    const double *wts;
    const double *k;
    const int32_t *labels;
    const int32_t *subset;
    const int32_t *assign;
    const double *a_tot;
    const int32_t *sizes;
    double m, four_m_sq;
    int integral;
    int32_t *out_target;
    uint8_t *out_moved;
    double *out_e_old;
    double *out_e_best;
    unsigned long long *cand;
};

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

// Find-or-insert c; tables are cleared to key -1 / value 0.0.
__device__ __forceinline__ uint32_t probe_insert(int32_t *keys, int32_t c, uint32_t mask,
                                                 bool *fresh) {
    uint32_t s = hslot(c, mask);
    while (true) {
        int32_t k = keys[s];
        if (k == c) {
            *fresh = false;
            return s;
        }
        if (k == -1) {
            int32_t old = atomicCAS(keys + s, -1, c);
            if (old == -1) {
                *fresh = true;
                return s;
            }
            if (old == c) {
                *fresh = false;
                return s;
            }
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

// Fold one 32-entry chunk (c, w per lane, c = -1 for none) into a table in
// adjacency order.  wb: 32 staged weights of this chunk (lane order).
__device__ __forceinline__ void fold_chunk(int32_t *keys, double *vals, uint32_t mask, int32_t c,
                                           const double *wb, int lane, int integral) {
    unsigned grp = __match_any_sync(FULL, c);
    int leader = __ffs(grp) - 1;
    if (c >= 0 && lane == leader) {
        bool fresh;
        uint32_t s = probe_insert(keys, c, mask, &fresh);
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

// ------------------------------------------------------------ tiers 2 / 3

// Block per vertex.  GLOBAL: tables live in a per-block global slab of `cap`
// slots (kept clean between vertices through the candidate list).
template <bool GLOBAL>
__global__ void __launch_bounds__(BLK) k_decide_blk(DecideArgs A, const int32_t *list, int64_t cnt,
                                                   int32_t *gkeys, double *gvals, int32_t *gcand,
                                                   int64_t cap) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ int32_t cbuf[BLK];
    __shared__ double wbuf[BLK];
    __shared__ double rg[BLK / 32];
    __shared__ int64_t rl[BLK / 32];
    __shared__ int32_t rc[BLK / 32];
    __shared__ double re[BLK / 32];
    __shared__ double s_e_old;
    __shared__ int s_ncand;
    int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    int32_t *keys;
    double *vals;
    int32_t *cands = nullptr;
    if (GLOBAL) {
        keys = gkeys + blockIdx.x * cap;
        vals = gvals + blockIdx.x * cap;
        cands = gcand + blockIdx.x * cap;
    } else {
        vals = reinterpret_cast<double *>(dsm);
        keys = reinterpret_cast<int32_t *>(dsm + sizeof(double) * T2_TS);
    }
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
        if (!GLOBAL) {
            for (uint32_t s = tid; s < ts; s += BLK) {
                keys[s] = -1;
                vals[s] = 0.0;
            }
        }
        if (tid == 0) s_ncand = 0;
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
                unsigned grp = __match_any_sync(FULL, c);
                if (c >= 0 && lane == __ffs(grp) - 1) {
                    bool fresh;
                    uint32_t s = probe_insert(keys, c, mask, &fresh);
                    if (GLOBAL && fresh) cands[atomicAdd(&s_ncand, 1)] = (int32_t)s;
                    double v = 0.0;
                    for (unsigned g = grp; g; g &= g - 1) v = dadd(v, wbuf[wid * 32 + __ffs(g) - 1]);
                    atomicAdd(vals + s, v);
                }
            } else if (wid == 0) {
                // one warp folds the sub-chunks in order: exact left folds
                int nsub = (int)((e1 - base + 31) / 32);
                if (nsub > BLK / 32) nsub = BLK / 32;
                for (int sc = 0; sc < nsub; sc++) {
                    int32_t cc = cbuf[sc * 32 + lane];
                    unsigned grp = __match_any_sync(FULL, cc);
                    if (cc >= 0 && lane == __ffs(grp) - 1) {
                        bool fresh;
                        uint32_t s = probe_insert(keys, cc, mask, &fresh);
                        if (GLOBAL && fresh) cands[atomicAdd(&s_ncand, 1)] = (int32_t)s;
                        double v = vals[s];
                        for (unsigned g = grp; g; g &= g - 1) v = dadd(v, wbuf[sc * 32 + __ffs(g) - 1]);
                        vals[s] = v;
                    }
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
        double bg = 0.0, be = 0.0;
        int32_t bc = c_old;
        int64_t bl = LBL(A.labels, c_old);
        int nc = 0;
        int64_t scan_n = GLOBAL ? (int64_t)s_ncand : (int64_t)ts;
        for (int64_t t = tid; t < scan_n; t += BLK) {
            uint32_t s = GLOBAL ? (uint32_t)cands[t] : (uint32_t)t;
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
        warp_best(bg, bl, bc, be);
        if (lane == 0) {
            rg[wid] = bg;
            rl[wid] = bl;
            rc[wid] = bc;
            re[wid] = be;
        }
        __syncthreads();
        if (wid == 0) {
            if (lane < BLK / 32) {
                bg = rg[lane];
                bl = rl[lane];
                bc = rc[lane];
                be = re[lane];
            } else {
                bg = 0.0;
                bl = LBL(A.labels, c_old);
                bc = c_old;
                be = 0.0;
            }
            warp_best(bg, bl, bc, be);
            if (lane == 0) finish_vertex(A, x, c_old, e_old, bg, bc, be);
        }
        if (GLOBAL) {
            // restore the slab to empty through the candidate list
            for (int64_t t = tid; t < scan_n; t += BLK) {
                uint32_t s = (uint32_t)cands[t];
                keys[s] = -1;
                vals[s] = 0.0;
            }
        }
        __syncthreads();
    }
    if (A.cand) {
        typedef cub::BlockReduce<unsigned long long, BLK> BR;
        __shared__ typename BR::TempStorage tmp;
        unsigned long long tot = BR(tmp).Sum(my_cand);
        if (threadIdx.x == 0 && tot) atomicAdd(A.cand, tot);
    }
}

// ------------------------------------------------------------ binning

__global__ void k_bin(const int64_t *off, const int32_t *subset, int64_t ns, int32_t *lists,
                      int64_t stride, unsigned long long *cnt, unsigned long long *maxdeg) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < ns;
         x += (int64_t)gridDim.x * blockDim.x) {
        int32_t i = subset[x];
        int64_t d = off[i + 1] - off[i];
        int t = d <= T0_MAXD ? 0 : d <= T1_MAXD ? 1 : d <= T2_MAXD ? 2 : 3;
        unsigned long long p = atomicAdd(cnt + t, 1ull);
        lists[t * stride + p] = (int32_t)x;
        if (t == 3) atomicMax(maxdeg, (unsigned long long)d);
    }
}

// Persistent zero-initialised hub slab (keys -1, vals 0), grown on demand.
struct HubSlab {
    int dev = -1;
    int32_t *keys = nullptr;
    double *vals = nullptr;
    int32_t *cands = nullptr;
    int64_t slots = 0;
};
static HubSlab g_slab;

__global__ void k_fill_i32(int32_t *p, int64_t n, int32_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

static void ensure_slab(int64_t slots, cudaStream_t s) {
    int dev;
    PLV_CUDA(cudaGetDevice(&dev));
    if (g_slab.dev == dev && g_slab.slots >= slots) return;
    if (g_slab.keys) {
        PLV_CUDA(cudaStreamSynchronize(s));
        cudaFree(g_slab.keys);
        cudaFree(g_slab.vals);
        cudaFree(g_slab.cands);
    }
    g_slab = HubSlab{};
    PLV_CUDA(cudaMalloc(&g_slab.keys, sizeof(int32_t) * slots));
    PLV_CUDA(cudaMalloc(&g_slab.vals, sizeof(double) * slots));
    PLV_CUDA(cudaMalloc(&g_slab.cands, sizeof(int32_t) * slots));
    k_fill_i32<<<grid_for(slots, 256), 256, 0, s>>>(g_slab.keys, slots, -1);
    PLV_LAUNCH_CHECK();
    PLV_CUDA(cudaMemsetAsync(g_slab.vals, 0, sizeof(double) * slots, s));
    g_slab.dev = dev;
    g_slab.slots = slots;
}

void decide(const int64_t *off, const int32_t *nbr, const double *wts, const double *k,
            const int32_t *labels, const int32_t *subset, int64_t ns, const int32_t *assign,
            const double *a_tot, const int32_t *sizes, double m, int integral, int32_t *out_target,
            uint8_t *out_moved, double *out_e_old, double *out_e_best, int64_t *cand_h,
            cudaStream_t s) {
    if (ns <= 0) {
        if (cand_h) *cand_h = 0;
        return;
    }
    Buf<int32_t> lists(4 * ns, s);
    Buf<unsigned long long> cnt(6, s);
    PLV_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(unsigned long long) * 6, s));
    k_bin<<<grid_for(ns, 256), 256, 0, s>>>(off, subset, ns, lists, ns, cnt, cnt.get() + 4);
    PLV_LAUNCH_CHECK();
    unsigned long long c[6];
    PLV_CUDA(cudaMemcpyAsync(c, cnt.get(), sizeof(c), cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
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
    A.cand = cand_h ? cnt.get() + 5 : nullptr;
    if (c[0]) {
        k_decide_t0<<<grid_for(c[0], 256), 256, 0, s>>>(A, lists.get(), c[0]);
        PLV_LAUNCH_CHECK();
    }
    if (c[1]) {
        k_decide_t1<<<grid_for(c[1], T1_WARPS), T1_WARPS * 32, 0, s>>>(A, lists.get() + ns, c[1]);
        PLV_LAUNCH_CHECK();
    }
    if (c[2]) {
        size_t smem = (sizeof(double) + sizeof(int32_t)) * T2_TS;
        static bool attr = false;
        if (!attr) {
            PLV_CUDA(cudaFuncSetAttribute(k_decide_blk<false>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr = true;
        }
        k_decide_blk<false><<<grid_for(c[2], 1, 148 * 8), BLK, smem, s>>>(
            A, lists.get() + 2 * ns, c[2], nullptr, nullptr, nullptr, 0);
        PLV_LAUNCH_CHECK();
    }
    if (c[3]) {
        int64_t md = (int64_t)c[4];
        int64_t cap = 64;
        while (cap < md + md / 2 + 2) cap <<= 1;
        int64_t blocks = (int64_t)c[3] < 148 * 2 ? (int64_t)c[3] : 148 * 2;
        // keep the slab under ~2 GiB
        while (blocks > 1 && blocks * cap * 16 > (2ll << 30)) blocks >>= 1;
        ensure_slab(blocks * cap, s);
        k_decide_blk<true><<<(unsigned)blocks, BLK, 0, s>>>(A, lists.get() + 3 * ns, c[3],
                                                            g_slab.keys, g_slab.vals,
                                                            g_slab.cands, cap);
        PLV_LAUNCH_CHECK();
    }
    if (cand_h) *cand_h = (int64_t)d2h(cnt.get() + 5, s);
}

// ================================================================== apply

struct ApplyArgs {
    const int64_t *off;
    const int32_t *nbr;
    const double *wts;
    const double *k;
    const double *selfw;
    const int32_t *subset;
    const int32_t *target;
    const uint8_t *moved;
    const double *e_old;
    const double *e_best;
    const int32_t *pos;  // subset position per vertex (-1 if absent), general mode
    int flags;
    const int32_t *assign;  // snapshot (unchanged until the scatter)
    double *a_tot;
    double *w_int;
    int32_t *sizes;
    double *ea;  // per subset index
    double *eb;
    unsigned long long *count;
};

// live community of neighbour j for the mover at subset index x
__device__ __forceinline__ int32_t live_comm(const ApplyArgs &A, int32_t j, int64_t x) {
    int64_t p;
    if (A.flags & PLV_F_IDENTITY)
        p = j;
    else
        p = A.pos[j];
    if (p >= 0 && p < x && A.moved[p]) return A.target[p];
    return A.assign[j];
}

__global__ void k_apply_edges(ApplyArgs A, int64_t ns) {
    unsigned long long mine = 0;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < ns;
         x += (int64_t)gridDim.x * blockDim.x) {
        if (!A.moved[x]) continue;
        int32_t i = A.subset[x];
        int32_t a = A.assign[i], b = A.target[x];
        if (a == b) continue;
        mine++;
        double e_a, e_b;
        if (A.flags & PLV_F_INDEPENDENT) {
            e_a = A.e_old[x];
            e_b = A.e_best[x];
        } else {
            e_a = 0.0;
            e_b = 0.0;
            for (int64_t e = A.off[i]; e < A.off[i + 1]; e++) {
                int32_t j = A.nbr[e];
                if (j == i) continue;
                int32_t c = live_comm(A, j, x);
                if (c == a)
                    e_a = dadd(e_a, A.wts[e]);
                else if (c == b)
                    e_b = dadd(e_b, A.wts[e]);
            }
        }
        double sw = A.selfw[i], ki = A.k[i];
        double ta = dadd(dmul(2.0, e_a), dmul(2.0, sw));
        double tb = dadd(dmul(2.0, e_b), dmul(2.0, sw));
        if (A.flags & PLV_F_INTEGRAL) {
            atomicAdd(A.w_int + a, -ta);
            atomicAdd(A.w_int + b, tb);
            atomicAdd(A.a_tot + a, -ki);
            atomicAdd(A.a_tot + b, ki);
        } else {
            A.ea[x] = ta;
            A.eb[x] = tb;
        }
        atomicSub(A.sizes + a, 1);
        atomicAdd(A.sizes + b, 1);
    }
    typedef cub::BlockReduce<unsigned long long, 256> BR;
    __shared__ typename BR::TempStorage tmp;
    unsigned long long tot = BR(tmp).Sum(mine);
    if (threadIdx.x == 0 && tot) atomicAdd(A.count, tot);
}

__global__ void k_move_flags(const uint8_t *moved, const int32_t *subset, const int32_t *target,
                             const int32_t *assign, int64_t ns, uint8_t *flag) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < ns;
         x += (int64_t)gridDim.x * blockDim.x)
        flag[x] = moved[x] && assign[subset[x]] != target[x];
}

__global__ void k_events(const int64_t *mv, int64_t nm, const int32_t *subset, const int32_t *target,
                         const int32_t *assign, uint32_t *ekey, int32_t *eval) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nm;
         q += (int64_t)gridDim.x * blockDim.x) {
        int64_t x = mv[q];
        ekey[2 * q] = (uint32_t)assign[subset[x]];
        ekey[2 * q + 1] = (uint32_t)target[x];
        eval[2 * q] = (int32_t)(2 * q);
        eval[2 * q + 1] = (int32_t)(2 * q + 1);
    }
}

__global__ void k_event_heads(const uint32_t *key, int64_t ne, uint8_t *head) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < ne;
         p += (int64_t)gridDim.x * blockDim.x)
        head[p] = (p == 0 || key[p] != key[p - 1]);
}

// One thread per community run: sequential fold in subset order.
__global__ void k_event_fold(const uint32_t *key, const int32_t *val, const int64_t *runs,
                             int64_t nr, int64_t ne, const int64_t *mv, const int32_t *subset,
                             const double *k, const double *ea, const double *eb, double *a_tot,
                             double *w_int) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nr;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t p0 = runs[r], p1 = (r + 1 < nr) ? runs[r + 1] : ne;
        uint32_t c = key[p0];
        double A = a_tot[c], W = w_int[c];
        for (int64_t p = p0; p < p1; p++) {
            int32_t v = val[p];
            int64_t x = mv[v >> 1];
            double ki = k[subset[x]];
            if (v & 1) {
                W = dadd(W, eb[x]);
                A = dadd(A, ki);
            } else {
                W = dsub(W, ea[x]);
                A = dsub(A, ki);
            }
        }
        a_tot[c] = A;
        w_int[c] = W;
    }
}

__global__ void k_scatter_assign(const uint8_t *moved, const int32_t *subset, const int32_t *target,
                                 int64_t ns, int32_t *assign) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < ns;
         x += (int64_t)gridDim.x * blockDim.x)
        if (moved[x]) assign[subset[x]] = target[x];
}

__global__ void k_pos_scatter(const int32_t *subset, int64_t ns, int32_t *pos, int *dup) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < ns;
         x += (int64_t)gridDim.x * blockDim.x) {
        int32_t old = atomicExch(pos + subset[x], (int32_t)x);
        if (old != -1) atomicOr(dup, 1);
    }
}

__global__ void k_pos_clear(const int32_t *subset, int64_t ns, int32_t *pos) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < ns;
         x += (int64_t)gridDim.x * blockDim.x)
        pos[subset[x]] = -1;
}

int64_t apply(const int64_t *off, const int32_t *nbr, const double *wts, const double *k,
              const double *selfw, int64_t n, const int32_t *subset, int64_t ns,
              const int32_t *target, const uint8_t *moved, const double *e_old,
              const double *e_best, int flags, int32_t *assign, double *a_tot, double *w_int,
              int32_t *sizes, cudaStream_t s) {
    if (ns <= 0) return 0;
    Buf<int32_t> pos;
    bool general = !(flags & (PLV_F_IDENTITY | PLV_F_INDEPENDENT));
    if (general) {
        pos.alloc(n, s);
        k_fill_i32<<<grid_for(n, 256), 256, 0, s>>>(pos, n, -1);
        PLV_LAUNCH_CHECK();
        Buf<int> dup(1, s);
        PLV_CUDA(cudaMemsetAsync(dup.get(), 0, sizeof(int), s));
        k_pos_scatter<<<grid_for(ns, 256), 256, 0, s>>>(subset, ns, pos, dup);
        PLV_LAUNCH_CHECK();
        if (d2h(dup.get(), s)) PLV_FAIL(PLV_EDUP, "subset lists a vertex more than once");
    }
    Buf<double> ea, eb;
    bool integral = flags & PLV_F_INTEGRAL;
    if (!integral) {
        ea.alloc(ns, s);
        eb.alloc(ns, s);
    }
    Buf<unsigned long long> count(1, s);
    PLV_CUDA(cudaMemsetAsync(count.get(), 0, sizeof(unsigned long long), s));
    ApplyArgs A{off, nbr, wts, k, selfw, subset, target, moved, e_old, e_best, pos.get(), flags,
                assign, a_tot, w_int, sizes, ea.get(), eb.get(), count.get()};
    k_apply_edges<<<grid_for(ns, 256), 256, 0, s>>>(A, ns);
    PLV_LAUNCH_CHECK();
    int64_t moves = (int64_t)d2h(count.get(), s);
    if (!integral && moves > 0) {
        Buf<uint8_t> flag(ns, s);
        k_move_flags<<<grid_for(ns, 256), 256, 0, s>>>(moved, subset, target, assign, ns, flag);
        PLV_LAUNCH_CHECK();
        Buf<int64_t> mv(ns, s);
        int64_t nm = select_flagged_index(flag, ns, mv, s);
        int64_t ne = 2 * nm;
        Buf<uint32_t> ekey(ne, s), ekey_s(ne, s);
        Buf<int32_t> eval(ne, s), eval_s(ne, s);
        k_events<<<grid_for(nm, 256), 256, 0, s>>>(mv, nm, subset, target, assign, ekey, eval);
        PLV_LAUNCH_CHECK();
        sort_pairs<uint32_t, int32_t>(ekey, ekey_s, eval, eval_s, ne, 0, bits_for(n > 1 ? n : 2),
                                      s);
        Buf<uint8_t> head(ne, s);
        k_event_heads<<<grid_for(ne, 256), 256, 0, s>>>(ekey_s, ne, head);
        PLV_LAUNCH_CHECK();
        Buf<int64_t> runs(ne, s);
        int64_t nr = select_flagged_index(head, ne, runs, s);
        k_event_fold<<<grid_for(nr, 128), 128, 0, s>>>(ekey_s, eval_s, runs, nr, ne, mv, subset, k,
                                                      ea, eb, a_tot, w_int);
        PLV_LAUNCH_CHECK();
    }
    k_scatter_assign<<<grid_for(ns, 256), 256, 0, s>>>(moved, subset, target, ns, assign);
    PLV_LAUNCH_CHECK();
    if (general) {
        k_pos_clear<<<grid_for(ns, 256), 256, 0, s>>>(subset, ns, pos);
        PLV_LAUNCH_CHECK();
    }
    return moves;
}

}  // namespace plv

extern "C" int plv_decide(const int64_t *off, const int32_t *nbr, const double *wts,
                          const double *k, const int32_t *labels, const int32_t *subset,
                          int64_t ns, const int32_t *assign, const double *a_tot,
                          const int32_t *sizes, double m, int32_t *out_target, uint8_t *out_moved,
                          double *out_e_old, double *out_e_best, int64_t *cand_h, void *stream) {
    PLV_ENTRY
    if (!(m > 0.0)) PLV_FAIL(PLV_EINVAL, "modularity undefined for edgeless graph");
    plv::decide(off, nbr, wts, k, labels, subset, ns, assign, a_tot, sizes, m, 0, out_target,
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
    plv::decide(off, nbr, wts, k, labels, subset, ns, assign, a_tot, sizes, m,
                (flags & PLV_F_INTEGRAL) ? 1 : 0, out_target, out_moved, out_e_old, out_e_best,
                cand_h, plv::S(stream));
    PLV_EXIT
}

extern "C" int plv_apply(const int64_t *off, const int32_t *nbr, const double *wts,
                         const double *k, const double *selfw, int64_t n, const int32_t *subset,
                         int64_t ns, const int32_t *target, const uint8_t *moved,
                         const double *e_old, const double *e_best, int flags, int32_t *assign,
                         double *a_tot, double *w_int, int32_t *sizes, int64_t *moves_h,
                         void *stream) {
    PLV_ENTRY
    int64_t mv = plv::apply(off, nbr, wts, k, selfw, n, subset, ns, target, moved, e_old, e_best,
                            flags, assign, a_tot, w_int, sizes, plv::S(stream));
    if (moves_h) *moves_h = mv;
    PLV_EXIT
}
