// decide.cu -- decide_moves (PL/_kernels.pyx:21-101) on device.
//
// The reference sums e_{i->C} per neighbour community in adjacency order
// (a sequential left fold per community) and takes the argmax of the Eq. 4
// gain under (gain desc, label asc), then applies the singleton-pair guard.
// Vertices of a stage are degree-binned once per plan:
//   tier 0  deg <= 12     thread per vertex, candidates in registers, folds
//                         in adjacency order (exact by construction)
//   tier 1  deg <= 128    warp per vertex, shared-memory hash table, 32-entry
//                         chunks folded in lane order (exact by construction)
//   tier 2  deg <= 680    block per vertex, 16 KB shared table    } certified
//   tier 3  deg <= 2048   block per vertex, 64 KB shared table    } parallel
//   tier 4  larger (hubs) all entries of the stage's hubs at once,} sums
//                         global hash tables                       }
// Certified parallel sums (tiers 2-4).  Reproducing a sequential fold needs
// its additions in order -- a dependent DADD chain of 8.2 cycles per add on
// B200 -- so tiers 2-4 first sum every community in ANY order with atomics,
// along with its term count L.  Both sums are within 2 gamma_{L-1} * sum of
// each other (gamma_k = k u / (1 - k u), u = 2^-53), which bounds how far
// every computed gain can be from the reference's.  The decision is kept only
// when it is certain: the best candidate's lower bound beats every other
// candidate's (and "stay"'s) upper bound.  Otherwise -- and whenever the vertex
// moves, because apply needs e_{i->c_old} and e_{i->best} bit-exact -- the
// few candidates whose intervals overlap are re-folded exactly in adjacency
// order (ordered block compaction of the row, then one thread adds) and the
// decision is taken on the exact values.  The result is the reference's
// decision and the reference's e values, bit for bit.  Integral graphs (all
// weights integers, 2m < 2^52) are exact in any order and skip the check.
#include "localmove.cuh"
#include "lm_device.cuh"
#include "csr.cuh"
#include <cub/cub.cuh>
#include <cstdlib>

namespace plv {

constexpr double U_RND = 1.1102230246251565e-16;  // 2^-53

// ---- optional per-block timeline (off unless plv_debug_trace(1) was called):
// thread 0 of a block records globaltimer stamps at up to 6 marks.
__device__ unsigned long long g_tr[1 << 21];
__device__ unsigned int g_tr_n;
__device__ int g_tr_on;
struct Trace {
    unsigned long long t[6];
    int n;
    __device__ __forceinline__ void mark() {
        if (n < 6) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t[n]));
        n++;
    }
    __device__ __forceinline__ void flush(int kid) {
        unsigned k = atomicAdd(&g_tr_n, 1u);
        if (k < (1u << 21) / 8) {
            unsigned long long *o = g_tr + 8 * k;
            o[0] = ((unsigned long long)kid << 32) | blockIdx.x;
            for (int i = 0; i < 6; i++) o[1 + i] = i < n ? t[i] : 0ull;
            o[7] = (unsigned long long)n;
        }
    }
};
#define TR_BEGIN                                    \
    const bool tr_on = g_tr_on == 1 && threadIdx.x == 0; \
    Trace tr;                                       \
    tr.n = 0;                                       \
    if (tr_on) tr.mark();
#define TR_MARK \
    if (tr_on) tr.mark();
#define TR_END(kid)    \
    if (tr_on) {       \
        tr.mark();     \
        tr.flush(kid); \
    }


// |sequential - any-order| bound for a sum of L positive terms near F.
// A sum of at most two positive terms is the same in every order (0 + a = a,
// a + b = b + a), so it carries no error.
__device__ __forceinline__ double sum_err(double F, int32_t L) {
    return L > 2 ? 2.01 * (double)(L - 1) * U_RND * F : 0.0;
}

// Bound on |gain from exact sums - gain from any-order sums| (see header):
// the sums' error divided by m plus the operations' own rounding.
__device__ __forceinline__ double gain_slack(double Fc, int32_t Lc, double Fo, int32_t Lo,
                                             double m, double g) {
    return 1.01 * ((sum_err(Fc, Lc) + sum_err(Fo, Lo)) / m) +
           8.0 * U_RND * (fabs(Fc - Fo) / m + fabs(g)) + 1e-300;
}

// Table slot of community c (comm_hash, lm_device.cuh).
__device__ __forceinline__ uint32_t hslot(int32_t c, uint32_t mask) { return comm_hash(c) & mask; }

// Open-addressing geometry: power-of-two tables (mask) and arbitrary-size
// tables (multiply-shift range reduction of the same hash), linear probing.
struct PowTab {
    uint32_t mask;
    __device__ __forceinline__ uint32_t first(int32_t c) const { return hslot(c, mask); }
    __device__ __forceinline__ uint32_t next(uint32_t s) const { return (s + 1) & mask; }
    __device__ __forceinline__ uint32_t size() const { return mask + 1; }
};

struct ModTab {
    uint32_t ts;
    __device__ __forceinline__ uint32_t first(int32_t c) const {
        return (uint32_t)(((uint64_t)hslot(c, 0xffffffffu) * ts) >> 32);
    }
    __device__ __forceinline__ uint32_t next(uint32_t s) const { return s + 1 == ts ? 0 : s + 1; }
    __device__ __forceinline__ uint32_t size() const { return ts; }
};

// Find-or-insert c; tables start cleared to key -1.
template <class Tab>
__device__ __forceinline__ uint32_t probe_insert(int32_t *keys, int32_t c, Tab T) {
    uint32_t s = T.first(c);
    while (true) {
        int32_t k = keys[s];
        if (k == c) return s;
        if (k == -1) {
            int32_t old = atomicCAS(keys + s, -1, c);
            if (old == -1 || old == c) return s;
        }
        s = T.next(s);
    }
}
__device__ __forceinline__ uint32_t probe_insert(int32_t *keys, int32_t c, uint32_t mask) {
    return probe_insert(keys, c, PowTab{mask});
}

// probe_insert that also reports whether this call inserted the key.
template <class Tab>
__device__ __forceinline__ uint32_t probe_insert_f(int32_t *keys, int32_t c, Tab T, bool *fresh) {
    uint32_t s = T.first(c);
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
        s = T.next(s);
    }
}
__device__ __forceinline__ uint32_t probe_insert_f(int32_t *keys, int32_t c, uint32_t mask,
                                                   bool *fresh) {
    return probe_insert_f(keys, c, PowTab{mask}, fresh);
}

template <class Tab>
__device__ __forceinline__ int probe_find(const int32_t *keys, int32_t c, Tab T) {
    uint32_t s = T.first(c);
    while (true) {
        int32_t k = keys[s];
        if (k == c) return (int)s;
        if (k == -1) return -1;
        s = T.next(s);
    }
}
__device__ __forceinline__ int probe_find(const int32_t *keys, int32_t c, uint32_t mask) {
    return probe_find(keys, c, PowTab{mask});
}

// Find-or-insert c by CAS alone (no separate probe load: one L2 round trip per
// probed slot); reports whether this call inserted the key.
__device__ __forceinline__ uint32_t probe_claim(int32_t *keys, int32_t c, uint32_t mask,
                                                bool *fresh) {
    uint32_t s = hslot(c, mask);
    while (true) {
        const int32_t old = atomicCAS(keys + s, -1, c);
        if (old == -1 || old == c) {
            *fresh = old == -1;
            return s;
        }
        s = (s + 1) & mask;
    }
}


__device__ __forceinline__ void warp_best(Best &b) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        Best o2;
        o2.g = __shfl_xor_sync(FULL, b.g, o);
        o2.l = __shfl_xor_sync(FULL, b.l, o);
        o2.c = __shfl_xor_sync(FULL, b.c, o);
        o2.e = __shfl_xor_sync(FULL, b.e, o);
        o2.n = __shfl_xor_sync(FULL, b.n, o);
        consider(b, o2.g, o2.l, o2.c, o2.e, o2.n);
    }
}

template <int NT>
struct BestSmem {
    Best w[NT / 32];
    Best out;
};

// Block argmax; the result is returned to every thread.
template <int NT>
__device__ __forceinline__ Best block_best(BestSmem<NT> &S, Best b) {
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    warp_best(b);
    if (lane == 0) S.w[wid] = b;
    __syncthreads();
    if (wid == 0) {
        Best c = lane < NT / 32 ? S.w[lane] : S.w[0];
        warp_best(c);
        if (lane == 0) S.out = c;
    }
    __syncthreads();
    Best r = S.out;
    __syncthreads();
    return r;
}


// ------------------------------------------------------------ tier 0


#ifndef T0_MINB
#define T0_MINB 2
#endif
// The general kernels of a first stage step aside when the state is singleton.
__device__ __forceinline__ bool single_state(const DecideArgs &A) {
    return A.notsingle && ld_state(A.notsingle) == 0;
}

__global__ void __launch_bounds__(256, T0_MINB) k_decide_t0(DecideArgs A, TierRef L, int64_t cnt) {
    if (single_state(A)) return;
    decide_t0_body(A, L, cnt, blockIdx.x, gridDim.x);
}

// Fold one 32-entry chunk (c, w per lane; c = -1 for none) into a table in
// adjacency order.  wb: the chunk's 32 weights staged in lane order.
template <class Tab>
__device__ __forceinline__ void fold_chunk(int32_t *keys, double *vals, Tab T, int32_t c,
                                           const double *wb, int lane) {
    unsigned grp = __match_any_sync(FULL, c);
    if (c >= 0 && lane == __ffs(grp) - 1) {
        uint32_t s = probe_insert(keys, c, T);
        double v = vals[s];  // 0.0 when fresh
        for (unsigned g = grp; g; g &= g - 1) v = dadd(v, wb[__ffs(g) - 1]);
        vals[s] = v;
    }
}

// ------------------------------------------------------------ tier 1

// Tier 1 over blocks [b, b + nb) of the launch (a warp per vertex).
// NW: warps per block of the launching kernel.
template <int NW>
__device__ __forceinline__ void decide_t1_body(const DecideArgs &A, const TierRef &L, int64_t cnt,
                                               int64_t b, int64_t nb) {
    __shared__ int32_t skeys[NW][T1_TS];
    __shared__ double svals[NW][T1_TS];
    __shared__ double swb[NW][32];
    int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int32_t *keys = skeys[wid];
    double *vals = svals[wid];
    double *wb = swb[wid];
    unsigned long long my_cand = 0;
    for (int64_t q = b * (int64_t)NW + wid; q < cnt; q += nb * (int64_t)NW) {
        const int64_t x = L.x[q];
        const int32_t i = L.vid[q];
        const int64_t e0 = L.row[q], e1 = L.end[q];
        const int32_t c_old = ld_state(A.assign + (i));
        int deg = (int)(e1 - e0);
        uint32_t ts = 32;
        while (ts < (uint32_t)(deg + deg / 2 + 2)) ts <<= 1;
        uint32_t mask = ts - 1;
        for (uint32_t s = lane; s < ts; s += 32) {
            keys[s] = -1;
            vals[s] = 0.0;
        }
        __syncwarp();
        // all (<= 4) chunks' loads first -- rows, then communities -- so the
        // warp waits for two round trips, not two per chunk; then the chunks
        // fold in adjacency order
        constexpr int NCH = (T1_MAXD + 31) / 32;
        int32_t jv[NCH], cv[NCH];
        double wv[NCH];
#pragma unroll
        for (int u = 0; u < NCH; u++) {
            const int64_t e = e0 + 32 * u + lane;
            jv[u] = e < e1 ? ld_row(A.nbr + (e)) : i;
            wv[u] = e < e1 ? ld_row(A.wts + (e)) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < NCH; u++) cv[u] = jv[u] != i ? ld_state(A.assign + jv[u]) : -1;
#pragma unroll
        for (int u = 0; u < NCH; u++) {
            if (e0 + 32 * u >= e1) break;
            wb[lane] = cv[u] >= 0 ? wv[u] : 0.0;
            __syncwarp();
            fold_chunk(keys, vals, PowTab{mask}, cv[u], wb, lane);
            __syncwarp();
        }
        double e_old = 0.0;
        if (lane == 0) {
            int s = probe_find(keys, c_old, mask);
            e_old = s >= 0 ? vals[s] : 0.0;
        }
        e_old = __shfl_sync(FULL, e_old, 0);
        double ki = A.k[i];
        double a_old_excl = dsub(ld_state(A.a_tot + (c_old)), ki);
        Best b{0.0, LBL(A.labels, c_old), c_old, 0.0, 0};
        int nc = 0;
        for (uint32_t s = lane; s < ts; s += 32) {
            int32_t c = keys[s];
            if (c < 0) continue;
            nc++;
            if (c == c_old) continue;
            consider(b, gain_of(vals[s], e_old, A.m, ki, a_old_excl, ld_state(A.a_tot + (c)), A.four_m_sq),
                     LBL(A.labels, c), c, vals[s], 0);
        }
        warp_best(b);
        my_cand += nc;
        if (lane == 0) finish_vertex(A, x, c_old, e_old, b.g, b.c, b.e);
        __syncwarp();
    }
    if (A.cand) {
        for (int o = 16; o > 0; o >>= 1) my_cand += __shfl_xor_sync(FULL, my_cand, o);
        if (lane == 0 && my_cand) atomicAdd(A.cand, my_cand);
    }
}

__global__ void __launch_bounds__(T1_WARPS * 32) k_decide_t1(DecideArgs A, TierRef L,
                                                              int64_t cnt) {
    if (single_state(A)) return;
    decide_t1_body<T1_WARPS>(A, L, cnt, blockIdx.x, gridDim.x);
}

// A small stage whose vertices all sit in tiers 0 and 1: both tiers in one
// launch (the first nb0 blocks take tier 0), on the stage's own stream --
// no fork / join around the tiers, and a programmatic launch after the
// previous kernel.
__global__ void __launch_bounds__(256) k_decide_t01(DecideArgs A, TierRef L0, int64_t cnt0,
                                                    TierRef L1, int64_t cnt1, int nb0) {
    pdl_wait();
    if (single_state(A)) return;
    if ((int)blockIdx.x < nb0)
        decide_t0_body(A, L0, cnt0, blockIdx.x, nb0);
    else
        decide_t1_body<8>(A, L1, cnt1, blockIdx.x - nb0, gridDim.x - nb0);
}

// ------------------------------------------------ certification machinery

template <int NT>
struct CertSmem {
    BestSmem<NT> bs;
    typename cub::BlockScan<int, NT>::TempStorage scan;
    int32_t *cidx;  // [NT * FU] ordered compaction of matching entries (set by the kernel)
    double *cw;     // [NT * FU]
    int32_t N[MAXS + 2];  // communities to fold exactly (N[0] = c_old)
    double acc[MAXS + 2];
    double f_old;
    int32_t l_old;
    int nn, nS, flag;  // flag: 1 stay overlaps, 2 overflow
    unsigned long long ncand;
};

// Sum of w over the lanes of this lane's match group `grp` (any order).  Every
// shuffle is a full-warp shuffle inside a warp-uniform loop: a shuffle under
// the per-group mask would split the warp into one serialised shuffle per
// distinct group.
__device__ __forceinline__ double group_sum(unsigned grp, double w) {
    const int n = __popc(grp);
    const int nmax = __reduce_max_sync(FULL, (unsigned)n);
    double v = 0.0;
    unsigned g = grp;
    for (int t = 0; t < nmax; t++) {
        const int src = g ? __ffs(g) - 1 : (int)(threadIdx.x & 31);
        const double x = __shfl_sync(FULL, w, src);
        if (g) {
            v = dadd(v, x);
            g &= g - 1;
        }
    }
    return v;
}

// Accumulate one entry (c, w) into the any-order table (sum and term count)
// and list the slot when this call inserted it.
template <class Tab, class CL>
__device__ __forceinline__ void accum_entry(int32_t *keys, double *vals, int32_t *cnt, Tab T,
                                            int32_t c, double w, int lane, CL *clist, int *ncl) {
    // every lane adds its own entry: shared-memory atomics serialise lanes
    // that hit the same slot, which measured cheaper than grouping the warp's
    // lanes by community first (match + group sums)
    bool fresh = false;
    uint32_t s = 0;
    if (c >= 0) {
        s = probe_insert_f(keys, c, T, &fresh);
        atomicAdd(vals + s, w);
        atomicAdd(cnt + s, 1);
    }
    unsigned fm = __ballot_sync(FULL, fresh);  // one list append per warp
    if (fm) {
        int first = __ffs(fm) - 1, pos = 0;
        if (lane == first) pos = atomicAdd(ncl, __popc(fm));
        pos = __shfl_sync(FULL, pos, first);
        if (fresh) clist[pos + __popc(fm & ((1u << lane) - 1))] = (CL)s;
    }
}

// |gain(exact sums) - gain(any-order sums)| bound without divisions (it is a
// bound, so the reciprocal's rounding is absorbed by the 1.01 / 8u factors).
__device__ __forceinline__ double gain_slack_r(double Fc, int32_t Lc, double Fo, int32_t Lo,
                                               double inv_m, double g) {
    // both sums exact -> the gain is computed from the reference's own
    // operands with the reference's operations: no slack at all
    if (Lc <= 2 && Lo <= 2) return 0.0;
    return 1.02 * ((sum_err(Fc, Lc) + sum_err(Fo, Lo)) * inv_m) +
           8.0 * U_RND * (fabs(Fc - Fo) * inv_m * 1.001 + fabs(g)) + 1e-300;
}

// Passes over the candidates (slots clist[0..ncl), or with clist == NULL every
// slot 0..ncl of the table, empty ones skipped) of the any-order table of
// vertex i: pass 1 finds the best on the approximate gains and stores every
// candidate's gain in vals[] and its slack (rounded up to float) in cnt[];
// pass 2 collects the candidates whose intervals overlap the best and clears
// the slots when `clear`.  Returns the approximate best.
template <class CL>
__device__ __forceinline__ uint32_t slot_at(const CL *clist, int p) {
    return clist ? (uint32_t)clist[p] : (uint32_t)p;
}

template <int NT, class Tab, class CL, int CU = 1>
__device__ Best certify_table(const DecideArgs &A, int32_t c_old, double ki, int32_t *keys,
                              double *vals, int32_t *cnt, Tab T, const CL *clist, int ncl,
                              CertSmem<NT> &S, bool clear) {
    const int tid = threadIdx.x;
    if (tid == 0) {
        int s = probe_find(keys, c_old, T);
        S.f_old = s >= 0 ? vals[s] : 0.0;
        S.l_old = s >= 0 ? cnt[s] : 0;
        S.nS = 0;
        S.flag = 0;
    }
    __syncthreads();
    const double f_old = S.f_old;
    const int32_t l_old_n = S.l_old;
    const double a_old_excl = dsub(ld_state(A.a_tot + (c_old)), ki);
    const double inv_m = 1.0 / A.m;
    const int64_t l_old = LBL(A.labels, c_old);
    Best b{0.0, l_old, c_old, 0.0, 0};
    // CU candidates per thread in flight: the slot, table and a_tot loads of
    // a batch are issued before any of them is used
    for (int p0 = tid; p0 < ncl; p0 += NT * CU) {
        uint32_t sl[CU];
        int32_t c[CU], L[CU];
        double F[CU], at[CU];
#pragma unroll
        for (int u = 0; u < CU; u++) sl[u] = p0 + u * NT < ncl ? slot_at(clist, p0 + u * NT) : 0;
#pragma unroll
        for (int u = 0; u < CU; u++) {
            const bool ok = p0 + u * NT < ncl;
            c[u] = ok ? keys[sl[u]] : -1;
            F[u] = ok ? vals[sl[u]] : 0.0;
            L[u] = ok ? cnt[sl[u]] : 0;
        }
#pragma unroll
        for (int u = 0; u < CU; u++) at[u] = c[u] >= 0 && c[u] != c_old ? ld_state(A.a_tot + c[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < CU; u++) {
            if (c[u] < 0 || c[u] == c_old) continue;
            double g = gain_of(F[u], f_old, A.m, ki, a_old_excl, at[u], A.four_m_sq);
            consider(b, g, LBL(A.labels, c[u]), c[u], F[u], L[u]);
            vals[sl[u]] = g;
            cnt[sl[u]] = __float_as_int(
                __double2float_ru(gain_slack_r(F[u], L[u], f_old, l_old_n, inv_m, g)));
        }
    }
    b = block_best<NT>(S.bs, b);
    const bool stay_best = b.c == c_old;
    const double slack_b = stay_best ? 0.0 : gain_slack_r(b.e, b.n, f_old, l_old_n, inv_m, b.g);
    const double lower = stay_best ? 0.0 : b.g - slack_b;
    unsigned long long nc = 0;
    for (int p0 = tid; p0 < ncl; p0 += NT * CU) {
        uint32_t sl[CU];
        int32_t c[CU];
        float slk[CU];
        double g[CU];
#pragma unroll
        for (int u = 0; u < CU; u++) sl[u] = p0 + u * NT < ncl ? slot_at(clist, p0 + u * NT) : 0;
#pragma unroll
        for (int u = 0; u < CU; u++) {
            const bool ok = p0 + u * NT < ncl;
            c[u] = ok ? keys[sl[u]] : -1;
            slk[u] = ok ? __int_as_float(cnt[sl[u]]) : 0.0f;
            g[u] = ok ? vals[sl[u]] : 0.0;
            nc += c[u] >= 0 ? 1 : 0;
        }
#pragma unroll
        for (int u = 0; u < CU; u++) {
            if (c[u] >= 0 && c[u] != c_old && c[u] != b.c) {
                // two exact gains were already ordered exactly by block_best
                double slv = (double)slk[u];
                if ((slv > 0.0 || slack_b > 0.0) && g[u] + slv >= lower) {
                    int k = atomicAdd(&S.nS, 1);
                    if (k < MAXS)
                        S.N[2 + k] = c[u];
                    else
                        atomicOr(&S.flag, 2);
                }
            }
            if (clear && c[u] >= 0) {
                keys[sl[u]] = -1;
                vals[sl[u]] = 0.0;
                cnt[sl[u]] = 0;
            }
        }
    }
    if (tid == 0) {
        // "stay" (exact gain 0) overlaps an inexact best
        if (!stay_best && slack_b > 0.0 && lower <= 0.0) S.flag |= 1;
        S.ncand = 0;
    }
    // the candidate statistic: one atomic per warp, no block-wide reduction
    if (A.cand) {
        for (int o = 16; o > 0; o >>= 1) nc += __shfl_xor_sync(FULL, nc, o);
        if ((tid & 31) == 0 && nc) atomicAdd(A.cand, nc);
    }
    __syncthreads();
    return b;
}

// Exact left folds (adjacency order) of the communities S.N[0..S.nn) over the
// row of i: ordered block compaction of the matching entries (each thread
// takes FU consecutive entries per chunk, loads in flight together), then
// thread 0 adds them in order.  S.cidx / S.cw hold NT * FU entries.  Results
// in S.acc.
template <int NT, int FU>
__device__ void exact_folds(const DecideArgs &A, int32_t i, CertSmem<NT> &S) {
    const int tid = threadIdx.x;
    const int64_t e0 = A.off[i], e1 = A.off[i + 1];
    const int nn = S.nn;
    if (tid < nn) S.acc[tid] = 0.0;
    __syncthreads();
    for (int64_t base = e0; base < e1; base += (int64_t)NT * FU) {
        const int64_t eb = base + (int64_t)tid * FU;
        int32_t j[FU], c[FU], idx[FU];
#pragma unroll
        for (int u = 0; u < FU; u++) j[u] = eb + u < e1 ? ld_row(A.nbr + (eb + u)) : i;
#pragma unroll
        for (int u = 0; u < FU; u++) c[u] = j[u] != i ? ld_state(A.assign + j[u]) : -1;
        int cntm = 0;
#pragma unroll
        for (int u = 0; u < FU; u++) {
            idx[u] = -1;
            if (c[u] >= 0)
                for (int t = 0; t < nn; t++)
                    if (S.N[t] == c[u]) {
                        idx[u] = t;
                        break;
                    }
            cntm += idx[u] >= 0;
        }
        int pos, total;
        cub::BlockScan<int, NT>(S.scan).ExclusiveSum(cntm, pos, total);
#pragma unroll
        for (int u = 0; u < FU; u++)
            if (idx[u] >= 0) {
                S.cidx[pos] = idx[u];
                S.cw[pos] = ld_row(A.wts + (eb + u));
                pos++;
            }
        __syncthreads();
        if (tid == 0) {
            double a0 = S.acc[0], a1 = nn > 1 ? S.acc[1] : 0.0;
            for (int t = 0; t < total; t++) {
                int k = S.cidx[t];
                double v = S.cw[t];
                if (k == 0)
                    a0 = dadd(a0, v);
                else if (k == 1)
                    a1 = dadd(a1, v);
                else
                    S.acc[k] = dadd(S.acc[k], v);
            }
            S.acc[0] = a0;
            if (nn > 1) S.acc[1] = a1;
        }
        __syncthreads();
    }
}

// After certify_table: either finish (certain, no move) or fold the needed
// communities exactly and decide on exact values.  Returns false on overflow
// (more than MAXS overlapping candidates): the caller must decide exactly.
template <int NT, int FU = 1>
__device__ bool resolve(const DecideArgs &A, int64_t x, int32_t i, int32_t c_old, double ki,
                        const Best &b, CertSmem<NT> &S) {
    const int tid = threadIdx.x;
    if (S.flag & 2) return false;
    const bool certain = S.nS == 0 && !(S.flag & 1);
    if (certain) {
        // certain: b is the exact best; the exact gain is > 0 iff b.g > 0
        // (an inexact best has lower > 0 when "stay" does not overlap it)
        bool moved = b.c != c_old && b.g > 0.0;
        if (moved && ld_state(A.sizes + c_old) == 1 && ld_state(A.sizes + b.c) == 1 &&
            LBL(A.labels, b.c) > LBL(A.labels, c_old))
            moved = false;
        // a mover whose two sums have <= 2 terms already holds the exact e values
        if (!moved || (b.n <= 2 && S.l_old <= 2)) {
            if (tid == 0) {
                if (moved)
                    finish_vertex(A, x, c_old, S.f_old, b.g, b.c, b.e);
                else
                    finish_vertex(A, x, c_old, S.f_old, 0.0, c_old, 0.0);
            }
            __syncthreads();
            return true;
        }
    }
    if (tid == 0) {
        S.N[0] = c_old;
        int nn = 1;
        if (b.c != c_old) S.N[nn++] = b.c;
        for (int t = 0; t < S.nS; t++) S.N[nn++] = S.N[2 + t];
        S.nn = nn;
    }
    __syncthreads();
    exact_folds<NT, FU>(A, i, S);
    if (tid == 0) {
        double a_old_excl = dsub(ld_state(A.a_tot + (c_old)), ki);
        Best e{0.0, LBL(A.labels, c_old), c_old, 0.0, 0};
        for (int t = 1; t < S.nn; t++) {
            int32_t c = S.N[t];
            consider(e, gain_of(S.acc[t], S.acc[0], A.m, ki, a_old_excl, ld_state(A.a_tot + (c)), A.four_m_sq),
                     LBL(A.labels, c), c, S.acc[t], 0);
        }
        finish_vertex(A, x, c_old, S.acc[0], e.g, e.c, e.e);
    }
    __syncthreads();
    return true;
}

// ------------------------------------------------------------ tier 2

// Exact fallback: in-order fold into the (clean) table, communities split
// over the warps so each community sees one ordered left fold, then the exact
// argmax.  Leaves the table clean.  cbuf / wbuf: NT staging slots (the
// CertSmem compaction buffers, idle here).
template <int NT, class Tab>
__device__ void table_exact(const DecideArgs &A, int64_t x, int32_t i, int32_t c_old, double ki,
                            int32_t *keys, double *vals, Tab T, CertSmem<NT> &S) {
    constexpr int NW = NT / 32;
    constexpr int LOGW = NW >= 32 ? 5 : NW >= 16 ? 4 : NW >= 8 ? 3 : NW >= 4 ? 2 : NW >= 2 ? 1 : 0;
    static_assert((1 << LOGW) == NW, "warps per block must be a power of two");
    int32_t *cbuf = S.cidx;
    double *wbuf = S.cw;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int64_t e0 = A.off[i], e1 = A.off[i + 1];
    __syncthreads();
    for (int64_t base = e0; base < e1; base += NT) {
        int64_t e = base + tid;
        int32_t c = -1;
        double w = 0.0;
        if (e < e1) {
            int32_t j = ld_row(A.nbr + (e));
            if (j != i) {
                c = ld_state(A.assign + (j));
                w = ld_row(A.wts + (e));
            }
        }
        cbuf[tid] = c;
        wbuf[tid] = w;
        __syncthreads();
        int nsub = (int)((e1 - base + 31) / 32);
        if (nsub > NW) nsub = NW;
        for (int sc = 0; sc < nsub; sc++) {
            int32_t cc = cbuf[sc * 32 + lane];
            bool mine = cc >= 0 &&
                        (LOGW == 0 || (int)(((uint32_t)cc * 0x85EBCA6Bu) >> (32 - LOGW)) == wid);
            if (__any_sync(FULL, mine))
                fold_chunk(keys, vals, T, mine ? cc : -1, wbuf + sc * 32, lane);
            __syncwarp();
        }
        __syncthreads();
    }
    if (tid == 0) {
        int s = probe_find(keys, c_old, T);
        S.f_old = s >= 0 ? vals[s] : 0.0;
    }
    __syncthreads();
    const double e_old = S.f_old, a_old_excl = dsub(ld_state(A.a_tot + (c_old)), ki);
    Best b{0.0, LBL(A.labels, c_old), c_old, 0.0, 0};
    for (uint32_t s = tid; s < T.size(); s += NT) {
        int32_t c = keys[s];
        if (c >= 0 && c != c_old)
            consider(b, gain_of(vals[s], e_old, A.m, ki, a_old_excl, ld_state(A.a_tot + (c)), A.four_m_sq),
                     LBL(A.labels, c), c, vals[s], 0);
    }
    b = block_best<NT>(S.bs, b);
    for (uint32_t s = tid; s < T.size(); s += NT) {
        keys[s] = -1;
        vals[s] = 0.0;
    }
    if (tid == 0) finish_vertex(A, x, c_old, e_old, b.g, b.c, b.e);
    __syncthreads();
}

// One block decides one vertex at a time from a shared-memory table `keys /
// vals / cntt` (clean on entry and exit) with candidate list `clist`:
// any-order accumulation of the row (U entries per thread in flight), the
// certification passes, then the exact resolution when needed.
template <int NT, int U, int FU, class Tab, class CL>
__device__ __forceinline__ void block_decide(const DecideArgs &A, int64_t x, int32_t i, int64_t e0,
                                             int64_t e1, Tab T, int32_t *keys, double *vals,
                                             int32_t *cntt, CL *clist, int *ncl, CertSmem<NT> &S,
                                             unsigned long long &my_cand, Trace *trp = nullptr) {
    const int tid = threadIdx.x, lane = tid & 31;
    const int32_t c_old = ld_state(A.assign + (i));
    const double ki = A.k[i];
    if (tid == 0) *ncl = 0;
    __syncthreads();
    for (int64_t b0 = e0; b0 < e1; b0 += (int64_t)NT * U) {
        int32_t j[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            int64_t e = b0 + u * NT + tid;
            j[u] = e < e1 ? ld_row(A.nbr + (e)) : i;
        }
        int32_t c[U];
        double w[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            int64_t e = b0 + u * NT + tid;
            bool ok = j[u] != i;  // out-of-range entries carry j = i
            c[u] = ok ? ld_state(A.assign + j[u]) : -1;
            w[u] = ok ? ld_row(A.wts + (e)) : 0.0;
        }
        if (trp && b0 == e0) {
            volatile int32_t sink = c[0];  // wait for the loads
            (void)sink;
            trp->mark();
        }
#pragma unroll
        for (int u = 0; u < U; u++) accum_entry(keys, vals, cntt, T, c[u], w[u], lane, clist, ncl);
    }
    __syncthreads();
    if (trp) trp->mark();
    Best b = certify_table<NT>(A, c_old, ki, keys, vals, cntt, T, clist, *ncl, S, true);
    if (trp) trp->mark();
    (void)my_cand;  // counted per warp in certify_table
    if (A.integral) {
        // exact in any order: the plain argmax is the reference's
        if (tid == 0) finish_vertex(A, x, c_old, S.f_old, b.g, b.c, b.e);
        __syncthreads();
        return;
    }
    if (!resolve<NT, FU>(A, x, i, c_old, ki, b, S))
        table_exact<NT>(A, x, i, c_old, ki, keys, vals, T, S);
}

constexpr int T2_FU = 1;
constexpr int T2A_NT = 128;  // threads per tier-2 block (64 and 256 measured slower)
constexpr int T2_U = 1;  // row entries per thread in flight during the accumulation (2 measured slower)
constexpr int T2_WIDE_MAX = 600;  // tiers 2-3 with at most this many vertices: wide blocks (64-1000 measured)

// Tiers 2 and 3: block per vertex, the table (TS slots) in dynamic shared
// memory; tier 2's small tables let 3x more vertices be in flight per SM.
template <int TS, int MAXD, int NT>
__global__ void __launch_bounds__(NT) k_decide_t2(DecideArgs A, TierRef L, int64_t cnt) {
    if (single_state(A)) return;
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ CertSmem<NT> S;
    __shared__ int32_t cidx[NT * T2_FU];
    __shared__ double cw[NT * T2_FU];
    __shared__ uint16_t clist[MAXD];  // candidate slots (<= degree of them)
    __shared__ int ncl;
    const int tid = threadIdx.x;
    if (tid == 0) {
        S.cidx = cidx;
        S.cw = cw;
    }
    double *vals = reinterpret_cast<double *>(dsm);
    int32_t *keys = reinterpret_cast<int32_t *>(dsm + sizeof(double) * TS);
    int32_t *cntt = keys + TS;
    unsigned long long my_cand = 0;
    for (uint32_t s = tid; s < TS; s += NT) {
        keys[s] = -1;
        vals[s] = 0.0;
        cntt[s] = 0;
    }
    TR_BEGIN
    for (int64_t q = blockIdx.x; q < cnt; q += gridDim.x) {
        const int64_t e0 = L.row[q], e1 = L.end[q];
        const int64_t deg = e1 - e0;
        uint32_t ts = 64;
        while (ts < (uint64_t)(deg + deg / 2 + 2)) ts <<= 1;
        block_decide<NT, T2_U, T2_FU>(A, L.x[q], L.vid[q], e0, e1, PowTab{ts - 1}, keys, vals, cntt,
                                   clist, &ncl, S, my_cand, tr_on && tr.n < 2 ? &tr : nullptr);
    }
    if (A.cand && tid == 0 && my_cand) atomicAdd(A.cand, my_cand);
    TR_END(NT == 1024 ? 5 : NT == 512 ? 6 : 7)
}

// ------------------------------------------------------------ tier 4 (hubs)

constexpr int HSB = 512;            // threads per hub pass block
constexpr int HSU = 8;              // table slots per thread in a pass block (2, 4, 8 measured)
constexpr int HTSL = HSB * HSU;     // table slots per pass block
constexpr int HCPAD = 32;           // per-hub counters one 128-byte line apart
constexpr int HUB_DENSE_KMAX = 32;  // stages with at most this many hubs may use dense arrays (16-128 measured)
constexpr int HFU = 4;              // row entries per thread per exact-fold chunk (hubs)

// A candidate near its slice's best: community, gain, slack (rounded up).
struct NearCand {
    int32_t c;
    float sl;
    double g;
};

// Per-stage hub scratch (device pointers; hub index q is stage-local).
// Idle state: sold = -1, counters 0, table slices clean.
struct HubScratch {
    const int64_t *row;  // [nh] first entry of the hub's row
    const int32_t *vid;  // [nh] the hub
    int32_t *sold;       // [nh] table slot of c_old (-1: absent)
    int32_t *ncnt;       // [nh * HCPAD]: [0] near candidates with slack, [1] exact ones
    NearCand *nearA;     // [nh * MAXS] near candidates with slack > 0
    NearCand *nearB;     // [nh * MAXS] near candidates with exact gains
    Best *part;          // [poff[nh]] pass-1 partial bests (one per slice)
    const int64_t *blk;  // pass blocks of the stage: (hub << 32) | slice
    const int64_t *poff; // [nh + 1] first partial of each hub
    int64_t nh;
    // dense mode (few hubs): per-hub arrays indexed by community, no claims
    DenseRec *drec;      // [dense_k * dn] sum / term count / first row position (idle:
                         // 0 / 0 / INT_MAX), one 16-byte record: an entry's three
                         // updates and the pass's three reads touch ONE 32-byte sector
    int32_t *cbuf;       // [entries] community of every hub entry (-1: self loop)
    int64_t dn;
};

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

// Every entry of every hub of the stage: any-order sums into the hub's slice
// of the global table (warp-aggregated per (hub, community)); the inserter of
// c_old records its slot.
template <bool DENSE>
__global__ void k_hub_accum(DecideArgs A, const int64_t *eoff, const int64_t *toff, int64_t nh,
                            int64_t E, int32_t *hkeys, double *hvals, int32_t *hcnt, HubScratch H) {
    if (A.notsingle) {  // a first stage: the singleton kernels may take it
        pdl_wait();
        if (ld_state(A.notsingle) == 0) return;
    }

    TR_BEGIN
    const int lane = threadIdx.x & 31;
    bool waited = false;
    // warp-uniform loop: the whole warp takes 32 consecutive entries per step
    for (int64_t w0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); w0 < E;
         w0 += (int64_t)gridDim.x * blockDim.x) {
        int64_t t = w0 + lane;
        int32_t c = -1, c_old = -1, i = -1, j = -1;
        double w = 0.0, wv = 0.0;
        int64_t q = 0;
        if (t < E) {  // the static part of the entry (graph, plan)
            q = hub_of(eoff, nh, t);
            i = H.vid[q];
            const int64_t e = H.row[q] + (t - eoff[q]);
            j = ld_row(A.nbr + (e));
            wv = ld_row(A.wts + (e));
        }
        if (!waited) {
            // launched programmatically: the loads above overlap the previous
            // stage's apply; the assignment and the tables only after it
            pdl_wait();
            waited = true;
        }
        if (t < E) {
            c_old = ld_state(A.assign + (i));
            if (j != i) {
                c = ld_state(A.assign + (j));
                w = wv;
            }
        }
        TR_MARK
        if (DENSE && t < E) H.cbuf[t] = c;
        if (DENSE) {  // every lane adds its own entry: plain reductions, no grouping
            if (c >= 0) {
                const int64_t d = q * H.dn + c;
                atomicAdd(&H.drec[d].val, w);
                atomicAdd(&H.drec[d].cnt, 1);
                atomicMin(&H.drec[d].mk, (int32_t)(t - eoff[q]));
            }
            continue;
        }
        // hash tables: group lanes by (hub, community), one claim per group
        const uint64_t key = c >= 0 ? (((uint64_t)q << 32) | (uint32_t)c) : ~0ull;
        const unsigned grp = __match_any_sync(FULL, key);
        const int leader = __ffs(grp) - 1;
        uint32_t s = 0;
        if (c >= 0 && lane == leader) {
            const int64_t base = toff[q];
            const uint32_t mask = (uint32_t)(toff[q + 1] - base - 1);
            bool fresh;
            s = probe_claim(hkeys + base, c, mask, &fresh);
            if (fresh && c == c_old) H.sold[q] = (int32_t)s;
        }
        s = __shfl_sync(FULL, s, leader);  // the group's slot; every lane adds its entry
        if (c >= 0) {
            const int64_t base = toff[q];
            atomicAdd(hvals + base + s, w);
            atomicAdd(hcnt + base + s, 1);
        }
    }
    TR_END(1)
}

// Bound on the certification slack of any candidate of vertex i (degree d,
// weighted degree ki): every sum is <= ki with <= d terms and |gain| <= 2 ki / m.
__device__ __forceinline__ double slack_max(double ki, int64_t d, double inv_m) {
    const double se = 2.01 * (double)(d > 1 ? d - 1 : 0) * U_RND * ki;
    return 1.1 * (1.02 * (2.0 * se * inv_m) + 8.0 * U_RND * (3.01 * ki * inv_m)) + 1e-300;
}

// The decision for hub q, by the block that completed its last pass item:
// the hub's best from the partials, the overlap test on the listed near
// candidates, then the decision.  Certain non-moves (and integral graphs)
// finish at once; otherwise the overlapping communities are folded exactly
// (or, past MAXS of them, the whole row through the hub's clean table slice)
// and the decision is taken on exact values.  Resets the hub's state.
__device__ __forceinline__ Best ldcg_best(const Best *p) {
    Best b;
    b.g = __ldcg(&p->g);
    b.l = __ldcg(&p->l);
    b.c = __ldcg(&p->c);
    b.e = __ldcg(&p->e);
    b.n = __ldcg(&p->n);
    return b;
}
__device__ __forceinline__ NearCand ldcg_near(const NearCand *p) {
    return NearCand{__ldcg(&p->c), __ldcg(&p->sl), __ldcg(&p->g)};
}

template <int NT, bool DENSE>
__device__ void hub_decide_one(const DecideArgs &A, const int32_t *list, const int64_t *toff,
                               int32_t *hkeys, double *hvals, int32_t *hcnt, const HubScratch &H,
                               int64_t q, CertSmem<NT> &S) {
    const int tid = threadIdx.x;
    const int64_t x = list[q];
    const int32_t i = H.vid[q];
    const int32_t c_old = ld_state(A.assign + (i));
    const double ki = A.k[i];
    const int64_t base = toff[q];
    // warp 0: the hub's best from the partials and the overlap test on the
    // near candidates (one per lane); the block waits once
    if (tid < 32) {
        const int lane = tid;
        Best bw{0.0, LBL(A.labels, c_old), c_old, 0.0, 0};
        for (int64_t t = H.poff[q] + lane; t < H.poff[q + 1]; t += 32) {
            const Best o = ldcg_best(H.part + t);
            consider(bw, o.g, o.l, o.c, o.e, o.n);
        }
        warp_best(bw);
        const int64_t dq = q * H.dn;
        const int32_t so = DENSE ? 0 : H.sold[q];
        const double f_old = DENSE ? H.drec[dq + c_old].val : so >= 0 ? hvals[base + so] : 0.0;
        const int32_t l_old = DENSE ? H.drec[dq + c_old].cnt : so >= 0 ? hcnt[base + so] : 0;
        const int na = __ldcg(H.ncnt + q * HCPAD), nb = __ldcg(H.ncnt + q * HCPAD + 1);
        const bool stay_best = bw.c == c_old;
        const double slack_b =
            stay_best ? 0.0 : gain_slack_r(bw.e, bw.n, f_old, l_old, 1.0 / A.m, bw.g);
        const double lower = stay_best ? 0.0 : bw.g - slack_b;
        int flag = 0;
        bool pa = false, pb = false;
        int32_t ca = -1, cb = -1;
        if (!A.integral) {
            if (na > MAXS || (slack_b > 0.0 && nb > MAXS)) flag |= 2;
            if (lane < na && lane < MAXS) {
                const NearCand o = ldcg_near(H.nearA + q * MAXS + lane);
                pa = o.c != bw.c && o.g + (double)o.sl >= lower;
                ca = o.c;
            }
            if (slack_b > 0.0 && lane < nb && lane < MAXS) {
                const NearCand o = ldcg_near(H.nearB + q * MAXS + lane);
                pb = o.c != bw.c && o.g >= lower;
                cb = o.c;
            }
            if (!stay_best && slack_b > 0.0 && lower <= 0.0) flag |= 1;  // "stay" overlaps
        }
        const unsigned ma = __ballot_sync(FULL, pa), mb = __ballot_sync(FULL, pb);
        const unsigned below = (1u << lane) - 1;
        const int nA = __popc(ma), nS = nA + __popc(mb);
        if (nS > MAXS) flag |= 2;
        if (pa && !(flag & 2)) S.N[2 + __popc(ma & below)] = ca;
        if (pb && !(flag & 2)) S.N[2 + nA + __popc(mb & below)] = cb;
        if (lane == 0) {
            S.bs.out = bw;
            S.nS = nS;
            S.flag = flag;
            S.f_old = f_old;
            S.l_old = l_old;
            // back to idle: c_old's slot / entries, the counters
            if (DENSE) {
                H.drec[dq + c_old] = DenseRec{0.0, 0, INT_MAX};
            } else {
                if (so >= 0) {
                    hkeys[base + so] = -1;
                    hvals[base + so] = 0.0;
                    hcnt[base + so] = 0;
                }
                H.sold[q] = -1;
            }
            H.ncnt[q * HCPAD] = 0;
            H.ncnt[q * HCPAD + 1] = 0;
            H.ncnt[q * HCPAD + 2] = 0;  // the pass-item ticket
        }
    }
    __syncthreads();
    const int nS = S.nS, flag = S.flag;
    const Best b = S.bs.out;
    const double f_old = S.f_old;
    const int32_t l_old = S.l_old;
    bool done = false;
    if (A.integral) {
        if (tid == 0) finish_vertex(A, x, c_old, f_old, b.g, b.c, b.e);
        done = true;
    } else if (nS == 0 && !flag) {
        bool moved = b.c != c_old && b.g > 0.0;  // certain: the exact best
        if (moved && ld_state(A.sizes + c_old) == 1 && ld_state(A.sizes + b.c) == 1 &&
            LBL(A.labels, b.c) > LBL(A.labels, c_old))
            moved = false;
        if (!moved || (b.n <= 2 && l_old <= 2)) {  // exact sums: no refold
            if (tid == 0) {
                if (moved)
                    finish_vertex(A, x, c_old, f_old, b.g, b.c, b.e);
                else
                    finish_vertex(A, x, c_old, f_old, 0.0, c_old, 0.0);
            }
            done = true;
        }
    }
    if (done) {
        __syncthreads();
        return;
    }
    if (!(flag & 2)) {
        if (tid == 0) {
            S.N[0] = c_old;
            int nn = 1;
            if (b.c != c_old) S.N[nn++] = b.c;
            for (int t = 0; t < nS; t++) S.N[nn++] = S.N[2 + t];
            S.nn = nn;
        }
        __syncthreads();
        exact_folds<NT, HFU>(A, i, S);
        if (tid == 0) {
            double a_old_excl = dsub(ld_state(A.a_tot + (c_old)), ki);
            Best e{0.0, LBL(A.labels, c_old), c_old, 0.0, 0};
            for (int t = 1; t < S.nn; t++) {
                int32_t c = S.N[t];
                consider(e,
                         gain_of(S.acc[t], S.acc[0], A.m, ki, a_old_excl, ld_state(A.a_tot + (c)),
                                 A.four_m_sq),
                         LBL(A.labels, c), c, S.acc[t], 0);
            }
            finish_vertex(A, x, c_old, S.acc[0], e.g, e.c, e.e);
        }
        __syncthreads();
        return;
    }
    // overflow: ordered folds of the whole row through the (clean) slice
    __syncthreads();
    table_exact<NT>(A, x, i, c_old, ki, hkeys + base, hvals + base,
                      PowTab{(uint32_t)(toff[q + 1] - base - 1)}, S);
}

// Pass block (hub q, table slice y): gains and slack of the slice's entries
// on the any-order sums, the slice's best (incl. "stay"), and every entry
// within slack_max of it -- a superset of the entries that can overlap the
// hub's best -- listed for the decision.  Clears the slice (c_old's slot is
// cleared by the decision, which reads it).
template <bool DENSE>
__global__ void __launch_bounds__(HSB) k_hub_pass(DecideArgs A, const int32_t *list,
                                                 const int64_t *eoff, const int64_t *toff,
                                                 int32_t *hkeys, double *hvals, int32_t *hcnt,
                                                 HubScratch H) {

    pdl_wait();  // the accumulation's sums
    if (single_state(A)) return;
    TR_BEGIN
    __shared__ CertSmem<HSB> S;
    __shared__ int32_t cidx[HSB * HFU];
    __shared__ double cw[HSB * HFU];
    __shared__ int s_last;
    constexpr int PU = DENSE ? 1 : HSU;  // items per thread
    constexpr int PTSL = HSB * PU;        // positions / slots per pass block
    const int tid = threadIdx.x;
    if (tid == 0) {
        S.cidx = cidx;
        S.cw = cw;
    }
    const int64_t pk = H.blk[blockIdx.x];
    const int64_t q = pk >> 32, y = pk & 0xffffffffll;
    const int32_t i = H.vid[q];
    const int32_t c_old = ld_state(A.assign + (i));
    const int64_t base = toff[q];
    const int64_t cap = toff[q + 1] - base;
    const int64_t dq = q * H.dn, deg = eoff[q + 1] - eoff[q];
    const int32_t so = DENSE ? 0 : H.sold[q];
    const double f_old = DENSE ? H.drec[dq + c_old].val : so >= 0 ? hvals[base + so] : 0.0;
    const int32_t l_old = DENSE ? H.drec[dq + c_old].cnt : so >= 0 ? hcnt[base + so] : 0;
    const double ki = A.k[i], a_old_excl = dsub(ld_state(A.a_tot + (c_old)), ki);
    const double inv_m = 1.0 / A.m;
    TR_MARK
    int32_t c[PU];
    double F[PU], g[PU];
    int32_t L[PU];
    float sl[PU];
    const int64_t s0 = y * PTSL + tid;
    double at[PU];
    if (DENSE) {
        // items are row positions; the first position of each community owns
        // it (every load of a position is issued at once, owner or not)
        int32_t cc[PU], mk[PU];
#pragma unroll
        for (int u = 0; u < PU; u++) {
            const int64_t t = s0 + u * HSB;
            cc[u] = t < deg ? H.cbuf[eoff[q] + t] : -1;
        }
#pragma unroll
        for (int u = 0; u < PU; u++) {
            const bool ok = cc[u] >= 0;
            const DenseRec rr = ok ? H.drec[dq + cc[u]] : DenseRec{0.0, 0, -1};
            mk[u] = rr.mk;
            F[u] = rr.val;
            L[u] = rr.cnt;
            at[u] = ok ? __ldg(A.a_tot + cc[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < PU; u++) c[u] = mk[u] == (int32_t)(s0 + u * HSB) ? cc[u] : -1;
    } else {
#pragma unroll
        for (int u = 0; u < PU; u++) {
            const int64_t s = s0 + u * HSB;
            c[u] = s < cap ? hkeys[base + s] : -1;
            F[u] = s < cap ? hvals[base + s] : 0.0;
            L[u] = s < cap ? hcnt[base + s] : 0;
        }
    }
    TR_MARK
    Best b{0.0, LBL(A.labels, c_old), c_old, 0.0, 0};
    unsigned long long nc = 0;
#pragma unroll
    for (int u = 0; u < PU; u++) {  // every gather in flight before any store
        nc += c[u] >= 0;
        if (c[u] == c_old) c[u] = -1;  // not a candidate (its slot stays)
        if (!DENSE) at[u] = c[u] >= 0 ? __ldg(A.a_tot + c[u]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < PU; u++) {
        if (c[u] < 0) continue;
        g[u] = gain_of(F[u], f_old, A.m, ki, a_old_excl, at[u], A.four_m_sq);
        sl[u] = __double2float_ru(gain_slack_r(F[u], L[u], f_old, l_old, inv_m, g[u]));
        consider(b, g[u], LBL(A.labels, c[u]), c[u], F[u], L[u]);
    }
#pragma unroll
    for (int u = 0; u < PU; u++) {
        const int64_t s = s0 + u * HSB;
        if (c[u] < 0) continue;
        if (DENSE) {
            H.drec[dq + c[u]] = DenseRec{0.0, 0, INT_MAX};
        } else {
            hkeys[base + s] = -1;
            hvals[base + s] = 0.0;
            hcnt[base + s] = 0;
        }
    }
    TR_MARK
    b = block_best<HSB>(S.bs, b);
    TR_MARK
    bool wrote = false;
    if (!A.integral) {
        const double thr = b.g - slack_max(ki, eoff[q + 1] - eoff[q], inv_m);
#pragma unroll
        for (int u = 0; u < PU; u++) {
            if (c[u] < 0 || g[u] + (double)sl[u] < thr) continue;
            const int cat = sl[u] > 0.0f ? 0 : 1;
            const int k = atomicAdd(H.ncnt + q * HCPAD + cat, 1);
            if (k < MAXS) (cat ? H.nearB : H.nearA)[q * MAXS + k] = NearCand{c[u], sl[u], g[u]};
            wrote = true;
        }
    }
    if (A.cand) {  // candidate statistic: one atomic per warp
        unsigned long long w = nc;
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(FULL, w, o);
        if ((tid & 31) == 0 && w) atomicAdd(A.cand, w);
    }
    if (tid == 0) {
        H.part[H.poff[q] + y] = b;
        wrote = true;
    }
    // the block finishing the hub's last item decides it (the writers
    // release their partial / near-list stores, one ticket, acquire)
    if (wrote) __threadfence();
    __syncthreads();
    if (tid == 0) {
        const int nsl = (int)(H.poff[q + 1] - H.poff[q]);
        s_last = atomicAdd(H.ncnt + q * HCPAD + 2, 1) == nsl - 1;
        if (s_last) __threadfence();
    }
    __syncthreads();
    TR_MARK
    if (s_last) hub_decide_one<HSB, DENSE>(A, list, toff, hkeys, hvals, hcnt, H, q, S);
    TR_END(2)
}


// ------------------------------------------------- singleton state
//
// The first stage of a phase's first iteration sees the singleton state
// (PL/modularity.py:47-56: assign[v] == v, every community one vertex).  Then
// decide_moves (PL/_kernels.pyx:21-101) needs no aggregation: rows hold
// distinct neighbours, so every neighbour j != i is its own community with
// e_{i->j} = 0.0 + w_ij = w_ij (one term, exact), e_{i->c_old} = 0.0, and the
// decision is the argmax of gain(w_ij) under (gain desc, label asc) against
// "stay" -- the same operands and operations as the general tiers, without
// tables, certification or the hub chain.  These kernels take the stage when
// *notsingle == 0 (launch_single_check: assign[v] == v and sizes[v] == 1 for
// every v); the general ones step aside.

// finish_vertex in the singleton state: both communities of the
// singleton-pair guard (PL/_kernels.pyx:92-98) have size 1 (k_single_check), so
// the guard is the label comparison alone -- no sizes gathers.
__device__ __forceinline__ void finish_single(const DecideArgs &A, int64_t x, int32_t c_old,
                                              double bg, int32_t bc, double be) {
    bool moved = bg > 0.0 && bc != c_old;
    if (moved && LBL(A.labels, bc) > LBL(A.labels, c_old)) moved = false;
    A.out_target[x] = moved ? bc : c_old;
    A.out_moved[x] = moved ? 1 : 0;
    A.out_e_old[x] = 0.0;
    A.out_e_best[x] = moved ? be : 0.0;
}

__device__ __forceinline__ void single_entry(const DecideArgs &A, int32_t i, double ki,
                                             double aoe, int32_t j, double w, Best &b) {
    const double g = gain_of(w, 0.0, A.m, ki, aoe, ld_state(A.a_tot + j), A.four_m_sq);
    consider(b, g, LBL(A.labels, j), j, w, 1);
}

// Tier 0, flattened: a warp takes 32 consecutive tier-0 vertices and walks
// their entries 32 at a time (one entry per lane: row loads adjacent, every
// a_tot gather of the chunk in flight, few registers); a segmented warp
// argmax folds each chunk into the per-vertex bests in shared memory -- the
// argmax is a total order, so its association does not matter.
constexpr int SF_WARPS = 8;
__global__ void __launch_bounds__(SF_WARPS * 32) k_single_t0(DecideArgs A, TierRef L, int64_t cnt) {
    if (!single_state(A)) return;
    __shared__ int s_off[SF_WARPS][33];
    __shared__ Best s_b[SF_WARPS][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long my = 0;
    for (int64_t q0 = ((int64_t)blockIdx.x * SF_WARPS + wid) * 32; q0 < cnt;
         q0 += (int64_t)gridDim.x * SF_WARPS * 32) {
        const int64_t q = q0 + lane;
        const bool has = q < cnt;
        const int32_t i = has ? L.vid[q] : 0;
        const int64_t e0 = has ? L.row[q] : 0;
        const int deg = has ? (int)(L.end[q] - e0) : 0;
        // entry offsets of the 32 vertices (warp exclusive scan)
        int inc = deg;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += y;
        }
        s_off[wid][lane + 1] = inc;
        if (lane == 0) s_off[wid][0] = 0;
        s_b[wid][lane] = Best{0.0, LBL(A.labels, i), i, 0.0, 0};  // "stay"
        __syncwarp();
        const int T = __shfl_sync(FULL, inc, 31);
        for (int c0 = 0; c0 < T; c0 += 32) {
            const int p = c0 + lane;
            int v = 0;  // owner: the last vertex with s_off[v] <= p
            if (p < T) {
                int lo = 0, hi = 32;
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (s_off[wid][mid] <= p)
                        lo = mid;
                    else
                        hi = mid;
                }
                v = lo;
            }
            const int32_t vi = __shfl_sync(FULL, i, v);
            const int64_t ve = __shfl_sync(FULL, e0, v);
            Best b{-INFINITY, INT64_MAX, -1, 0.0, 0};  // neutral
            if (p < T) {
                const int64_t e = ve + (p - s_off[wid][v]);
                const int32_t j = ld_row(A.nbr + e);
                if (j != vi) {
                    const double w = ld_row(A.wts + e);
                    const double ki = A.k[vi];
                    const double aoe = dsub(ld_state(A.a_tot + vi), ki);
                    my++;
                    b = Best{gain_of(w, 0.0, A.m, ki, aoe, ld_state(A.a_tot + j), A.four_m_sq),
                             LBL(A.labels, j), j, w, 1};
                }
            }
            // segmented argmax over the chunk (segments: owners)
            const int vv = p < T ? v : 32;
            for (int o = 1; o < 32; o <<= 1) {
                Best y;
                y.g = __shfl_down_sync(FULL, b.g, o);
                y.l = __shfl_down_sync(FULL, b.l, o);
                y.c = __shfl_down_sync(FULL, b.c, o);
                y.e = __shfl_down_sync(FULL, b.e, o);
                y.n = __shfl_down_sync(FULL, b.n, o);
                const int yv = __shfl_down_sync(FULL, vv, o);
                if (lane + o < 32 && yv == vv) consider(b, y.g, y.l, y.c, y.e, y.n);
            }
            // the first lane of each segment in the chunk now holds its best
            const int pv = __shfl_up_sync(FULL, vv, 1);
            if (vv < 32 && (lane == 0 || pv != vv)) {
                Best h = s_b[wid][vv];
                consider(h, b.g, b.l, b.c, b.e, b.n);
                s_b[wid][vv] = h;
            }
            __syncwarp();
        }
        if (has) {
            const Best b = s_b[wid][lane];
            finish_single(A, L.x[q], i, b.g, b.c, b.e);
        }
        __syncwarp();
    }
    if (A.cand) {
        for (int o = 16; o > 0; o >>= 1) my += __shfl_xor_sync(FULL, my, o);
        if (lane == 0 && my) atomicAdd(A.cand, my);
    }
}

// warp per vertex (tier 1)
__global__ void __launch_bounds__(256) k_single_warp(DecideArgs A, TierRef L, int64_t cnt) {
    if (!single_state(A)) return;
    const int lane = threadIdx.x & 31;
    unsigned long long my = 0;
    for (int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; q < cnt;
         q += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t x = L.x[q];
        const int32_t i = L.vid[q];
        const int64_t e0 = L.row[q], e1 = L.end[q];
        const double ki = A.k[i];
        const double aoe = dsub(ld_state(A.a_tot + i), ki);
        Best b{0.0, LBL(A.labels, i), i, 0.0, 0};
        for (int64_t c0 = e0; c0 < e1; c0 += 128) {
            int32_t jj[4];
            double ww[4], at[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int64_t e = c0 + 32 * u + lane;
                jj[u] = e < e1 ? ld_row(A.nbr + e) : i;
                ww[u] = e < e1 ? ld_row(A.wts + e) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; u++) at[u] = jj[u] != i ? ld_state(A.a_tot + jj[u]) : 0.0;
#pragma unroll
            for (int u = 0; u < 4; u++) {
                if (jj[u] == i) continue;
                my++;
                consider(b, gain_of(ww[u], 0.0, A.m, ki, aoe, at[u], A.four_m_sq),
                         LBL(A.labels, jj[u]), jj[u], ww[u], 1);
            }
        }
        warp_best(b);
        if (lane == 0) finish_single(A, x, i, b.g, b.c, b.e);
    }
    if (A.cand) {
        for (int o = 16; o > 0; o >>= 1) my += __shfl_xor_sync(FULL, my, o);
        if (lane == 0 && my) atomicAdd(A.cand, my);
    }
}

// block per vertex (tiers 2-4, hubs included)
constexpr int SB_NT = 512;
__global__ void __launch_bounds__(SB_NT) k_single_block(DecideArgs A, TierRef L, int64_t cnt) {
    if (!single_state(A)) return;
    __shared__ BestSmem<SB_NT> S;
    unsigned long long my = 0;
    for (int64_t q = blockIdx.x; q < cnt; q += gridDim.x) {
        const int64_t x = L.x[q];
        const int32_t i = L.vid[q];
        const int64_t e0 = L.row[q], e1 = L.end[q];
        const double ki = A.k[i];
        const double aoe = dsub(ld_state(A.a_tot + i), ki);
        Best b{0.0, LBL(A.labels, i), i, 0.0, 0};
        for (int64_t c0 = e0; c0 < e1; c0 += 4 * SB_NT) {
            int32_t jj[4];
            double ww[4], at[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int64_t e = c0 + (int64_t)SB_NT * u + threadIdx.x;
                jj[u] = e < e1 ? ld_row(A.nbr + e) : i;
                ww[u] = e < e1 ? ld_row(A.wts + e) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; u++) at[u] = jj[u] != i ? ld_state(A.a_tot + jj[u]) : 0.0;
#pragma unroll
            for (int u = 0; u < 4; u++) {
                if (jj[u] == i) continue;
                my++;
                consider(b, gain_of(ww[u], 0.0, A.m, ki, aoe, at[u], A.four_m_sq),
                         LBL(A.labels, jj[u]), jj[u], ww[u], 1);
            }
        }
        b = block_best<SB_NT>(S, b);
        if (threadIdx.x == 0) finish_single(A, x, i, b.g, b.c, b.e);
    }
    if (A.cand) {
        for (int o = 16; o > 0; o >>= 1) my += __shfl_xor_sync(FULL, my, o);
        if ((threadIdx.x & 31) == 0 && my) atomicAdd(A.cand, my);
    }
}

// (sizes too: the singleton kernels then know both sizes of the singleton-pair
// guard without gathering them)
__global__ void k_single_check(const int32_t *assign, const int32_t *sizes, int64_t n, int *bad) {
    bool b = false;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x)
        b |= assign[v] != (int32_t)v || sizes[v] != 1;
    if (__syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
}

cudaGraphNode_t add_single_check_nodes(cudaGraph_t g, cudaGraphNode_t dep, const int32_t *assign,
                                       const int32_t *sizes, int64_t n, int *bad) {
    cudaMemsetParams mp = {};
    mp.dst = bad;
    mp.value = 0;
    mp.elementSize = sizeof(int);
    mp.width = 1;
    mp.height = 1;
    cudaGraphNode_t ms, ks;
    PLV_CUDA(cudaGraphAddMemsetNode(&ms, g, &dep, 1, &mp));
    cudaKernelNodeParams kp = {};
    void *args[] = {(void *)&assign, (void *)&sizes, (void *)&n, (void *)&bad};
    kp.func = (void *)k_single_check;
    kp.gridDim = dim3(grid_for(n > 0 ? n : 1, 256, 148 * 16));
    kp.blockDim = dim3(256);
    kp.kernelParams = args;
    PLV_CUDA(cudaGraphAddKernelNode(&ks, g, &ms, 1, &kp));
    count_launch();
    return ks;
}

void launch_single_check(const int32_t *assign, const int32_t *sizes, int64_t n, int *bad,
                         cudaStream_t st) {
    PLV_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
    if (n > 0) {
        k_single_check<<<grid_for(n, 256, 148 * 16), 256, 0, st>>>(assign, sizes, n, bad);
        PLV_LAUNCH_CHECK();
    }
}

static void launch_single_tier(const DecideArgs &A, TierRef L, int64_t cnt, int t,
                               cudaStream_t st) {
    if (!cnt) return;
#ifndef PLV_SINGLE_FLAT_MAXT
#define PLV_SINGLE_FLAT_MAXT 1  // tiers decided by the flattened kernel (0..this)
#endif
    if (t <= PLV_SINGLE_FLAT_MAXT)
        k_single_t0<<<grid_for(cnt, SF_WARPS * 32), SF_WARPS * 32, 0, st>>>(A, L, cnt);
    else if (t == 1)
        k_single_warp<<<grid_for(cnt, 8), 256, 0, st>>>(A, L, cnt);
    else
        k_single_block<<<grid_for(cnt, 1, 148 * 8), SB_NT, 0, st>>>(A, L, cnt);
    PLV_LAUNCH_CHECK();
}

}  // namespace plv
#include "ahead.cuh"
namespace plv {

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
        uint32_t t = d <= T0_MAXD    ? 0
                     : d <= T1_MAXD  ? 1
                     : d <= T2A_MAXD ? 2
                     : d <= T2_MAXD  ? 3
                                     : 4;
        uint32_t kk = (uint32_t)(a * NTIER + t);
        key[g] = kk;
        // one atomic per (warp, bucket): a stage's tier-0 bucket takes millions
        const unsigned act = __activemask();
        const unsigned grp = __match_any_sync(act, kk);
        if ((threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(hist + kk, (unsigned long long)__popc(grp));
    }
}

__global__ void k_tier_local(const uint32_t *skey, const int32_t *sidx, const int64_t *stage_off,
                             int64_t total, const int64_t *off, const int32_t *vtx, int32_t *local,
                             int32_t *vid, int64_t *row, int64_t *end) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < total;
         p += (int64_t)gridDim.x * blockDim.x) {
        local[p] = (int32_t)(sidx[p] - stage_off[skey[p] / NTIER]);
        const int32_t i = vtx[sidx[p]];
        vid[p] = i;
        row[p] = off[i];
        end[p] = off[i + 1];
    }
}

__global__ void k_hub_degrees(const int64_t *off, const int32_t *vtx, const int64_t *stage_off,
                              const int32_t *local, const int64_t *hub_pos, const int64_t *hub_stage,
                              int64_t nh, int64_t *deg, int64_t *row, int32_t *vid) {
    for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < nh;
         h += (int64_t)gridDim.x * blockDim.x) {
        int32_t i = vtx[stage_off[hub_stage[h]] + local[hub_pos[h]]];
        deg[h] = off[i + 1] - off[i];
        row[h] = off[i];
        vid[h] = i;
    }
}

__global__ void k_fill_drec(DenseRec *p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = DenseRec{0.0, 0, INT_MAX};
}

__global__ void k_fill_i32_d(int32_t *p, int64_t n, int32_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

void Plan::release() {
    cudaDeviceSynchronize();  // buffers go back to the pool idle
    void *ps[] = {tier_list, tier_vid, tier_row, tier_end, hub_eoff, hub_toff, hub_poff, hub_blk, hub_row, hub_vid, hkeys,
                  hvals,     hcnt,     hsold,    hncnt,    hnear,   hpart,
                  drec,      cbuf};
    for (void *p : ps)
        pool_free(p);
    tier_list = nullptr;
    tier_vid = nullptr;
    tier_row = tier_end = nullptr;
    hub_eoff = hub_toff = hub_poff = hub_blk = hub_row = nullptr;
    hub_vid = nullptr;
    hkeys = hcnt = hsold = hncnt = nullptr;
    hvals = nullptr;
    hnear = nullptr;
    hpart = nullptr;
    drec = nullptr;
    cbuf = nullptr;
    if (ah) {
        ah->release();
        delete ah;
        ah = nullptr;
    }
}

void plan_build(Plan &P, const int64_t *off, const int32_t *vtx, const int64_t *stage_off_h,
                int64_t nst, int64_t n, cudaStream_t s, const int32_t *nbr, const double *wts,
                bool ahead_ok) {
    int64_t total = stage_off_h[nst];
    P.st.assign(nst, StagePlan{});
    for (int64_t a = 0; a < nst; a++) {
        P.st[a].off = stage_off_h[a];
        P.st[a].ns = stage_off_h[a + 1] - stage_off_h[a];
    }
    P.tier_list = dalloc<int32_t>(total);
    if (total == 0) return;
    Buf<int64_t> d_soff(nst + 1, s);
    PLV_CUDA(cudaMemcpyAsync(d_soff.get(), stage_off_h, sizeof(int64_t) * (nst + 1),
                             cudaMemcpyHostToDevice, s));
    Buf<uint32_t> key(total, s), skey(total, s);
    Buf<int32_t> gidx(total, s), sidx(total, s);
    Buf<unsigned long long> hist(NTIER * nst, s);
    PLV_CUDA(cudaMemsetAsync(hist.get(), 0, sizeof(unsigned long long) * NTIER * nst, s));
    k_tier_keys<<<grid_for(total, 256), 256, 0, s>>>(off, vtx, d_soff, nst, total, key, hist);
    PLV_LAUNCH_CHECK();
    iota_i32(gidx, total, s);
    sort_pairs<uint32_t, int32_t>(key, skey, gidx, sidx, total, 0, bits_for(NTIER * nst + NTIER), s);
    P.tier_vid = dalloc<int32_t>(total);
    P.tier_row = dalloc<int64_t>(total);
    P.tier_end = dalloc<int64_t>(total);
    k_tier_local<<<grid_for(total, 256), 256, 0, s>>>(skey, sidx, d_soff, total, off, vtx,
                                                      P.tier_list, P.tier_vid, P.tier_row,
                                                      P.tier_end);
    PLV_LAUNCH_CHECK();
    std::vector<unsigned long long> h(NTIER * nst);
    PLV_CUDA(cudaMemcpyAsync(h.data(), hist.get(), sizeof(unsigned long long) * NTIER * nst,
                             cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    // dense hub arrays: as many per-stage slots as 4 GB allows, at most HUB_DENSE_KMAX
    P.dense_k = n > 0 ? (int64_t)(4e9 / (16.0 * (double)n)) : 0;
    if (P.dense_k > HUB_DENSE_KMAX) P.dense_k = HUB_DENSE_KMAX;
    int64_t pos = 0;
    std::vector<int64_t> hub_pos, hub_stage;
    for (int64_t a = 0; a < nst; a++) {
        StagePlan &sp = P.st[a];
        for (int t = 0; t < NTIER; t++) {
            sp.tstart[t] = pos;
            sp.tcount[t] = (int64_t)h[NTIER * a + t];
            pos += sp.tcount[t];
        }
    }
    // small high-degree stages of an integral coloured phase: ahead tables
    if (ahead_ok && nbr && wts) ahead_plan(P, off, nbr, wts, vtx, stage_off_h, d_soff, nst, n, s);
    for (int64_t a = 0; a < nst; a++) {
        StagePlan &sp = P.st[a];
        if (sp.ahead) {
            for (int t = 0; t < NTIER; t++) sp.tcount[t] = 0;
            continue;
        }
        // a small colour class with hubs: its block-tier vertices join the
        // hub tier (their lists directly precede it) -- one vertex per block
        // is a long serial chain, the hub tier spreads every row over the GPU
        const int64_t nb = sp.tcount[2] + sp.tcount[3];
        if (sp.tcount[4] && nb && nb + sp.tcount[4] <= P.dense_k) {
            sp.tstart[4] = sp.tstart[2];
            sp.tcount[4] += nb;
            sp.tcount[2] = sp.tcount[3] = 0;
        }
        for (int64_t z = 0; z < sp.tcount[4]; z++) {
            hub_pos.push_back(sp.tstart[4] + z);
            hub_stage.push_back(a);
        }
    }
    int64_t nh = (int64_t)hub_pos.size();
    if (nh == 0) return;
    Buf<int64_t> d_hpos(nh, s), d_hst(nh, s), d_deg(nh, s), d_row(nh, s);
    Buf<int32_t> d_vid(nh, s);
    PLV_CUDA(cudaMemcpyAsync(d_hpos.get(), hub_pos.data(), sizeof(int64_t) * nh,
                             cudaMemcpyHostToDevice, s));
    PLV_CUDA(cudaMemcpyAsync(d_hst.get(), hub_stage.data(), sizeof(int64_t) * nh,
                             cudaMemcpyHostToDevice, s));
    k_hub_degrees<<<grid_for(nh, 256), 256, 0, s>>>(off, vtx, d_soff, P.tier_list, d_hpos, d_hst,
                                                   nh, d_deg, d_row, d_vid);
    PLV_LAUNCH_CHECK();
    std::vector<int64_t> deg(nh), row(nh);
    std::vector<int32_t> vid(nh);
    PLV_CUDA(cudaMemcpyAsync(deg.data(), d_deg.get(), sizeof(int64_t) * nh, cudaMemcpyDeviceToHost,
                             s));
    PLV_CUDA(cudaMemcpyAsync(row.data(), d_row.get(), sizeof(int64_t) * nh, cudaMemcpyDeviceToHost,
                             s));
    PLV_CUDA(cudaMemcpyAsync(vid.data(), d_vid.get(), sizeof(int32_t) * nh, cudaMemcpyDeviceToHost,
                             s));
    PLV_CUDA(cudaStreamSynchronize(s));
    std::vector<int64_t> eoff, toff, poff, blk, hrow;
    std::vector<int32_t> hvid;
    int64_t h0 = 0, max_parts = 1;
    for (int64_t a = 0; a < nst; a++) {
        StagePlan &sp = P.st[a];
        sp.hub_base = (int64_t)eoff.size();
        sp.hub_blk_base = (int64_t)blk.size();
        int64_t acc = 0, tacc = 0, pacc = 0;
        eoff.push_back(0);
        toff.push_back(0);
        poff.push_back(0);
        // few hubs: dense per-hub community arrays (no claims), items are row
        // positions; else hash tables, items are table slices
        sp.hub_dense = sp.tcount[4] > 0 && sp.tcount[4] <= P.dense_k;
        for (int64_t z = 0; z < sp.tcount[4]; z++) {
            int64_t d = deg[h0 + z];
            int64_t cap = 64;
            while (cap < 2 * d + 2) cap <<= 1;
            int64_t sl = sp.hub_dense ? (d + HSB - 1) / HSB : (cap + HTSL - 1) / HTSL;
            for (int64_t y = 0; y < sl; y++) blk.push_back((z << 32) | y);
            acc += d;
            tacc += cap;
            pacc += sl;
            eoff.push_back(acc);
            toff.push_back(tacc);
            poff.push_back(pacc);
            hrow.push_back(row[h0 + z]);
            hvid.push_back(vid[h0 + z]);
        }
        hrow.push_back(0);  // indexed like eoff
        hvid.push_back(0);
        h0 += sp.tcount[4];
        sp.hub_entries = acc;
        sp.hub_nblk = pacc;
        max_parts = pacc > max_parts ? pacc : max_parts;
        P.max_hub_entries = acc > P.max_hub_entries ? acc : P.max_hub_entries;
        if (sp.hub_dense) P.max_dense_entries = acc > P.max_dense_entries ? acc : P.max_dense_entries;
        P.max_hubs = sp.tcount[4] > P.max_hubs ? sp.tcount[4] : P.max_hubs;
        P.max_table = tacc > P.max_table ? tacc : P.max_table;
    }
    P.hub_eoff = dalloc<int64_t>(eoff.size());
    P.hub_toff = dalloc<int64_t>(toff.size());
    P.hub_poff = dalloc<int64_t>(poff.size());
    P.hub_blk = dalloc<int64_t>(blk.size());
    P.hub_row = dalloc<int64_t>(hrow.size());
    P.hub_vid = dalloc<int32_t>(hvid.size());
    PLV_CUDA(cudaMemcpyAsync(P.hub_row, hrow.data(), sizeof(int64_t) * hrow.size(),
                             cudaMemcpyHostToDevice, s));
    PLV_CUDA(cudaMemcpyAsync(P.hub_vid, hvid.data(), sizeof(int32_t) * hvid.size(),
                             cudaMemcpyHostToDevice, s));
    PLV_CUDA(cudaMemcpyAsync(P.hub_eoff, eoff.data(), sizeof(int64_t) * eoff.size(),
                             cudaMemcpyHostToDevice, s));
    PLV_CUDA(cudaMemcpyAsync(P.hub_toff, toff.data(), sizeof(int64_t) * toff.size(),
                             cudaMemcpyHostToDevice, s));
    PLV_CUDA(cudaMemcpyAsync(P.hub_poff, poff.data(), sizeof(int64_t) * poff.size(),
                             cudaMemcpyHostToDevice, s));
    PLV_CUDA(cudaMemcpyAsync(P.hub_blk, blk.data(), sizeof(int64_t) * blk.size(),
                             cudaMemcpyHostToDevice, s));
    int64_t T = P.max_table;
    P.hkeys = dalloc<int32_t>(T);
    P.hvals = dalloc<double>(T);
    P.hcnt = dalloc<int32_t>(T);
    k_fill_i32_d<<<grid_for(T, 256), 256, 0, s>>>(P.hkeys, T, -1);
    PLV_LAUNCH_CHECK();
    PLV_CUDA(cudaMemsetAsync(P.hvals, 0, sizeof(double) * T, s));
    PLV_CUDA(cudaMemsetAsync(P.hcnt, 0, sizeof(int32_t) * T, s));
    int64_t H = P.max_hubs;
    P.hsold = dalloc<int32_t>(H);
    k_fill_i32_d<<<grid_for(H, 256), 256, 0, s>>>(P.hsold, H, -1);
    PLV_LAUNCH_CHECK();
    P.hncnt = dalloc<int32_t>(HCPAD * H);
    PLV_CUDA(cudaMemsetAsync(P.hncnt, 0, sizeof(int32_t) * HCPAD * H, s));
    P.hnear = dalloc<NearCand>(2 * H * MAXS);
    if (P.max_dense_entries) {
        P.dn = n;
        const int64_t D = P.dense_k * n;
        P.drec = dalloc<DenseRec>(D);
        P.cbuf = dalloc<int32_t>(P.max_dense_entries);
        k_fill_drec<<<grid_for(D, 256), 256, 0, s>>>(P.drec, D);
        PLV_LAUNCH_CHECK();
    }
    P.hpart = dalloc<Best>(max_parts);
    PLV_CUDA(cudaStreamSynchronize(s));
}

static size_t t2_smem(int ts) { return (sizeof(double) + 2 * sizeof(int32_t)) * ts; }

void ensure_decide_attrs() {
    static int dev_done = -1;
    int dev;
    PLV_CUDA(cudaGetDevice(&dev));
    if (dev_done == dev) return;
    PLV_CUDA(cudaFuncSetAttribute(k_decide_t2<T2A_TS, T2A_MAXD, T2A_NT>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)t2_smem(T2A_TS)));
    PLV_CUDA(cudaFuncSetAttribute(k_decide_t2<T2_TS, T2_MAXD, BLK>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)t2_smem(T2_TS)));
    PLV_CUDA(cudaFuncSetAttribute(k_decide_t2<T2A_TS, T2A_MAXD, 512>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)t2_smem(T2A_TS)));
    PLV_CUDA(cudaFuncSetAttribute(k_decide_t2<T2_TS, T2_MAXD, 1024>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)t2_smem(T2_TS)));
    dev_done = dev;
}

void launch_decide(const Plan &P, int64_t a, DecideArgs A, cudaStream_t st) {
    cudaStream_t ts[NTIER] = {st, st, st, st, st};
    launch_decide_tiers(P, a, A, ts);
}

static bool launch_small_t01(const Plan &P, int64_t a, const DecideArgs &A, cudaStream_t st);

void launch_decide_par(const Plan &P, int64_t a, DecideArgs A, cudaStream_t st,
                       const cudaStream_t *side, cudaEvent_t fork, const cudaEvent_t *join) {
    // tier t < NTIER - 1 on its own stream side[t]; the hubs on `st`
    if (launch_small_t01(P, a, A, st)) return;
    const StagePlan &sp = P.st[a];
    cudaStream_t ts[NTIER] = {st, st, st, st, st};
    bool forked = false;
    for (int t = 0; t < NTIER - 1; t++) {
        if (!sp.tcount[t]) continue;
        if (!forked) PLV_CUDA(cudaEventRecord(fork, st));
        forked = true;
        PLV_CUDA(cudaStreamWaitEvent(side[t], fork, 0));
        ts[t] = side[t];
    }
    launch_decide_tiers(P, a, A, ts);
    for (int t = 0; t < NTIER - 1; t++) {
        if (!sp.tcount[t]) continue;
        PLV_CUDA(cudaEventRecord(join[t], side[t]));
        PLV_CUDA(cudaStreamWaitEvent(st, join[t], 0));
    }
}

static TierRef tier_ref(const Plan &P, const StagePlan &sp, int t) {
    const int64_t o = sp.tstart[t];
    return TierRef{P.tier_list + o, P.tier_vid + o, P.tier_row + o, P.tier_end + o};
}

constexpr int64_t T01_FUSE_MAX = 65536;  // vertices of a stage decided by k_decide_t01

static bool launch_small_t01(const Plan &P, int64_t a, const DecideArgs &A, cudaStream_t st) {
    const StagePlan &sp = P.st[a];
    if (sp.tcount[2] || sp.tcount[3] || sp.tcount[4]) return false;
    const int64_t tot = sp.tcount[0] + sp.tcount[1];
    if (!tot || tot > T01_FUSE_MAX) return false;
    const int nb0 = sp.tcount[0] ? (int)grid_for(sp.tcount[0], 256) : 0;
    const int nb1 = sp.tcount[1] ? (int)grid_for(sp.tcount[1], 8) : 0;  // 8 warps per block
    launch_pdl(k_decide_t01, nb0 + nb1, 256, 0, st, A, tier_ref(P, sp, 0), sp.tcount[0],
               tier_ref(P, sp, 1), sp.tcount[1], nb0);
    if (A.notsingle)
        for (int t = 0; t < 2; t++) launch_single_tier(A, tier_ref(P, sp, t), sp.tcount[t], t, st);
    return true;
}

void launch_decide_tiers(const Plan &P, int64_t a, DecideArgs A, const cudaStream_t *ts) {
    const StagePlan &sp = P.st[a];
    if (sp.ahead) {
        ahead_launch_decide(P, a, A, ts[NTIER - 1]);
        return;
    }
    if (sp.tcount[0]) {
        k_decide_t0<<<grid_for(sp.tcount[0], 256), 256, 0, ts[0]>>>(A, tier_ref(P, sp, 0),
                                                                    sp.tcount[0]);
        PLV_LAUNCH_CHECK();
    }
    if (sp.tcount[1]) {
        k_decide_t1<<<grid_for(sp.tcount[1], T1_WARPS), T1_WARPS * 32, 0, ts[1]>>>(
            A, tier_ref(P, sp, 1), sp.tcount[1]);
        PLV_LAUNCH_CHECK();
    }
    // few vertices (a late colour class): one wide block each, so a vertex's
    // latency-bound rounds shrink; many: narrow blocks, more vertices per SM
    if (sp.tcount[2] > T2_WIDE_MAX) {
        k_decide_t2<T2A_TS, T2A_MAXD, T2A_NT><<<grid_for(sp.tcount[2], 1, 1 << 30), T2A_NT,
                                             t2_smem(T2A_TS), ts[2]>>>(
            A, tier_ref(P, sp, 2), sp.tcount[2]);
        PLV_LAUNCH_CHECK();
    } else if (sp.tcount[2]) {
        k_decide_t2<T2A_TS, T2A_MAXD, 512><<<(unsigned)sp.tcount[2], 512, t2_smem(T2A_TS), ts[2]>>>(
            A, tier_ref(P, sp, 2), sp.tcount[2]);
        PLV_LAUNCH_CHECK();
    }
    if (sp.tcount[3] > T2_WIDE_MAX) {
        k_decide_t2<T2_TS, T2_MAXD, BLK><<<grid_for(sp.tcount[3], 1, 1 << 30), BLK,
                                           t2_smem(T2_TS), ts[3]>>>(
            A, tier_ref(P, sp, 3), sp.tcount[3]);
        PLV_LAUNCH_CHECK();
    } else if (sp.tcount[3]) {
        k_decide_t2<T2_TS, T2_MAXD, 1024><<<(unsigned)sp.tcount[3], 1024, t2_smem(T2_TS), ts[3]>>>(
            A, tier_ref(P, sp, 3), sp.tcount[3]);
        PLV_LAUNCH_CHECK();
    }
    if (A.notsingle)  // a first stage: the singleton kernels, after each tier's own
        for (int t = 0; t < NTIER; t++)
            launch_single_tier(A, tier_ref(P, sp, t), sp.tcount[t], t, ts[t]);
    cudaStream_t st = ts[4];
    if (sp.tcount[4]) {
        const int32_t *list = P.tier_list + sp.tstart[4];
        const int64_t *eoff = P.hub_eoff + sp.hub_base;
        const int64_t *toff = P.hub_toff + sp.hub_base;
        int64_t nh = sp.tcount[4], E = sp.hub_entries;
        const int64_t Hm = P.max_hubs;
        HubScratch H{P.hub_row + sp.hub_base,
                     P.hub_vid + sp.hub_base,
                     P.hsold,
                     P.hncnt,
                     (NearCand *)P.hnear,
                     (NearCand *)P.hnear + Hm * MAXS,
                     P.hpart,
                     P.hub_blk + sp.hub_blk_base,
                     P.hub_poff + sp.hub_base,
                     nh,
                     P.drec,
                     P.cbuf,
                     P.dn};
        unsigned g2 = (unsigned)sp.hub_nblk;
        if (sp.hub_dense) {
            launch_pdl(k_hub_accum<true>, grid_for(E, 256), 256, 0, st, A, eoff, toff, nh, E,
                       P.hkeys, P.hvals, P.hcnt, H);
            launch_pdl(k_hub_pass<true>, g2, HSB, 0, st, A, list, eoff, toff, P.hkeys, P.hvals,
                       P.hcnt, H);
        } else {
            launch_pdl(k_hub_accum<false>, grid_for(E, 256), 256, 0, st, A, eoff, toff, nh, E,
                       P.hkeys, P.hvals, P.hcnt, H);
            launch_pdl(k_hub_pass<false>, g2, HSB, 0, st, A, list, eoff, toff, P.hkeys, P.hvals,
                       P.hcnt, H);
        }
    }
}

void ahead_stats(const Plan &P, int64_t *out) {
    for (int t = 0; t < 5; t++) out[t] = 0;
    if (!P.ah) return;
    for (const StagePlan &sp : P.st) out[0] += sp.ahead;
    out[1] = P.ah->nvert;
    out[2] = (int64_t)P.ah->wins.size();
    out[3] = P.ah->nfix;
    out[4] = P.ah->nslots;
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
    A.inv_m = 1.0 / m;
    A.inv_f = 1.0 / A.four_m_sq;
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
    Plan P;
    int64_t soff[2] = {0, ns};
    Buf<unsigned long long> cand(1, s);
    PLV_CUDA(cudaMemsetAsync(cand.get(), 0, sizeof(unsigned long long), s));
    try {
        plan_build(P, off, subset, soff, 1, 0, s);
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

// Debug timeline: plv_debug_trace(on) enables / disables recording (and
// resets the buffer); plv_debug_trace_read copies n records of 8 u64:
// [kernel id << 32 | block, stamps t0..t5, number of stamps].
extern "C" int plv_debug_trace(int on) {
    unsigned int z = 0;
    if (cudaMemcpyToSymbol(plv::g_tr_on, &on, sizeof(int)) != cudaSuccess) return -4;
    if (cudaMemcpyToSymbol(plv::g_tr_n, &z, sizeof(z)) != cudaSuccess) return -4;
    return 0;
}

extern "C" int plv_debug_trace_read(unsigned long long *out, int64_t max_records, int64_t *n) {
    unsigned int cnt = 0;
    if (cudaMemcpyFromSymbol(&cnt, plv::g_tr_n, sizeof(cnt)) != cudaSuccess) return -4;
    int64_t m = cnt;
    if (m > (1 << 21) / 8) m = (1 << 21) / 8;
    if (m > max_records) m = max_records;
    if (m && cudaMemcpyFromSymbol(out, plv::g_tr, sizeof(unsigned long long) * 8 * m) != cudaSuccess)
        return -4;
    *n = m;
    return 0;
}
