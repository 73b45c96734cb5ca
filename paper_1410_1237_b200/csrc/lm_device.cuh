// lm_device.cuh -- device pieces of local moving shared by decide.cu,
// apply.cu and phase_small.cu: the gain and argmax order of decide_moves
// (PL/_kernels.pyx:77-98), tier 0's exact per-vertex decide, and apply's
// live communities and per-mover deltas (PL/_kernels.pyx:104-145).
#pragma once
#include "localmove.cuh"
#include <cub/cub.cuh>

namespace plv {

#ifndef T0_INPLACE
#define T0_INPLACE 0
#endif
#ifndef T0_FILTER
#define T0_FILTER 1  // approximate gains select the candidates evaluated exactly
#endif

__device__ __forceinline__ int64_t LBL(const int32_t *labels, int32_t c) {
    return labels ? (int64_t)labels[c] : (int64_t)c;
}

// Community hash of the decide tables: murmur3's 32-bit finaliser (community
// ids of a hub's neighbours share low bits, so a plain multiplicative hash
// clusters).
__device__ __forceinline__ uint32_t comm_hash(int32_t c) {
    uint32_t h = (uint32_t)c;
    h ^= h >> 16;
    h *= 0x85EBCA6Bu;
    h ^= h >> 13;
    h *= 0xC2B2AE35u;
    h ^= h >> 16;
    return h;
}

// Ahead tables (ahead.cuh): `cap` slots (any size: multiply-shift range
// reduction of the hash, linear probing).  Find-or-insert community c by CAS
// alone; reports whether this call inserted the key.  The table always keeps
// an empty slot.
__device__ __forceinline__ uint32_t ahead_first(int32_t c, uint32_t cap) {
    return (uint32_t)(((uint64_t)comm_hash(c) * cap) >> 32);
}
__device__ __forceinline__ uint32_t ahead_claim(AheadRec *t, int32_t c, uint32_t cap, bool *fresh) {
    uint32_t s = ahead_first(c, cap);
    while (true) {
        const int32_t old = atomicCAS(&t[s].key, -1, c);
        if (old == -1 || old == c) {
            *fresh = old == -1;
            return s;
        }
        s = s + 1 == cap ? 0 : s + 1;
    }
}

// One fix entry per thread: the ahead vertex `src` of this stage moved from
// community a to b, so its weight in the table of the later ahead vertex
// `dst` moves with it (exact: integral weights).  b's slot may be new; if b is
// dst's own community, dst's c_old slot is recorded.
__device__ __forceinline__ void ahead_fixup(const AheadFix &F, unsigned blk) {
    const int64_t e = (int64_t)(blk - F.pb) * blockDim.x + threadIdx.x;
    if (e >= F.n) return;
    const int32_t src = F.src[e];
    const int2 mv = __ldcg(F.amove + src);
    if (mv.x < 0) return;
    const int32_t dst = F.dst[e];
    const double w = F.w[e];
    AheadRec *t = F.tab + F.tbase[dst];
    const uint32_t cap = F.tcap[dst];
    uint32_t s = ahead_first(mv.x, cap);
    for (uint32_t it = 0; it < cap; it++) {  // a's slot exists: src was counted there
        if (__ldcg(&t[s].key) == mv.x) break;
        s = s + 1 == cap ? 0 : s + 1;
    }
    atomicAdd(&t[s].val, -w);
    bool fresh;
    const uint32_t s2 = ahead_claim(t, mv.y, cap, &fresh);
    atomicAdd(&t[s2].val, w);
    if (fresh && mv.y == F.cold[dst]) F.sold[dst] = (int32_t)s2;
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

// Final decision of PL/_kernels.pyx:92-98.
__device__ __forceinline__ void finish_vertex(const DecideArgs &A, int64_t x, int32_t c_old,
                                              double e_old, double bg, int32_t bc, double be) {
    bool moved = bg > 0.0 && bc != c_old;
    if (moved && ld_state(A.sizes + c_old) == 1 && ld_state(A.sizes + bc) == 1 &&
        LBL(A.labels, bc) > LBL(A.labels, c_old))
        moved = false;  // singleton-pair guard
    A.out_target[x] = moved ? bc : c_old;
    A.out_moved[x] = moved ? 1 : 0;
    A.out_e_old[x] = e_old;
    A.out_e_best[x] = moved ? be : e_old;
}

struct Best {
    double g;
    int64_t l;
    int32_t c;
    double e;
    int32_t n;  // term count of e (certification)
};

__device__ __forceinline__ void consider(Best &b, double g, int64_t l, int32_t c, double e,
                                         int32_t n) {
    if (better(g, l, b.g, b.l)) b = Best{g, l, c, e, n};
}

// A tier's vertices: stage-local index x (outputs), vertex i, row [row, end),
// laid out by the plan so a kernel's first loads are coalesced and independent.
struct TierRef {
    const int32_t *x;
    const int32_t *vid;
    const int64_t *row, *end;
};

// Tier 0 over blocks [b, b + nb) of the launch (a thread per vertex).
__device__ __forceinline__ void decide_t0_body(const DecideArgs &A, const TierRef &L, int64_t cnt,
                                               int64_t b, int64_t nb) {
    unsigned long long my_cand = 0;
    for (int64_t q = b * (int64_t)blockDim.x + threadIdx.x; q < cnt;
         q += nb * (int64_t)blockDim.x) {
        const int64_t x = L.x[q];
        const int32_t i = L.vid[q];
        const int64_t e0 = L.row[q];
        const int deg = (int)(L.end[q] - e0);
        const int32_t c_old = ld_state(A.assign + (i));
        // all row loads, then all community loads, in flight together
        int32_t jj[T0_MAXD], cc[T0_MAXD];
        double ww[T0_MAXD];
#pragma unroll
        for (int t = 0; t < T0_MAXD; t++) {
            jj[t] = t < deg ? ld_row(A.nbr + (e0 + t)) : i;
            ww[t] = t < deg ? ld_row(A.wts + (e0 + t)) : 0.0;
        }
#pragma unroll
        for (int t = 0; t < T0_MAXD; t++) cc[t] = jj[t] != i ? ld_state(A.assign + jj[t]) : -1;
#if T0_INPLACE
        // in place: a "head" is the first entry of its community; its weight
        // becomes the community's sum folded forward in adjacency order
        // (0.0 + w_first + ... is w_first + ...; PL/_kernels.pyx:64-75)
        bool head[T0_MAXD];
        int nc = 0;
#pragma unroll
        for (int t = 0; t < T0_MAXD; t++) {
            bool h = t < deg && cc[t] >= 0;
#pragma unroll
            for (int u = 0; u < t; u++) h = h && cc[u] != cc[t];
            head[t] = h;
            if (h) {
                double v = ww[t];
#pragma unroll
                for (int u = t + 1; u < T0_MAXD; u++)
                    if (u < deg && cc[u] == cc[t]) v = dadd(v, ww[u]);
                ww[t] = v;
                nc++;
            }
        }
        my_cand += nc;
        double e_old = 0.0;
#pragma unroll
        for (int t = 0; t < T0_MAXD; t++)
            if (head[t] && cc[t] == c_old) e_old = ww[t];
        double ki = A.k[i];
        double a_old_excl = dsub(ld_state(A.a_tot + (c_old)), ki);
        Best b{0.0, LBL(A.labels, c_old), c_old, 0.0, 0};
#pragma unroll
        for (int t = 0; t < T0_MAXD; t++) {
            if (head[t] && cc[t] != c_old) {
                int32_t c = cc[t];
                consider(b, gain_of(ww[t], e_old, A.m, ki, a_old_excl, ld_state(A.a_tot + c),
                                    A.four_m_sq),
                         LBL(A.labels, c), c, ww[t], 0);
            }
        }
#else
        int32_t keys[T0_MAXD];
        double vals[T0_MAXD];
        int nc = 0;
#pragma unroll
        for (int t = 0; t < T0_MAXD; t++) {
            if (t < deg) {
                if (cc[t] >= 0) {
                    const int32_t c = cc[t];
                    const double w = ww[t];
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
        double a_old_excl = dsub(ld_state(A.a_tot + (c_old)), ki);
        Best b{0.0, LBL(A.labels, c_old), c_old, 0.0, 0};
#if T0_FILTER
        // The exact gain costs two float64 divisions per candidate (a quarter
        // of this kernel's stall samples).  Approximate gains first
        // (reciprocal multiplies: the sums and products are the exact ones,
        // each quotient is within 3 ulp and the final sum within 2, so the
        // exact gain lies within gm of ga); only a candidate that can still be
        // the exact best, or tie with it, is evaluated exactly:
        //   exact best k with g_k > 0:  ga_k + gm_k >= g_k >= g_j >= ga_j - gm_j
        // for every j, and g_k > 0 bounds from below too.  A best with
        // g_k <= 0 never moves the vertex (finish_vertex), with or without it.
        double at[T0_MAXD];
#pragma unroll
        for (int s = 0; s < T0_MAXD; s++)
            at[s] = s < nc && keys[s] != c_old ? ld_state(A.a_tot + keys[s]) : 0.0;
        const double tk = dmul(2.0, ki), tka = dmul(tk, a_old_excl);
        double lo = 0.0;
#pragma unroll
        for (int s = 0; s < T0_MAXD; s++) {
            if (s < nc && keys[s] != c_old) {
                const double t2 = dsub(vals[s], e_old) * A.inv_m;
                const double t3 = dsub(tka, dmul(tk, at[s])) * A.inv_f;
                lo = fmax(lo, (t2 + t3) - (1.8e-15 * (fabs(t2) + fabs(t3)) + 1e-300));
            }
        }
#pragma unroll
        for (int s = 0; s < T0_MAXD; s++) {
            if (s < nc && keys[s] != c_old) {
                const double t2 = dsub(vals[s], e_old) * A.inv_m;
                const double t3 = dsub(tka, dmul(tk, at[s])) * A.inv_f;
                if ((t2 + t3) + (1.8e-15 * (fabs(t2) + fabs(t3)) + 1e-300) < lo) continue;
                int32_t c = keys[s];
                consider(b, gain_of(vals[s], e_old, A.m, ki, a_old_excl, at[s], A.four_m_sq),
                         LBL(A.labels, c), c, vals[s], 0);
            }
        }
#else
#pragma unroll
        for (int s = 0; s < T0_MAXD; s++) {
            if (s < nc && keys[s] != c_old) {
                int32_t c = keys[s];
                consider(b, gain_of(vals[s], e_old, A.m, ki, a_old_excl, ld_state(A.a_tot + (c)), A.four_m_sq),
                         LBL(A.labels, c), c, vals[s], 0);
            }
        }
#endif
#endif
        finish_vertex(A, x, c_old, e_old, b.g, b.c, b.e);
    }
    if (A.cand) {
        typedef cub::BlockReduce<unsigned long long, 256> BR;
        __shared__ typename BR::TempStorage tmp;
        unsigned long long tot = BR(tmp).Sum(my_cand);
        if (threadIdx.x == 0 && tot) atomicAdd(A.cand, tot);
    }
}

// Live community of neighbour j for the mover at subset index x.
__device__ __forceinline__ int32_t live_comm(const StageArgs &A, int32_t j, int64_t x) {
    int64_t p = (A.flags & PLV_F_IDENTITY) ? (int64_t)j : (int64_t)A.pos[j];
    if (p >= 0 && p < x && A.moved[p]) return A.target[p];
    return A.assign[j];
}

// Deltas of one mover: 2 e_a + 2 sw leaving a, 2 e_b + 2 sw joining b (the
// reference's `w_int[a] -= 2.0 * e_a + 2.0 * sw`, PL/_kernels.pyx:137-142),
// stored for the ordered fold, or added with atomics for integral graphs;
// sizes are integers either way.
__device__ __forceinline__ void mover_deltas(const StageArgs &A, int64_t x, int32_t i, int32_t a,
                                             int32_t b, double e_a, double e_b, bool integral) {
    if (A.live_a) {  // live-only pass: the folds are the product
        A.live_a[x] = e_a;
        A.live_b[x] = e_b;
        return;
    }
    double sw = A.selfw[i], ki = A.k[i];
    double ta = dadd(dmul(2.0, e_a), dmul(2.0, sw));
    double tb = dadd(dmul(2.0, e_b), dmul(2.0, sw));
    if (integral) {
        atomicAdd(A.w_int + a, -ta);
        atomicAdd(A.w_int + b, tb);
        atomicAdd(A.a_tot + a, -ki);
        atomicAdd(A.a_tot + b, ki);
    } else {
        A.ta[x] = ta;
        A.tb[x] = tb;
    }
    atomicSub(A.sizes + a, 1);
    atomicAdd(A.sizes + b, 1);
}

// Event deltas in sorted order: leaving a (-(2 e_a + 2 sw), -k_i), joining b
// (+(2 e_b + 2 sw), +k_i).  x - y and x + (-y) round identically, so folding
// the signed deltas reproduces `w_int[a] -= ...; a_tot[a] -= ki` exactly.
__device__ __forceinline__ void event_delta(const StageArgs &A, int32_t v, double &dw,
                                            double &da) {
    int64_t x = v >> 1;
    double ki = A.k[A.subset[x]];
    if (v & 1) {
        dw = A.tb[x];
        da = ki;
    } else {
        dw = -A.ta[x];
        da = -ki;
    }
}

// One warp applies a tiny independent stage (<= 32 VPL vertices, 64 VPL
// events): lane l owns vertices l, l + 32, ... and their leave / join events;
// the (community, event) keys are ordered by a bitonic network in shared
// memory (sk, sw, sa: 64 VPL entries each), then the first lane of every
// community run folds its deltas in event order -- the reference's
// sequential apply (PL/_kernels.pyx:116-144) restated exactly.  State loads
// are coherent (k_tail runs it between stages of one launch).
template <int VPL>
__device__ __forceinline__ void apply_tiny_warp(const StageArgs &A, unsigned long long *sk,
                                                double *sw, double *sa) {
    constexpr int NE = 64 * VPL;
    const int lane = threadIdx.x & 31;
    const int64_t ns = A.ns;
    const unsigned long long S = (unsigned long long)SENTINEL << 32;
    unsigned nmv = 0;
#pragma unroll
    for (int v = 0; v < VPL; v++) {
        const int x = lane + 32 * v;
        bool mv = false;
        int32_t a = 0, b = 0;
        if (x < ns) {
            const int32_t i = ld_state(A.subset + x);
            b = ld_state(A.target + x);
            a = ld_state(A.assign + i);
            mv = ld_state(A.moved + x) && a != b;
            if (mv) {
                const double s2 = dmul(2.0, A.selfw[i]);
                const double ki = A.k[i];
                sw[2 * x] = -dadd(dmul(2.0, ld_state(A.e_old + x)), s2);  // leave a
                sa[2 * x] = -ki;
                sw[2 * x + 1] = dadd(dmul(2.0, ld_state(A.e_best + x)), s2);  // join b
                sa[2 * x + 1] = ki;
                atomicSub(A.sizes + a, 1);
                atomicAdd(A.sizes + b, 1);
                nmv++;
            }
        }
        sk[2 * x] = mv ? ((unsigned long long)(uint32_t)a << 32) | (uint64_t)(2 * x) : S | (2 * x);
        sk[2 * x + 1] =
            mv ? ((unsigned long long)(uint32_t)b << 32) | (uint64_t)(2 * x + 1) : S | (2 * x + 1);
    }
    __syncwarp();
    // bitonic sort of NE keys, VPL compare-exchanges per lane per step
    for (int k = 2; k <= NE; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
            for (int v = 0; v < VPL; v++) {
                const int pr = lane + 32 * v;
                const int i0 = 2 * j * (pr / j) + (pr % j), i1 = i0 + j;
                const bool up = (i0 & k) == 0;
                const unsigned long long x = sk[i0], y = sk[i1];
                if ((x > y) == up) {
                    sk[i0] = y;
                    sk[i1] = x;
                }
            }
            __syncwarp();
        }
    for (int p = lane; p < NE; p += 32) {
        const uint32_t c = (uint32_t)(sk[p] >> 32);
        if (c == SENTINEL) continue;
        if (p > 0 && (uint32_t)(sk[p - 1] >> 32) == c) continue;
        double W = ld_state(A.w_int + c), At = ld_state(A.a_tot + c);
        for (int q = p; q < NE && (uint32_t)(sk[q] >> 32) == c; q++) {
            const int e = (int)(sk[q] & 0xffffffffull);
            W = dadd(W, sw[e]);
            At = dadd(At, sa[e]);
        }
        A.w_int[c] = W;
        A.a_tot[c] = At;
    }
#pragma unroll
    for (int v = 0; v < VPL; v++) {
        const int x = lane + 32 * v;
        if (x < ns && ld_state(A.moved + x)) A.assign[ld_state(A.subset + x)] = ld_state(A.target + x);
    }
    for (int o = 16; o > 0; o >>= 1) nmv += __shfl_xor_sync(0xffffffffu, nmv, o);
    if (lane == 0 && nmv) atomicAdd(A.moves, (unsigned long long)nmv);
    __syncwarp();
}

}  // namespace plv
