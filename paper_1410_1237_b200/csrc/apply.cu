// apply.cu -- apply_moves (PL/_kernels.pyx:104-145) on device, bit-exactly.
//
// The reference applies the decided moves one by one in subset order against
// the live assignment.  Restated in parallel:
//  1. e_a / e_b of every mover: sequential folds in adjacency order over the
//     neighbours whose *live* community is a / b -- the target of an
//     earlier-moved subset vertex, else the snapshot.  In a colour class no
//     neighbour is in the subset, so decide's e_old / e_best are those folds
//     already (PLV_F_INDEPENDENT).
//  2. events (community, subset position, delta) for a_tot and w_internal,
//     stable radix sort by community, and one thread per community folds its
//     events in subset order starting from the current value -- the same
//     additions in the same order as the sequential loop.  Integral graphs
//     (PLV_F_INTEGRAL) add with atomics: every partial sum is an exact integer.
//  3. sizes with integer atomics; the assignment is scattered last.
// Stages of colour classes with <= 2048 vertices run steps 1-3 in one CTA.
#include "localmove.cuh"
#include "lm_device.cuh"
#include "csr.cuh"
#include "pairwise.cuh"
#include <cub/cub.cuh>
#include <cstdlib>

#ifndef AH_TRIGGER
#define AH_TRIGGER 0
#endif

namespace plv {

__global__ void k_fill_i32_a(int32_t *p, int64_t n, int32_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}


// One warp per high-degree mover: live e_a / e_b as ordered folds (the
// matching lanes of each 32-entry chunk are added in lane order).
__device__ __forceinline__ void stage_big_warps(const StageArgs &A, int64_t gw, int64_t nw) {
    const int lane = threadIdx.x & 31;
    const int64_t cnt = (int64_t)*A.nbig;
    const bool integral = A.flags & PLV_F_INTEGRAL;
    for (int64_t q = gw; q < cnt; q += nw) {
        const int64_t x = A.big[q];
        const int32_t i = A.subset[x], b = A.target[x], a = A.assign[i];
        const int64_t e0 = A.off[i], e1 = A.off[i + 1];
        double fa = 0.0, fb = 0.0;
        // four 32-entry chunks per round: their loads (row, then live
        // community) are in flight together; the folds stay in entry order
        constexpr int G = 4;
        for (int64_t g0 = e0; g0 < e1; g0 += 32 * G) {
            int32_t jj[G], cc[G];
            double ww[G];
#pragma unroll
            for (int u = 0; u < G; u++) {
                const int64_t e = g0 + 32 * u + lane;
                jj[u] = e < e1 ? A.nbr[e] : i;
                ww[u] = e < e1 ? A.wts[e] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < G; u++) cc[u] = jj[u] != i ? live_comm(A, jj[u], x) : -1;
#pragma unroll
            for (int u = 0; u < G; u++) {
                const int32_t c = cc[u];
                const double w = ww[u];
                unsigned ma = __ballot_sync(FULL, c == a);
                unsigned mb = __ballot_sync(FULL, c == b && c != a);
                for (unsigned mm = ma; mm; mm &= mm - 1)
                    fa = dadd(fa, __shfl_sync(FULL, w, __ffs(mm) - 1));
                for (unsigned mm = mb; mm; mm &= mm - 1)
                    fb = dadd(fb, __shfl_sync(FULL, w, __ffs(mm) - 1));
            }
        }
        if (lane == 0) mover_deltas(A, x, i, a, b, fa, fb, integral);
    }
}

// One block per huge mover (> APPLY_HUGE entries): the row's entries whose
// live community is a or b are compacted in order (block scan), then thread 0
// folds them -- the chain is only the matching entries, the scan is parallel.
constexpr int64_t APPLY_HUGE = 2048;
// Movers with longer rows fold their live e_a / e_b with a whole warp: a
// thread's fold is a chain of dependent loads per entry (neighbour, position,
// live community), a warp's is one round per 32 entries.
constexpr int64_t APPLY_THREAD_MAX = 8;

__device__ __forceinline__ void stage_huge_block(const StageArgs &A, int64_t b0, int64_t nb) {
    typedef cub::BlockScan<int, 256> Scan;
    __shared__ typename Scan::TempStorage scan;
    __shared__ int8_t sidx[256];
    __shared__ double sw[256];
    const int tid = threadIdx.x;
    const int64_t cnt = (int64_t)*A.nhuge;
    const bool integral = A.flags & PLV_F_INTEGRAL;
    for (int64_t q = b0; q < cnt; q += nb) {
        const int64_t x = A.huge[q];
        const int32_t i = A.subset[x], b = A.target[x], a = A.assign[i];
        const int64_t e0 = A.off[i], e1 = A.off[i + 1];
        // Fast path: if no neighbour that precedes i in the subset has moved,
        // every live community is the snapshot one and decide's exact folds
        // e_old / e_best are e_a / e_b.  Rows are sorted and the subset is
        // ascending, so only the row prefix j < i can hold such neighbours --
        // short for the low-id hubs of R-MAT graphs.
        bool early = false;
        for (int64_t base = e0; base < e1; base += 256) {
            const int64_t e = base + tid;
            bool past = true;
            if (e < e1) {
                const int32_t j = A.nbr[e];
                past = j >= i;
                if (!past) {
                    const int64_t p =
                        (A.flags & PLV_F_IDENTITY) ? (int64_t)j : (int64_t)A.pos[j];
                    early |= p >= 0 && p < x && A.moved[p];
                }
            }
            if (__syncthreads_or(early || past)) break;
        }
        if (!__syncthreads_or(early)) {
            if (tid == 0) mover_deltas(A, x, i, a, b, A.e_old[x], A.e_best[x], integral);
            continue;
        }
        double fa = 0.0, fb = 0.0;  // thread 0's accumulators
        for (int64_t base = e0; base < e1; base += 256) {
            int64_t e = base + tid;
            int k = -1;
            double w = 0.0;
            if (e < e1) {
                int32_t j = A.nbr[e];
                if (j != i) {
                    int32_t c = live_comm(A, j, x);
                    k = c == a ? 0 : (c == b ? 1 : -1);
                    if (k >= 0) w = A.wts[e];
                }
            }
            int pos, total;
            Scan(scan).ExclusiveSum(k >= 0 ? 1 : 0, pos, total);
            if (k >= 0) {
                sidx[pos] = (int8_t)k;
                sw[pos] = w;
            }
            __syncthreads();
            if (tid == 0)
                for (int t = 0; t < total; t++) {
                    if (sidx[t] == 0)
                        fa = dadd(fa, sw[t]);
                    else
                        fb = dadd(fb, sw[t]);
                }
            __syncthreads();
        }
        if (tid == 0) mover_deltas(A, x, i, a, b, fa, fb, integral);
    }
}

// Live e_a / e_b of the movers k_stage_prep deferred: the first APPLY_HB
// blocks take the huge ones (a block each), the others the big ones (a warp
// each) -- one launch for both.
constexpr int APPLY_HB = 148 * 4;
constexpr int APPLY_BB = 148 * 8;

__global__ void __launch_bounds__(256) k_stage_live(StageArgs A) {
    pdl_wait();  // launched programmatically after its predecessor
    if (blockIdx.x < APPLY_HB) {
        stage_huge_block(A, blockIdx.x, APPLY_HB);
    } else {
        const int64_t b = blockIdx.x - APPLY_HB;
        stage_big_warps(A, (b * blockDim.x + threadIdx.x) >> 5,
                        ((int64_t)(gridDim.x - APPLY_HB) * blockDim.x) >> 5);
    }
}

// Per subset index x: events + deltas (+ sizes, moves, and the assignment
// scatter for independent stages).  Low-degree movers fold their live
// e_a / e_b here; high-degree ones go to the k_stage_big worklist.
__global__ void __launch_bounds__(256) k_stage_prep(StageArgs A) {
#if AH_TRIGGER
    if (A.fx.tab) pdl_trigger();  // an ahead stage: the next pass may preload its plan
#endif
    pdl_wait();  // launched programmatically after its predecessor
    // an ahead stage: the blocks from fx.pb on push its movers' weights into
    // the ahead tables of later stages (ahead.cuh)
    if (A.fx.n && blockIdx.x >= A.fx.pb) {
        ahead_fixup(A.fx, blockIdx.x);
        return;
    }
    if (A.lcnt && blockIdx.x == 0 && threadIdx.x == 0) *A.lcnt = 0ull;  // long runs of this stage
    const bool indep = A.flags & PLV_F_INDEPENDENT;
    const bool integral = A.flags & PLV_F_INTEGRAL;
    int lane = threadIdx.x & 31;
    int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)(A.fx.n ? A.fx.pb : gridDim.x) * blockDim.x) >> 5;
    unsigned long long my_moves = 0;
    for (int64_t base = gw * 32; base < A.ns; base += nw * 32) {
        int64_t x = base + lane;
        bool mover = false, big = false;
        int32_t i = 0, a = 0, b = 0;
        const bool live_only = A.live_a != nullptr;
        if (x < A.ns && (!live_only || (x >= A.xlo && x < A.xhi))) {
            i = A.subset[x];
            b = A.target[x];
            a = A.assign[i];
            mover = A.moved[x] && a != b;
            if (!integral && !live_only) {
                A.ekey[2 * x] = mover ? (uint32_t)a : SENTINEL;
                A.ekey[2 * x + 1] = mover ? (uint32_t)b : SENTINEL;
                A.eval[2 * x] = (int32_t)(2 * x);
                A.eval[2 * x + 1] = (int32_t)(2 * x + 1);
                if (mover && A.ccnt) {  // the counting sort's histogram (k_mid_*)
                    atomicAdd(A.ccnt + a, 1);
                    atomicAdd(A.ccnt + b, 1);
                }
            }
        }
        double e_a = 0.0, e_b = 0.0;
        if (mover) {
            if (!live_only) my_moves++;
            if (indep) {
                e_a = A.e_old[x];
                e_b = A.e_best[x];
            } else {
                int64_t e0 = A.off[i], e1 = A.off[i + 1];
                const int deg = (int)(e1 - e0);
                big = deg > APPLY_THREAD_MAX;
                if (!big) {
                    // every load of a level in flight together (row, then
                    // positions, then live communities); the fold stays in order
                    int32_t jj[APPLY_THREAD_MAX], cc[APPLY_THREAD_MAX];
                    double ww[APPLY_THREAD_MAX];
#pragma unroll
                    for (int t = 0; t < APPLY_THREAD_MAX; t++) {
                        jj[t] = t < deg ? A.nbr[e0 + t] : i;
                        ww[t] = t < deg ? A.wts[e0 + t] : 0.0;
                    }
#pragma unroll
                    for (int t = 0; t < APPLY_THREAD_MAX; t++)
                        cc[t] = jj[t] != i ? live_comm(A, jj[t], x) : -1;
#pragma unroll
                    for (int t = 0; t < APPLY_THREAD_MAX; t++) {
                        if (cc[t] < 0) continue;
                        if (cc[t] == a)
                            e_a = dadd(e_a, ww[t]);
                        else if (cc[t] == b)
                            e_b = dadd(e_b, ww[t]);
                    }
                }
            }
        }
        // high-degree movers are folded by a whole warp (k_stage_big), huge
        // ones by a whole block (k_stage_huge)
        if (big) {
            if (A.off[i + 1] - A.off[i] > APPLY_HUGE)
                A.huge[atomicAdd(A.nhuge, 1ull)] = (int32_t)x;
            else
                A.big[atomicAdd(A.nbig, 1ull)] = (int32_t)x;
        }
        if (mover && !big) mover_deltas(A, x, i, a, b, e_a, e_b, integral);
        if (mover && A.dirty) {
            A.dirty[pw_node_of(A.tree_n, A.tree_d0, a)] = 1;
            A.dirty[pw_node_of(A.tree_n, A.tree_d0, b)] = 1;
        }
        if (mover && A.chash)
            atomicXor(A.chash, mix64(((unsigned long long)i << 32) ^ (unsigned int)a ^
                                     0x9E3779B97F4A7C15ull) ^
                                   mix64(((unsigned long long)i << 32) ^ (unsigned int)b ^
                                         0x9E3779B97F4A7C15ull));
        // independent stages: no stage vertex reads another's assignment, so
        // the scatter can happen here
        if (indep && mover) A.assign[i] = b;
    }
    for (int o = 16; o > 0; o >>= 1) my_moves += __shfl_xor_sync(FULL, my_moves, o);
    if (lane == 0 && my_moves) atomicAdd(A.moves, my_moves);
}


// Sequential fold of the run of community c starting at p; the deltas come
// straight from the sorted event ids (loads batched so only the additions
// are serial).
__device__ __forceinline__ void fold_events(const StageArgs &A, const uint32_t *key,
                                            const int32_t *val, int64_t p, int64_t ne, double &W,
                                            double &At) {
    const uint32_t c = key[p];
    while (true) {
        double w[8], a[8];
        bool ok[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            int64_t q = p + u;
            ok[u] = q < ne && key[q] == c;
            w[u] = 0.0;
            a[u] = 0.0;
            if (ok[u]) event_delta(A, val[q], w[u], a[u]);
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
            if (!ok[u]) return;
            W = dadd(W, w[u]);
            At = dadd(At, a[u]);
        }
        p += 8;
    }
}

constexpr int SHORT_EVENTS = 32;  // longer community runs are folded by a whole block

__global__ void k_stage_fold(StageArgs A, const uint32_t *key, const int32_t *val, int64_t ne,
                             int64_t *lrun, unsigned long long *lcnt, double *dW, double *dA) {
    pdl_wait();  // launched programmatically after its predecessor
    const bool indep = A.flags & PLV_F_INDEPENDENT;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < ne;
         p += (int64_t)gridDim.x * blockDim.x) {
        uint32_t c = key[p];
        if (c == SENTINEL) continue;
        {  // every event's delta, in sorted order, for the long-run folds
            double w, a;
            event_delta(A, val[p], w, a);
            dW[p] = w;
            dA[p] = a;
        }
        if (p > 0 && key[p - 1] == c) continue;
        if (p + SHORT_EVENTS < ne && key[p + SHORT_EVENTS] == c) {
            lrun[atomicAdd(lcnt, 1ull)] = p;
            continue;
        }
        double W = A.w_int[c], At = A.a_tot[c];
        fold_events(A, key, val, p, ne, W, At);
        A.w_int[c] = W;
        A.a_tot[c] = At;
    }
    // every live fold has read the assignment by now: scatter the moves
    if (!indep)
        for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < A.ns;
             x += (int64_t)gridDim.x * blockDim.x)
            if (A.moved[x]) A.assign[A.subset[x]] = A.target[x];
    if (blockIdx.x == 0 && threadIdx.x == 0 && A.nbig) A.nbig[0] = A.nbig[1] = 0ull;  // next stage
}

// Long community runs: one block each, block-staged ordered folds.
__global__ void __launch_bounds__(256) k_stage_fold_long(StageArgs A, const uint32_t *key,
                                                        const double *dW, const double *dA,
                                                        int64_t ne, const int64_t *lrun,
                                                        unsigned long long *lcnt) {
    pdl_wait();  // launched programmatically after its predecessor
    __shared__ double sb[4 * FOLD_CH];
    __shared__ int64_t s_end;
    const int64_t cnt = (int64_t)*lcnt;
    for (int64_t w = blockIdx.x; w < cnt; w += gridDim.x) {
        const int64_t p = lrun[w];
        const uint32_t c = key[p];
        if (threadIdx.x == 0) {
            int64_t a = p, b = ne;  // first position past the run
            while (a < b) {
                int64_t mid = (a + b) >> 1;
                if (key[mid] <= c)
                    a = mid + 1;
                else
                    b = mid;
            }
            s_end = a;
        }
        __syncthreads();
        double W = A.w_int[c], At = A.a_tot[c];
        block_fold2(
            [=] __device__(int64_t t, double &x, double &y) {
                x = dW[p + t];
                y = dA[p + t];
            },
            s_end - p, W, At, sb);
        if (threadIdx.x == 0) {
            A.w_int[c] = W;
            A.a_tot[c] = At;
        }
        __syncthreads();
    }
}

// A stage of a small graph (at most MID_N communities): the events' stable
// sort by community as a counting sort over the communities -- histogram
// (k_stage_prep counts its movers' events), one-block scan, scatter of the
// event ids (any order), then each community's segment put in ascending event
// id (the stable order of PL/_kernels.pyx:116-144) and folded with the
// operations of k_stage_fold -- three short launches instead of the device
// radix sort's four plus the two fold launches.  The capped 10,000-iteration phases of small coarse graphs
// pay these per iteration.  ccnt[] is zero between stages (the fold clears it).
constexpr int64_t MID_N = 32768;
#ifndef MID_LOCAL_N
#define MID_LOCAL_N 16
#endif
constexpr int MID_LOCAL = MID_LOCAL_N;  // longer segments are ranked by the whole block

// One block; the counts staged through shared memory so every global access
// is coalesced (dynamic smem: n ints).
__global__ void __launch_bounds__(1024) k_mid_scan(const int32_t *ccnt, int32_t *cur, int64_t n) {
    pdl_wait();
    typedef cub::BlockScan<int, 1024> Scan;
    __shared__ typename Scan::TempStorage tmp;
    extern __shared__ int32_t sc[];
    for (int64_t c = threadIdx.x; c < n; c += 1024) sc[c] = ccnt[c];
    __syncthreads();
    const int64_t per = (n + 1023) / 1024;
    const int64_t c0 = threadIdx.x * per, c1 = c0 + per < n ? c0 + per : n;
    int sum = 0;
    for (int64_t c = c0; c < c1; c++) sum += sc[c];
    int base;
    Scan(tmp).ExclusiveSum(sum, base);
    for (int64_t c = c0; c < c1; c++) {
        const int v = sc[c];
        sc[c] = base;
        base += v;
    }
    __syncthreads();
    for (int64_t c = threadIdx.x; c < n; c += 1024) cur[c] = sc[c];
}

__global__ void k_mid_scatter(StageArgs A, int32_t *cur, int32_t *ids) {
    pdl_wait();
    const int64_t ne = 2 * A.ns;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < ne;
         p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t c = A.ekey[p];
        if (c != SENTINEL) ids[atomicAdd(cur + c, 1)] = (int32_t)p;  // (eval[p] == p)
    }
}

// Thread c: community c's segment [cur[c] - ccnt[c], cur[c]).
constexpr int MID_RANK2 = 128;                    // segments ranked by counting
constexpr int MID_WORDS = (int)(2 * MID_N / 32);  // bitmap words of the event ids
constexpr size_t MID_FOLD_SMEM = sizeof(double) * 4 * FOLD_CH + 2 * sizeof(uint32_t) * MID_WORDS;
__global__ void __launch_bounds__(256) k_mid_fold(StageArgs A, int32_t *ccnt, const int32_t *cur,
                                                  const int32_t *ids, int32_t *tmp, int64_t n,
                                                  double *dW, double *dA) {
    pdl_wait();
    __shared__ int s_nlong;
    __shared__ int32_t s_long[256];
    const int tid = threadIdx.x;
    if (tid == 0) s_nlong = 0;
    __syncthreads();
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + tid;
    const int L = c < n ? ccnt[c] : 0;
    const int s0 = c < n ? cur[c] - L : 0;
    if (L > MID_LOCAL) {
        s_long[atomicAdd(&s_nlong, 1)] = (int32_t)c;
    } else if (L > 0) {
        int32_t e[MID_LOCAL];
#pragma unroll
        for (int t = 0; t < MID_LOCAL; t++) e[t] = t < L ? ids[s0 + t] : INT32_MAX;
        // insertion sort (ascending event id); most segments hold 1-4 events
        if (L > 1 && L <= 4) {
#pragma unroll
            for (int t = 1; t < 4; t++) {
#pragma unroll
                for (int u = 3; u > 0; u--)
                    if (u <= t && e[u] < e[u - 1]) {
                        const int32_t x = e[u];
                        e[u] = e[u - 1];
                        e[u - 1] = x;
                    }
            }
        } else if (L > 4) {
#pragma unroll
            for (int t = 1; t < MID_LOCAL; t++) {
#pragma unroll
                for (int u = MID_LOCAL - 1; u > 0; u--)
                    if (u <= t && e[u] < e[u - 1]) {
                        const int32_t x = e[u];
                        e[u] = e[u - 1];
                        e[u - 1] = x;
                    }
            }
        }
        // the deltas' loads first, the ordered additions after
        double dw[MID_LOCAL], da[MID_LOCAL];
#pragma unroll
        for (int t = 0; t < MID_LOCAL; t++) {
            dw[t] = 0.0;
            da[t] = 0.0;
            if (t < L) event_delta(A, e[t], dw[t], da[t]);
        }
        double W = A.w_int[c], At = A.a_tot[c];
#pragma unroll
        for (int t = 0; t < MID_LOCAL; t++) {
            if (t >= L) break;
            W = dadd(W, dw[t]);
            At = dadd(At, da[t]);
        }
        A.w_int[c] = W;
        A.a_tot[c] = At;
    }
    if (c < n && L) ccnt[c] = 0;  // back to idle
    __syncthreads();
    // long segments of this block's communities, one at a time by the whole
    // block: every event's rank among the segment's ids -- by counting up to
    // MID_RANK2 events, beyond that from a bitmap of the ids and the prefix
    // popcounts of its words (ids are unique and below 2 ns <= 65536) -- then
    // the deltas in ranked order in parallel and the ordered fold staged
    // through shared memory (block_fold2), as k_stage_fold_long does
    extern __shared__ double dyn[];
    double *sb = dyn;                                  // 4 * FOLD_CH doubles
    uint32_t *bm = (uint32_t *)(dyn + 4 * FOLD_CH);    // MID_WORDS words
    int *pre = (int *)(bm + MID_WORDS);                // MID_WORDS prefix popcounts
    typedef cub::BlockScan<int, 256> Scan;
    __shared__ typename Scan::TempStorage scan_tmp;
    const int nlong = s_nlong;
    const int nwords = (int)((2 * A.ns + 31) >> 5);
    for (int w = 0; w < nlong; w++) {
        const int64_t cl = s_long[w];
        const int Ll = cur[cl] - (cl ? cur[cl - 1] : 0);  // (cur[] holds the segment ends)
        const int sl = cur[cl] - Ll;
        if (Ll <= MID_RANK2) {
            for (int t = tid; t < Ll; t += blockDim.x) {
                const int32_t v = ids[sl + t];
                int r = 0;
                for (int u = 0; u < Ll; u++) r += ids[sl + u] < v;
                tmp[sl + r] = v;
            }
        } else {
            for (int q = tid; q < nwords; q += blockDim.x) bm[q] = 0u;
            __syncthreads();
            for (int t = tid; t < Ll; t += blockDim.x) {
                const int32_t v = ids[sl + t];
                atomicOr(&bm[v >> 5], 1u << (v & 31));
            }
            __syncthreads();
            const int per = (nwords + 255) / 256;
            const int q0 = tid * per, q1 = q0 + per < nwords ? q0 + per : nwords;
            int sum = 0;
            for (int q = q0; q < q1; q++) sum += __popc(bm[q]);
            int base;
            Scan(scan_tmp).ExclusiveSum(sum, base);
            for (int q = q0; q < q1; q++) {
                pre[q] = base;
                base += __popc(bm[q]);
            }
            __syncthreads();
            for (int t = tid; t < Ll; t += blockDim.x) {
                const int32_t v = ids[sl + t];
                tmp[sl + pre[v >> 5] + __popc(bm[v >> 5] & ((1u << (v & 31)) - 1u))] = v;
            }
        }
        __syncthreads();
        for (int t = tid; t < Ll; t += blockDim.x) event_delta(A, tmp[sl + t], dW[sl + t], dA[sl + t]);
        __syncthreads();
        double W = A.w_int[cl], At = A.a_tot[cl];
        block_fold2(
            [=] __device__(int64_t t, double &x, double &y) {
                x = dW[sl + t];
                y = dA[sl + t];
            },
            Ll, W, At, sb);
        if (tid == 0) {
            A.w_int[cl] = W;
            A.a_tot[cl] = At;
        }
        __syncthreads();
    }
    // every live fold has read the assignment by now: scatter the moves
    if (!(A.flags & PLV_F_INDEPENDENT))
        for (int64_t x = blockIdx.x * (int64_t)blockDim.x + tid; x < A.ns;
             x += (int64_t)gridDim.x * blockDim.x)
            if (A.moved[x]) A.assign[A.subset[x]] = A.target[x];
    if (blockIdx.x == 0 && tid == 0 && A.nbig) A.nbig[0] = A.nbig[1] = 0ull;  // next stage
}

__global__ void k_stage_scatter(StageArgs A) {
    pdl_wait();  // launched programmatically after its predecessor
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < A.ns;
         x += (int64_t)gridDim.x * blockDim.x)
        if (A.moved[x]) A.assign[A.subset[x]] = A.target[x];
    if (blockIdx.x == 0 && threadIdx.x == 0 && A.nbig) A.nbig[0] = A.nbig[1] = 0ull;  // next stage
}

// One CTA applies a small independent stage: event keys in registers, block
// radix sort, deltas staged in shared memory, ordered per-community folds and
// the scatter, in one launch.  Dynamic smem: 2 * SA_THREADS * SA_ITEMS doubles.
// (SA_ITEMS, the events per thread, shadows the namespace constant.)
template <int SA_ITEMS>
__global__ void __launch_bounds__(SA_THREADS) k_stage_apply_small(StageArgs A, int nb) {

    pdl_wait();  // the decide outputs
    static_assert(SA_ITEMS % 2 == 0, "two events (leave, join) per vertex per thread");
    typedef cub::BlockRadixSort<uint32_t, SA_THREADS, SA_ITEMS, int32_t> Sort;
    __shared__ union {
        typename Sort::TempStorage sort;
        struct {
            uint32_t key[SA_THREADS * SA_ITEMS];
            int32_t val[SA_THREADS * SA_ITEMS];
        } s;
    } sm;
    extern __shared__ double sdel[];  // dW then dA
    __shared__ unsigned long long s_moves;
    const int tid = threadIdx.x;
    const int64_t ne = 2 * A.ns;
    if (tid == 0) s_moves = 0;
    __syncthreads();
    uint32_t keys[SA_ITEMS];
    int32_t vals[SA_ITEMS];
    unsigned long long mv = 0;
    // this thread's SA_ITEMS / 2 vertices (events 2x, 2x + 1): every load of a
    // level is issued before any is used (the stores below would otherwise
    // order each vertex's loads after the previous vertex's stores)
    constexpr int VPT = SA_ITEMS / 2;
    const int64_t x0 = (int64_t)tid * VPT;
    int32_t iv[VPT], bv[VPT], av[VPT];
    bool mvr[VPT];
#pragma unroll
    for (int k = 0; k < VPT; k++) {
        const int64_t x = x0 + k;
        const bool ok = x < A.ns;
        iv[k] = ok ? A.subset[x] : 0;
        bv[k] = ok ? A.target[x] : 0;
        mvr[k] = ok && A.moved[x];
    }
#pragma unroll
    for (int k = 0; k < VPT; k++) av[k] = mvr[k] ? A.assign[iv[k]] : 0;
    double sw[VPT], eo[VPT], eb[VPT];
#pragma unroll
    for (int k = 0; k < VPT; k++) {
        mvr[k] = mvr[k] && av[k] != bv[k];
        sw[k] = mvr[k] ? A.selfw[iv[k]] : 0.0;
        eo[k] = mvr[k] ? A.e_old[x0 + k] : 0.0;
        eb[k] = mvr[k] ? A.e_best[x0 + k] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < VPT; k++) {
        const int64_t x = x0 + k;
        keys[2 * k] = mvr[k] ? (uint32_t)av[k] : SENTINEL;
        keys[2 * k + 1] = mvr[k] ? (uint32_t)bv[k] : SENTINEL;
        vals[2 * k] = (int32_t)(2 * x);
        vals[2 * k + 1] = (int32_t)(2 * x + 1);
        if (mvr[k]) {
            A.ta[x] = dadd(dmul(2.0, eo[k]), dmul(2.0, sw[k]));
            A.tb[x] = dadd(dmul(2.0, eb[k]), dmul(2.0, sw[k]));
            atomicSub(A.sizes + av[k], 1);
            atomicAdd(A.sizes + bv[k], 1);
            mv++;
        }
    }
    Sort(sm.sort).Sort(keys, vals, 0, nb);
    __syncthreads();
#pragma unroll
    for (int it = 0; it < SA_ITEMS; it++) {
        sm.s.key[tid * SA_ITEMS + it] = keys[it];
        sm.s.val[tid * SA_ITEMS + it] = vals[it];
    }
    if (mv) atomicAdd(&s_moves, mv);
    __syncthreads();
    double *dW = sdel, *dA = sdel + SA_THREADS * SA_ITEMS;
    {  // event deltas, every level's loads in flight together
        int32_t ev[SA_ITEMS], vx[SA_ITEMS];
#pragma unroll
        for (int it = 0; it < SA_ITEMS; it++) {
            const int64_t p = tid + (int64_t)it * SA_THREADS;
            ev[it] = (p < ne && sm.s.key[p] != SENTINEL) ? sm.s.val[p] : -1;
        }
#pragma unroll
        for (int it = 0; it < SA_ITEMS; it++) vx[it] = ev[it] >= 0 ? A.subset[ev[it] >> 1] : 0;
        double kk[SA_ITEMS], tt[SA_ITEMS];
#pragma unroll
        for (int it = 0; it < SA_ITEMS; it++) {
            kk[it] = ev[it] >= 0 ? A.k[vx[it]] : 0.0;
            tt[it] = ev[it] >= 0 ? ((ev[it] & 1) ? A.tb[ev[it] >> 1] : A.ta[ev[it] >> 1]) : 0.0;
        }
#pragma unroll
        for (int it = 0; it < SA_ITEMS; it++) {
            if (ev[it] < 0) continue;
            const int64_t p = tid + (int64_t)it * SA_THREADS;
            // leaving a: -(2 e_a + 2 sw), -k_i; joining b: +(2 e_b + 2 sw), +k_i (event_delta)
            dW[p] = (ev[it] & 1) ? tt[it] : -tt[it];
            dA[p] = (ev[it] & 1) ? kk[it] : -kk[it];
        }
    }
    __syncthreads();
    for (int64_t p = tid; p < ne; p += SA_THREADS) {
        uint32_t c = sm.s.key[p];
        if (c == SENTINEL) continue;
        if (p > 0 && sm.s.key[p - 1] == c) continue;
        double W = A.w_int[c], At = A.a_tot[c];
        for (int64_t q = p; q < ne && sm.s.key[q] == c; q++) {
            W = dadd(W, dW[q]);
            At = dadd(At, dA[q]);
        }
        A.w_int[c] = W;
        A.a_tot[c] = At;
    }
    __syncthreads();
    for (int64_t x = tid; x < A.ns; x += SA_THREADS)
        if (A.moved[x]) A.assign[A.subset[x]] = A.target[x];
    if (tid == 0 && s_moves) atomicAdd(A.moves, s_moves);
}

// One warp applies a tiny independent stage (<= 32 VPL vertices, 64 VPL
// events): lane l owns vertices l, l + 32, ... and their leave / join events;
// the (community, event) keys are ordered by a bitonic network in shared
// memory, then the first lane of every community run folds its deltas in
// event order.  Same arithmetic and order as k_stage_apply_small, a fraction
// of its barriers.
template <int VPL>
__global__ void __launch_bounds__(32) k_stage_apply_tiny(StageArgs A) {
    pdl_wait();  // the decide outputs
    __shared__ unsigned long long sk[64 * VPL];
    __shared__ double sw[64 * VPL], sa[64 * VPL];
    apply_tiny_warp<VPL>(A, sk, sw, sa);
}

__global__ void k_pos_scatter(const int32_t *subset, int64_t ns, int32_t *pos, int *dup) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < ns;
         x += (int64_t)gridDim.x * blockDim.x) {
        int32_t old = atomicExch(pos + subset[x], (int32_t)x);
        if (old != -1) atomicOr(dup, 1);
    }
}

void ApplyBuffers::alloc(int64_t ta_len, int64_t max_ns, int64_t n, cudaStream_t s) {
    ta = dalloc<double>(ta_len);
    tb = dalloc<double>(ta_len);
    int64_t ne = 2 * (max_ns ? max_ns : 1);
    ekey = dalloc<uint32_t>(ne);
    ekey2 = dalloc<uint32_t>(ne);
    eval = dalloc<int32_t>(ne);
    eval2 = dalloc<int32_t>(ne);
    dW = dalloc<double>(ne);
    dA = dalloc<double>(ne);
    big_cap = max_ns ? max_ns : 1;
    big = dalloc<int32_t>(2 * big_cap);  // big movers, then huge movers
    nbig = dalloc<unsigned long long>(2);
    PLV_CUDA(cudaMemsetAsync(nbig, 0, 2 * sizeof(unsigned long long), s));
    lrun = dalloc<int64_t>(ne);
    lcnt = dalloc<unsigned long long>(1);
    PLV_CUDA(cudaMemsetAsync(lcnt, 0, sizeof(unsigned long long), s));
    nb = bits_for(n + 1);  // SENTINEL's low nb bits exceed every community id
    this->n = n;
    if (n > 0 && n <= MID_N) {  // the counting sort of a small graph's stages
        ccnt = dalloc<int32_t>(n);
        ccur = dalloc<int32_t>(n);
        PLV_CUDA(cudaMemsetAsync(ccnt, 0, sizeof(int32_t) * n, s));
    }
    PLV_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, ekey, ekey2, eval, eval2, ne, 0, nb, s));
    tmp = pool_alloc(bytes);
    static int dev_done = -1;
    int dev;
    PLV_CUDA(cudaGetDevice(&dev));
    if (dev_done != dev) {
        PLV_CUDA(cudaFuncSetAttribute(k_mid_scan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(sizeof(int32_t) * MID_N)));
        PLV_CUDA(cudaFuncSetAttribute(k_mid_fold, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)MID_FOLD_SMEM));
        PLV_CUDA(cudaFuncSetAttribute(k_stage_apply_small<SA_ITEMS>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(2 * SA_THREADS * SA_ITEMS * sizeof(double))));
        dev_done = dev;
    }
}

void ApplyBuffers::release() {
    cudaDeviceSynchronize();  // buffers go back to the pool idle
    void *ps[] = {ta, tb, ekey, ekey2, eval, eval2, tmp, dW, dA, lrun, lcnt, big, nbig, ccnt, ccur};
    ccnt = ccur = nullptr;
    for (void *p : ps)
        pool_free(p);
    big = nullptr;
    nbig = nullptr;
    lrun = nullptr;
    lcnt = nullptr;
    ta = tb = nullptr;
    ekey = ekey2 = nullptr;
    eval = eval2 = nullptr;
    dW = dA = nullptr;
    tmp = nullptr;
}

static bool mid_off() {  // PLV_APPLY_MID=0: the device radix sort for every stage
    const char *e = getenv("PLV_APPLY_MID");
    return e && e[0] == '0';
}

void launch_live(StageArgs S, const ApplyBuffers &B, cudaStream_t st) {
    if (S.ns == 0 || S.xhi <= S.xlo) return;
    S.big = B.big;
    S.nbig = B.nbig;
    S.huge = B.big + B.big_cap;
    S.nhuge = B.nbig + 1;
    S.lcnt = nullptr;
    S.dirty = nullptr;
    S.chash = nullptr;
    launch_pdl(k_stage_prep, grid_for((S.ns + 31) / 32 * 32, 256, 148 * 16), 256, 0, st, S);
    launch_pdl(k_stage_live, APPLY_HB + APPLY_BB, 256, 0, st, S);
    PLV_CUDA(cudaMemsetAsync(B.nbig, 0, 2 * sizeof(unsigned long long), st));
}

void launch_apply(StageArgs S, const ApplyBuffers &B, cudaStream_t st) {
    if (S.ns == 0) return;
    S.ekey = B.ekey;
    S.eval = B.eval;
    bool indep = S.flags & PLV_F_INDEPENDENT;
    bool integral = S.flags & PLV_F_INTEGRAL;
    if (indep && !integral && S.ns <= 32) {  // (a second vertex per lane measured slower)
        launch_pdl(k_stage_apply_tiny<1>, 1, 32, 0, st, S);
        return;
    }
    if (indep && !integral && S.ns <= SMALL_APPLY_MAX) {
        // events per thread sized to the stage (2 events per vertex)
        if (2 * S.ns <= 2 * SA_THREADS)
            launch_pdl(k_stage_apply_small<2>, 1, SA_THREADS, 4 * SA_THREADS * sizeof(double), st, S,
                       B.nb);
        else if (2 * S.ns <= 4 * SA_THREADS)
            launch_pdl(k_stage_apply_small<4>, 1, SA_THREADS, 8 * SA_THREADS * sizeof(double), st, S,
                       B.nb);
        else
            launch_pdl(k_stage_apply_small<SA_ITEMS>, 1, SA_THREADS,
                       2 * SA_THREADS * SA_ITEMS * sizeof(double), st, S, B.nb);
        return;
    }
    S.big = B.big;
    S.nbig = B.nbig;
    S.huge = B.big + B.big_cap;
    S.nhuge = B.nbig + 1;
    S.lcnt = B.lcnt;
    // worklist counters are zero on entry: allocation clears them, and the
    // apply that used them last cleared them after its last reader
    const bool mid = !integral && B.n <= MID_N && B.ccnt && !mid_off();
    if (mid) S.ccnt = B.ccnt;
    unsigned nbp = grid_for((S.ns + 31) / 32 * 32, 256, 148 * 16);
    if (S.fx.n) {  // + one thread per fix entry of an ahead stage
        S.fx.pb = nbp;
        nbp += (unsigned)((S.fx.n + 255) / 256);
    }
    launch_pdl(k_stage_prep, nbp, 256, 0, st, S);
    if (!indep) {
        launch_pdl(k_stage_live, APPLY_HB + APPLY_BB, 256, 0, st, S);
    }
    if (mid) {
        const int64_t ne = 2 * S.ns;
        launch_pdl(k_mid_scan, 1, 1024, sizeof(int32_t) * (size_t)B.n, st, (const int32_t *)B.ccnt,
                   B.ccur, B.n);
        launch_pdl(k_mid_scatter, grid_for(ne, 256), 256, 0, st, S, B.ccur, B.eval2);
        launch_pdl(k_mid_fold, grid_for(B.n > S.ns ? B.n : S.ns, 256), 256, MID_FOLD_SMEM, st, S,
                   B.ccnt, (const int32_t *)B.ccur, (const int32_t *)B.eval2, (int32_t *)B.ekey2,
                   B.n, B.dW, B.dA);
    } else if (!integral) {
        int64_t ne = 2 * S.ns;
        size_t bytes = B.bytes;
        PLV_CUDA(cub::DeviceRadixSort::SortPairs(B.tmp, bytes, B.ekey, B.ekey2, B.eval, B.eval2, ne,
                                                 0, B.nb, st));
        // folds of short community runs + the scatter; long runs next
        launch_pdl(k_stage_fold, grid_for(ne > S.ns ? ne : S.ns, 256), 256, 0, st, S,
                   (const uint32_t *)B.ekey2, (const int32_t *)B.eval2, ne, B.lrun, B.lcnt, B.dW,
                   B.dA);
        launch_pdl(k_stage_fold_long, 148 * 2, 256, 0, st, S, (const uint32_t *)B.ekey2,
                   (const double *)B.dW, (const double *)B.dA, ne, (const int64_t *)B.lrun,
                   B.lcnt);
    } else if (!indep) {
        launch_pdl(k_stage_scatter, grid_for(S.ns, 256), 256, 0, st, S);
    }
}

// One-off apply over `subset` (synchronises; returns the move count).
static int64_t apply_once(const int64_t *off, const int32_t *nbr, const double *wts,
                          const double *k, const double *selfw, int64_t n, const int32_t *subset,
                          int64_t ns, const int32_t *target, const uint8_t *moved,
                          const double *e_old, const double *e_best, int flags, int32_t *assign,
                          double *a_tot, double *w_int, int32_t *sizes, cudaStream_t s) {
    if (ns <= 0) return 0;
    Buf<int32_t> pos;
    bool general = !(flags & (PLV_F_IDENTITY | PLV_F_INDEPENDENT));
    if (general) {
        pos.alloc(n, s);
        k_fill_i32_a<<<grid_for(n, 256), 256, 0, s>>>(pos, n, -1);
        PLV_LAUNCH_CHECK();
        Buf<int> dup(1, s);
        PLV_CUDA(cudaMemsetAsync(dup.get(), 0, sizeof(int), s));
        k_pos_scatter<<<grid_for(ns, 256), 256, 0, s>>>(subset, ns, pos, dup);
        PLV_LAUNCH_CHECK();
        if (d2h(dup.get(), s)) PLV_FAIL(PLV_EDUP, "subset lists a vertex more than once");
    }
    ApplyBuffers B;
    Buf<unsigned long long> moves(1, s);
    PLV_CUDA(cudaMemsetAsync(moves.get(), 0, sizeof(unsigned long long), s));
    int64_t result = 0;
    try {
        B.alloc(ns, ns, n, s);
        StageArgs S{off, nbr, wts, k, selfw, subset, ns, target, moved, e_old, e_best, pos.get(),
                    flags, assign, a_tot, w_int, sizes, B.ta, B.tb, nullptr, nullptr, moves.get()};
        launch_apply(S, B, s);
        result = (int64_t)d2h(moves.get(), s);
    } catch (...) {
        cudaStreamSynchronize(s);
        B.release();
        throw;
    }
    PLV_CUDA(cudaStreamSynchronize(s));
    B.release();
    return result;
}

}  // namespace plv

extern "C" int plv_apply(const int64_t *off, const int32_t *nbr, const double *wts,
                         const double *k, const double *selfw, int64_t n, const int32_t *subset,
                         int64_t ns, const int32_t *target, const uint8_t *moved,
                         const double *e_old, const double *e_best, int flags, int32_t *assign,
                         double *a_tot, double *w_int, int32_t *sizes, int64_t *moves_h,
                         void *stream) {
    PLV_ENTRY
    int64_t mv = plv::apply_once(off, nbr, wts, k, selfw, n, subset, ns, target, moved, e_old,
                                 e_best, flags, assign, a_tot, w_int, sizes, plv::S(stream));
    if (moves_h) *moves_h = mv;
    PLV_EXIT
}
