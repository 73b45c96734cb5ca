// pairwise.cuh -- numpy's float64 pairwise summation, bit-exact on device.
//
// numpy reduces a contiguous float64 array with pairwise_sum: n < 8 is a
// sequential fold from 0.0; n <= 128 uses eight strided accumulators combined
// as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) followed by a sequential tail;
// larger n splits at n2 = n/2 - (n/2 % 8) and adds the two halves.
// ndarray.sum() = 0.0 + pairwise(a) (reference call sites PL/graph.py:80,
// PL/modularity.py:64) and np.add.reduceat over [s, e) = a[s] +
// pairwise(a[s+1:e]) (PL/graph.py:121, PL/engine.py:253).  Verified against
// numpy 2.3.5 by tests/test_oracle_pins.py.
#pragma once
#include "common.cuh"
#include <vector>

namespace plv {

struct Ident {
    __device__ __forceinline__ double operator()(double x) const { return x; }
};

// (x / two_m)^2, the modularity penalty term np.square(a_tot / two_m).
struct SqScaled {
    double two_m;
    __device__ __forceinline__ double operator()(double x) const {
        double t = __ddiv_rn(x, two_m);
        return __dmul_rn(t, t);
    }
};

template <class F>
__device__ double pw_leaf(const double *a, int64_t n, F f) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res = __dadd_rn(res, f(a[i]));
        return res;
    }
    double r0 = f(a[0]), r1 = f(a[1]), r2 = f(a[2]), r3 = f(a[3]);
    double r4 = f(a[4]), r5 = f(a[5]), r6 = f(a[6]), r7 = f(a[7]);
    int64_t i;
    int64_t lim = n - (n % 8);
    for (i = 8; i < lim; i += 8) {
        r0 = __dadd_rn(r0, f(a[i + 0]));
        r1 = __dadd_rn(r1, f(a[i + 1]));
        r2 = __dadd_rn(r2, f(a[i + 2]));
        r3 = __dadd_rn(r3, f(a[i + 3]));
        r4 = __dadd_rn(r4, f(a[i + 4]));
        r5 = __dadd_rn(r5, f(a[i + 5]));
        r6 = __dadd_rn(r6, f(a[i + 6]));
        r7 = __dadd_rn(r7, f(a[i + 7]));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                           __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
    for (; i < n; i++) res = __dadd_rn(res, f(a[i]));
    return res;
}

__host__ __device__ __forceinline__ int64_t pw_split(int64_t n) {
    int64_t n2 = n / 2;
    return n2 - (n2 % 8);
}

// Serial pairwise sum of a[0:n) (one thread), explicit stack (depth <= 64).
template <class F>
__device__ double pw_serial(const double *a, int64_t n, F f) {
    if (n <= 128) return pw_leaf(a, n, f);
    // Post-order walk: stack of pending right halves and partial left sums.
    int64_t st_off[64], st_n[64];
    double st_val[64];
    int st_state[64];  // 0: left pending, 1: right pending
    int sp = 0;
    st_off[0] = 0; st_n[0] = n; st_state[0] = 0;
    double ret = 0.0;
    while (sp >= 0) {
        int64_t off = st_off[sp], len = st_n[sp];
        if (len <= 128) {
            ret = pw_leaf(a + off, len, f);
            sp--;
            // propagate into parent
            while (sp >= 0) {
                if (st_state[sp] == 0) {
                    st_val[sp] = ret;
                    st_state[sp] = 1;
                    int64_t n2 = pw_split(st_n[sp]);
                    // push right child
                    sp++;
                    st_off[sp] = st_off[sp - 1] + n2;
                    st_n[sp] = st_n[sp - 1] - n2;
                    st_state[sp] = 0;
                    break;
                } else {
                    ret = __dadd_rn(st_val[sp], ret);
                    sp--;
                }
            }
        } else {
            int64_t n2 = pw_split(len);
            sp++;
            st_off[sp] = off;
            st_n[sp] = n2;
            st_state[sp] = 0;
        }
    }
    return ret;
}

// Offset/length of the node with path `path` at depth `d` of the tree of n.
__host__ __device__ __forceinline__ void pw_node(int64_t n, int d, uint64_t path,
                                                 int64_t *lo, int64_t *len) {
    int64_t o = 0, s = n;
    for (int b = d - 1; b >= 0; b--) {
        int64_t n2 = pw_split(s);
        if ((path >> b) & 1ull) {
            o += n2;
            s -= n2;
        } else {
            s = n2;
        }
    }
    *lo = o;
    *len = s;
}

// Index of the depth-d node of the tree of n that holds element c.
__host__ __device__ __forceinline__ uint64_t pw_node_of(int64_t n, int d, int64_t c) {
    int64_t o = 0, s = n;
    uint64_t path = 0;
    for (int b = d - 1; b >= 0; b--) {
        const int64_t n2 = pw_split(s);
        if (c - o >= n2) {
            o += n2;
            s -= n2;
            path |= 1ull << b;
        } else {
            s = n2;
        }
    }
    return path;
}

// Smallest depth at which every node of the tree of n has <= `cap` elements
// (cap >= 256 guarantees no leaf sits above that depth, so the top of the
// tree is a perfect binary tree of 2^d nodes).
inline int pw_depth(int64_t n, int64_t cap = 256) {
    // The distinct node sizes per depth form a small set (they stay within a
    // narrow band), so track the whole set.
    std::vector<int64_t> cur{n}, nxt;
    int d = 0;
    while (true) {
        int64_t mx = 0, mn = INT64_MAX;
        for (int64_t v : cur) {
            mx = v > mx ? v : mx;
            mn = v < mn ? v : mn;
        }
        if (mx <= cap) return d;
        if (mn <= 128) throw std::runtime_error("pairwise tree: leaf above split depth");
        nxt.clear();
        for (int64_t v : cur) {
            int64_t a = pw_split(v);
            for (int64_t c : {a, v - a}) {
                bool seen = false;
                for (int64_t x : nxt) seen |= (x == c);
                if (!seen) nxt.push_back(c);
            }
        }
        cur.swap(nxt);
        d++;
    }
}

// The same node values with a warp per node: a node of <= 256 elements is a
// leaf, two leaves, or a leaf plus a split right half (two leaves); each leaf
// goes to an octet of lanes, lane k of the octet owning accumulator r_k
// (elements k, k+8, ... below the multiple of 8), the accumulators combined
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) by xor-shuffles -- numpy's operation
// order -- then the tail added by the octet's first lane.
template <class F>
__device__ __forceinline__ double pw_leaf_octet(const double *a, int64_t n, F f, int k) {
    // n <= 128: lane k's accumulator takes elements k, k+8, ... (< lim); all
    // of its loads are issued before the first addition (independent of the
    // chain), then the additions run in numpy's order
    double r = 0.0;
    const int64_t lim = n >= 8 ? n - (n % 8) : 0;
    double buf[16];
#pragma unroll
    for (int u = 0; u < 16; u++) {
        const int64_t i = k + 8 * u;
        buf[u] = i < lim ? a[i] : 0.0;
    }
    double tail[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
        const int64_t i = lim + u;
        tail[u] = (k == 0 && i < n) ? a[i] : 0.0;
    }
    if (lim) {
        r = f(buf[0]);
#pragma unroll
        for (int u = 1; u < 16; u++)
            if (k + 8 * u < lim) r = __dadd_rn(r, f(buf[u]));
    }
    double t = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
    t = __dadd_rn(t, __shfl_xor_sync(0xffffffffu, t, 2));
    t = __dadd_rn(t, __shfl_xor_sync(0xffffffffu, t, 4));
    if (k == 0) {
        double res = lim ? t : 0.0;
#pragma unroll
        for (int u = 0; u < 8; u++)
            if (lim + u < n) res = __dadd_rn(res, f(tail[u]));
        t = res;
    }
    return t;  // valid in the octet's first lane
}

template <class F>
__device__ __forceinline__ double pw_node_warp(const double *a, int64_t n, int d0, uint64_t t,
                                               F f) {
    const int lane = threadIdx.x & 31, oct = lane >> 3, k = lane & 7;
    int64_t lo, len;
    pw_node(n, d0, t, &lo, &len);
    int64_t off[3] = {0, 0, 0}, ln[3] = {len, 0, 0};
    int nleaf = 1;
    if (len > 128) {
        const int64_t n2 = pw_split(len);
        ln[0] = n2;
        off[1] = n2;
        ln[1] = len - n2;
        nleaf = 2;
        if (ln[1] > 128) {
            const int64_t m2 = pw_split(ln[1]);
            off[2] = off[1] + m2;
            ln[2] = ln[1] - m2;
            ln[1] = m2;
            nleaf = 3;
        }
    }
    const int o = oct < 3 ? oct : 2;
    const int64_t my_len = oct < nleaf ? ln[o] : 0;
    const double v = pw_leaf_octet(a + lo + off[o], my_len, f, k);
    const double vL = __shfl_sync(0xffffffffu, v, 0);
    const double vR = __shfl_sync(0xffffffffu, v, 8);
    const double vRR = __shfl_sync(0xffffffffu, v, 16);
    return nleaf == 1 ? vL : nleaf == 2 ? __dadd_rn(vL, vR) : __dadd_rn(vL, __dadd_rn(vR, vRR));
}

// Host-side launchers (pairwise.cu).
// out_dev[0] = 0.0 + pairwise(f(a[0:n))) ; f = Ident or SqScaled.
void pw_sum_async(const double *a, int64_t n, double *out_dev, cudaStream_t s);
void pw_sum_sq_async(const double *a, int64_t n, double two_m, double *out_dev, cudaStream_t s);
// out[t] = w[st] (+ pairwise(w[st+1:en])) for segments t of the sorted run
// list starts[0..M) (segment t ends at starts[t+1], the last at R).
int64_t pw_scratch_doubles(int64_t n);
int64_t modularity_scratch_doubles(int64_t n);
// Zero the scratch's ticket once after allocating it (it resets itself).
void modularity_scratch_init(double *scratch, cudaStream_t s);
// q = pairwise(w_int)/2m - pairwise((a_tot/2m)^2); scratch: modularity_scratch_doubles(n).
void modularity_async(const double *w_int, const double *a_tot, int64_t n, double m, double *out,
                      double *scratch, cudaStream_t s);
// Incremental variant (same bits): only the depth-d0 nodes flagged in
// `dirty` (cnt bytes, cleared here) are recomputed, the others keep their
// value from the previous call on the same scratch -- unless *full_if_zero
// is 0 (the first iteration of a device loop), then all are.  Returns false
// (nothing launched) when the tree is too large for the one-launch kernel.
bool modularity_inc_supported(int64_t n, int *d0);
void modularity_async_inc(const double *w_int, const double *a_tot, int64_t n, double m,
                          double *out, double *scratch, uint8_t *dirty,
                          const int64_t *full_if_zero, cudaStream_t s);
void reduceat_async(const double *w, const int64_t *starts, int64_t M, int64_t R, double *out,
                    cudaStream_t s);

}  // namespace plv
