// pairwise.cu -- device reductions with numpy's pairwise tree (bit-exact).
//
// Whole-array sum: the tree of n is cut at the first depth d0 where every
// node has <= 256 elements.  Above d0 the tree is a perfect binary tree (no
// node there is a leaf), so after one warp per depth-d0 node has computed its
// subtree (<= 3 leaves, an octet of lanes each), the remaining levels are an
// aligned perfect pairwise reduction: value(level, p) = value(p0) + value(p1).
#include "pairwise.cuh"

namespace plv {

template <class F>
__global__ void k_pw_nodes_warp(const double *__restrict__ a, int64_t n, int d0, double *vals,
                                F f) {
    const int lane = threadIdx.x & 31, oct = lane >> 3, k = lane & 7;
    const uint64_t cnt = 1ull << d0;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t t = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < cnt; t += nw) {
        int64_t lo, len;
        pw_node(n, d0, t, &lo, &len);
        // the node's leaves: [len] or [L, R] or [L, [RL, RR]]
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
        if (lane == 0)
            vals[t] = nleaf == 1 ? vL : nleaf == 2 ? __dadd_rn(vL, vR) : __dadd_rn(vL, __dadd_rn(vR, vRR));
    }
}

// Reduce groups of 2^kb consecutive values (a perfect subtree each) to one
// (ping-pong in shared memory). When `final` the single remaining value is
// written as 0.0 + root.
__global__ void k_pw_tree2(const double *in, int64_t count, int kb, double *out, int final) {
    extern __shared__ double sm[];
    int64_t group = 1ll << kb;
    double *A = sm, *B = sm + group;
    int64_t base = blockIdx.x * group;
    for (int64_t i = threadIdx.x; i < group; i += blockDim.x)
        A[i] = (base + i < count) ? in[base + i] : 0.0;
    __syncthreads();
    for (int64_t width = group; width > 1; width >>= 1) {
        int64_t half = width >> 1;
        for (int64_t i = threadIdx.x; i < half; i += blockDim.x)
            B[i] = __dadd_rn(A[2 * i], A[2 * i + 1]);
        __syncthreads();
        double *t = A; A = B; B = t;
    }
    if (threadIdx.x == 0) out[blockIdx.x] = final ? __dadd_rn(0.0, A[0]) : A[0];
}

__global__ void k_zero1(double *out) { out[0] = 0.0; }

int64_t pw_scratch_doubles(int64_t n) {
    if (n <= 0) return 2;
    int64_t cnt = 1ll << pw_depth(n);
    return cnt + (cnt + 1023) / 1024 + 2;
}

// scratch: nullptr (stream-ordered allocation) or pw_scratch_doubles(n) doubles.
template <class F>
static void pw_launch(const double *a, int64_t n, double *out_dev, cudaStream_t s, F f,
                      double *scratch = nullptr) {
    if (n <= 0) {
        k_zero1<<<1, 1, 0, s>>>(out_dev);
        PLV_LAUNCH_CHECK();
        return;
    }
    int d0 = pw_depth(n);
    int64_t cnt = 1ll << d0;
    Buf<double> own;
    if (!scratch) {
        own.alloc(pw_scratch_doubles(n), s);
        scratch = own.get();
    }
    double *v0 = scratch, *v1 = scratch + cnt;
    k_pw_nodes_warp<<<grid_for(cnt * 32, 256, 148 * 32), 256, 0, s>>>(a, n, d0, v0, f);
    PLV_LAUNCH_CHECK();
    // reduce the perfect top tree, 2^10 values per block per pass
    double *src = v0, *dst = v1;
    int64_t count = cnt;
    int levels = d0;
    while (true) {
        int kb = levels < 10 ? levels : 10;
        int64_t blocks = count >> kb;
        int final = (kb == levels);
        size_t smem = sizeof(double) * 2 * ((size_t)1 << kb);
        k_pw_tree2<<<(unsigned)blocks, 256, smem, s>>>(src, count, kb, final ? out_dev : dst, final);
        PLV_LAUNCH_CHECK();
        if (final) break;
        levels -= kb;
        count = blocks;
        double *t = src; src = dst; dst = t;
    }
}

void pw_sum_async(const double *a, int64_t n, double *out_dev, cudaStream_t s) {
    pw_launch(a, n, out_dev, s, Ident{});
}

void pw_sum_sq_async(const double *a, int64_t n, double two_m, double *out_dev, cudaStream_t s) {
    pw_launch(a, n, out_dev, s, SqScaled{two_m});
}

__global__ void k_mod_finish(const double *sw, const double *sq, double two_m, double *out) {
    out[0] = __dsub_rn(__ddiv_rn(sw[0], two_m), sq[0]);
}

// Modularity in one launch (trees of <= MODF_MAX_NODES depth-d0 nodes): warps
// compute the depth-d0 node values of both arrays, the last block to finish
// (threadfence + ticket) reduces the two perfect top trees in shared memory
// -- the same additions as k_pw_tree2 -- and writes Q.  The ticket resets
// itself, so the scratch needs zeroing once (modularity_scratch_init).
constexpr int64_t MODF_MAX_NODES = 8192;
constexpr int MODF_THREADS = 512;
constexpr unsigned FULLW = 0xffffffffu;

__global__ void __launch_bounds__(MODF_THREADS) k_mod_fused(const double *__restrict__ w_int,
                                                            const double *__restrict__ a_tot,
                                                            int64_t n, int d0, double two_m,
                                                            double *vals, unsigned int *ticket,
                                                            double *out, uint8_t *dirty,
                                                            const int64_t *full_if_zero) {
    pdl_wait();  // the apply's totals
    __shared__ double sA[2 * MODF_MAX_NODES / 32], sB[2 * MODF_MAX_NODES / 32 / 32 + 2];
    __shared__ bool s_last;
    const uint64_t cnt = 1ull << d0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const bool full = !dirty || *full_if_zero == 0;
    for (uint64_t t = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < 2 * cnt;
         t += nw) {
        if (!full && !dirty[t < cnt ? t : t - cnt]) continue;  // value kept from last call
        const double v = t < cnt ? pw_node_warp(w_int, n, d0, t, Ident{})
                                 : pw_node_warp(a_tot, n, d0, t - cnt, SqScaled{two_m});
        if (lane == 0) vals[t] = v;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // The two perfect top trees (cnt leaves each), 32 consecutive values per
    // warp and round: xor-butterflies add (2i, 2i+1), then pairs of those, ...
    // -- the tree's own additions (lane 0 always holds the left operand).
    const double *src = vals;
    double *dst = sA;
    bool global_src = true;
    uint64_t w = cnt;
    while (w > 1) {
        const uint64_t g = w < 32 ? w : 32, gpa = w / g;
        for (uint64_t gi = warp; gi < 2 * gpa; gi += nwarps) {
            const uint64_t h = gi >= gpa ? 1 : 0, k = gi - h * gpa;
            const uint64_t idx = h * w + k * g + lane;
            double v = 0.0;
            if ((uint64_t)lane < g) v = global_src ? __ldcg(src + idx) : src[idx];
            for (uint64_t o = 1; o < g; o <<= 1) v = __dadd_rn(v, __shfl_xor_sync(FULLW, v, (int)o));
            if (lane == 0) dst[h * gpa + k] = v;
        }
        __syncthreads();
        w = gpa;
        src = dst;
        global_src = false;
        dst = dst == sA ? sB : sA;
    }
    if (dirty)
        for (uint64_t t = threadIdx.x; t < cnt; t += blockDim.x) dirty[t] = 0;
    if (threadIdx.x == 0) {
        const double r0 = global_src ? __ldcg(src) : src[0];
        const double r1 = global_src ? __ldcg(src + 1) : src[1];
        const double sw = __dadd_rn(0.0, r0), sq = __dadd_rn(0.0, r1);
        out[0] = __dsub_rn(__ddiv_rn(sw, two_m), sq);
        *ticket = 0u;
    }
}

int64_t modularity_scratch_doubles(int64_t n) { return 2 * pw_scratch_doubles(n) + 4; }

void modularity_scratch_init(double *scratch, cudaStream_t s) {
    PLV_CUDA(cudaMemsetAsync(scratch, 0, sizeof(double), s));
}

void modularity_async(const double *w_int, const double *a_tot, int64_t n, double m, double *out,
                      double *scratch, cudaStream_t s) {
    double two_m = 2.0 * m;
    unsigned int *ticket = (unsigned int *)scratch;
    scratch += 2;
    if (n > 0) {
        const int d0 = pw_depth(n);
        const int64_t cnt = 1ll << d0;
        if (cnt <= MODF_MAX_NODES) {
            launch_pdl(k_mod_fused, grid_for(2 * cnt * 32, MODF_THREADS, 148 * 8), MODF_THREADS, 0,
                       s, w_int, a_tot, n, d0, two_m, scratch, ticket, out, (uint8_t *)nullptr,
                       (const int64_t *)nullptr);
            return;
        }
    }
    int64_t ps = pw_scratch_doubles(n);
    double *tmp = scratch + 2 * ps;
    pw_launch(w_int, n, tmp, s, Ident{}, scratch);
    pw_launch(a_tot, n, tmp + 1, s, SqScaled{two_m}, scratch + ps);
    k_mod_finish<<<1, 1, 0, s>>>(tmp, tmp + 1, two_m, out);
    PLV_LAUNCH_CHECK();
}

bool modularity_inc_supported(int64_t n, int *d0) {
    if (n <= 0) return false;
    *d0 = pw_depth(n);
    return (1ll << *d0) <= MODF_MAX_NODES;
}

void modularity_async_inc(const double *w_int, const double *a_tot, int64_t n, double m,
                          double *out, double *scratch, uint8_t *dirty,
                          const int64_t *full_if_zero, cudaStream_t s) {
    int d0 = 0;
    if (!modularity_inc_supported(n, &d0)) PLV_FAIL(PLV_EINVAL, "incremental modularity: tree too large");
    const int64_t cnt = 1ll << d0;
    launch_pdl(k_mod_fused, grid_for(2 * cnt * 32, MODF_THREADS, 148 * 8), MODF_THREADS, 0, s,
               w_int, a_tot, n, d0, 2.0 * m, scratch + 2, (unsigned int *)scratch, out, dirty,
               full_if_zero);
}

// ---------------------------------------------------------------- reduceat

constexpr int64_t SEG_SERIAL_MAX = 4096;

constexpr int64_t SEG_BLOCK_NODES = 4096;  // mid segments: <= 4096 depth-d0 nodes, one block

__global__ void k_reduceat_short(const double *__restrict__ w, const int64_t *__restrict__ starts,
                                 int64_t M, int64_t R, double *out, int64_t *mid_list,
                                 unsigned long long *mid_cnt, int64_t *long_list,
                                 unsigned long long *long_cnt) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t st = starts[t];
        int64_t en = (t + 1 < M) ? starts[t + 1] : R;
        int64_t len = en - st;
        if (len <= 1) {
            out[t] = w[st];
        } else if (len - 1 <= SEG_SERIAL_MAX) {
            out[t] = __dadd_rn(w[st], pw_serial(w + st + 1, len - 1, Ident{}));
        } else if (len - 1 <= SEG_BLOCK_NODES * 128) {
            mid_list[atomicAdd(mid_cnt, 1ull)] = t;
        } else {
            long_list[atomicAdd(long_cnt, 1ull)] = t;
        }
    }
}

// Depth at which every node of the pairwise tree of n has <= 256 elements,
// with no leaf above it (pw_depth on device: the largest node of a depth is
// the repeated right half, the smallest the repeated left half); -1 if a leaf
// sits above it (the host path decides then).
__device__ __forceinline__ int pw_depth_dev(int64_t n) {
    int64_t mx = n, mn = n;
    int d = 0;
    while (mx > 256) {
        if (mn <= 128) return -1;
        mx = mx - pw_split(mx);
        mn = pw_split(mn);
        d++;
    }
    return d;
}

// One block per mid segment: w[st] + pairwise(w[st+1:en]) -- a warp per
// depth-d0 node (pw_node_warp), then the perfect top tree pair by pair.
__global__ void __launch_bounds__(512) k_reduceat_mid(const double *__restrict__ w,
                                                      const int64_t *__restrict__ starts,
                                                      int64_t M, int64_t R, double *out,
                                                      const int64_t *mid_list,
                                                      const unsigned long long *mid_cnt,
                                                      int64_t *long_list,
                                                      unsigned long long *long_cnt) {
    __shared__ double vals[SEG_BLOCK_NODES];
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t cnt = (int64_t)*mid_cnt;
    for (int64_t q = blockIdx.x; q < cnt; q += gridDim.x) {
        const int64_t t = mid_list[q];
        const int64_t st = starts[t], en = (t + 1 < M) ? starts[t + 1] : R;
        const double *a = w + st + 1;
        const int64_t L = en - st - 1;
        const int d0 = pw_depth_dev(L);
        if (d0 < 0 || ((int64_t)1 << d0) > SEG_BLOCK_NODES) {
            if (threadIdx.x == 0) long_list[atomicAdd(long_cnt, 1ull)] = t;
            continue;
        }
        const int64_t nn = (int64_t)1 << d0;
        for (int64_t j = warp; j < nn; j += nw) {
            const double v = pw_node_warp(a, L, d0, (uint64_t)j, Ident{});
            if ((threadIdx.x & 31) == 0) vals[j] = v;
        }
        __syncthreads();
        for (int64_t h = nn >> 1; h >= 1; h >>= 1) {  // (2i, 2i+1) -> i, level by level
            double v[SEG_BLOCK_NODES / 512];
#pragma unroll
            for (int u = 0; u < SEG_BLOCK_NODES / 512; u++) {
                const int64_t i = threadIdx.x + (int64_t)u * 512;
                v[u] = i < h ? __dadd_rn(vals[2 * i], vals[2 * i + 1]) : 0.0;
            }
            __syncthreads();
#pragma unroll
            for (int u = 0; u < SEG_BLOCK_NODES / 512; u++) {
                const int64_t i = threadIdx.x + (int64_t)u * 512;
                if (i < h) vals[i] = v[u];
            }
            __syncthreads();
        }
        // ndarray.sum's leading 0.0 is the identity for these (positive) weights
        if (threadIdx.x == 0) out[t] = __dadd_rn(w[st], vals[0]);
        __syncthreads();
    }
}

__global__ void k_seg_finish(const double *w, int64_t st, const double *tail, double *out_t) {
    out_t[0] = __dadd_rn(w[st], tail[0]);
}

__global__ void k_seg_bounds(const int64_t *starts, int64_t M, int64_t R, const int64_t *list,
                             const unsigned long long *cnt, int64_t *se) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < (int64_t)*cnt;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = list[q];
        se[2 * q] = starts[t];
        se[2 * q + 1] = (t + 1 < M) ? starts[t + 1] : R;
    }
}

void reduceat_async(const double *w, const int64_t *starts, int64_t M, int64_t R, double *out,
                    cudaStream_t s) {
    if (M <= 0) return;
    Buf<int64_t> mid_list(M, s), long_list(M, s);
    Buf<unsigned long long> cnts(2, s);
    PLV_CUDA(cudaMemsetAsync(cnts.get(), 0, 2 * sizeof(unsigned long long), s));
    k_reduceat_short<<<grid_for(M, 256), 256, 0, s>>>(w, starts, M, R, out, mid_list.get(),
                                                     cnts.get(), long_list.get(), cnts.get() + 1);
    PLV_LAUNCH_CHECK();
    k_reduceat_mid<<<148 * 2, 512, 0, s>>>(w, starts, M, R, out, mid_list.get(), cnts.get(),
                                          long_list.get(), cnts.get() + 1);
    PLV_LAUNCH_CHECK();
    unsigned long long nl = d2h(cnts.get() + 1, s);
    if (!nl) return;
    // the rare segments of more than 2^19 terms: the whole-array pairwise
    // launcher each; their bounds come back in one copy
    Buf<int64_t> se(2 * nl, s);
    k_seg_bounds<<<grid_for(nl, 256), 256, 0, s>>>(starts, M, R, long_list.get(), cnts.get() + 1,
                                                  se.get());
    PLV_LAUNCH_CHECK();
    std::vector<int64_t> lst(nl), seh(2 * nl);
    PLV_CUDA(cudaMemcpyAsync(lst.data(), long_list.get(), sizeof(int64_t) * nl,
                             cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaMemcpyAsync(seh.data(), se.get(), sizeof(int64_t) * 2 * nl,
                             cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    Buf<double> tail(nl, s);
    for (unsigned long long q = 0; q < nl; q++) {
        const int64_t t = lst[q], st = seh[2 * q], en = seh[2 * q + 1];
        pw_sum_async(w + st + 1, en - st - 1, tail.get() + q, s);
        // pw_sum adds a leading 0.0; 0.0 + x == x for every x the weights
        // produce (x > 0), so the tail value is the pairwise sum itself.
        k_seg_finish<<<1, 1, 0, s>>>(w, st, tail.get() + q, out + t);
        PLV_LAUNCH_CHECK();
    }
}

}  // namespace plv

// ------------------------------------------------------------- C ABI

extern "C" int plv_sum(const double *a, int64_t n, double *out, void *stream) {
    PLV_ENTRY
    if (n < 0) PLV_FAIL(PLV_EINVAL, "plv_sum: negative length");
    plv::pw_sum_async(a, n, out, plv::S(stream));
    PLV_EXIT
}

extern "C" int plv_modularity(const double *w_int, const double *a_tot, int64_t n, double m,
                              double *out, void *stream) {
    PLV_ENTRY
    cudaStream_t s = plv::S(stream);
    if (!(m > 0.0)) PLV_FAIL(PLV_EINVAL, "modularity undefined for edgeless graph");
    plv::Buf<double> scratch(plv::modularity_scratch_doubles(n), s);
    plv::modularity_scratch_init(scratch.get(), s);
    plv::modularity_async(w_int, a_tot, n, m, out, scratch.get(), s);
    PLV_EXIT
}
