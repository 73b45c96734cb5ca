// post.cu -- post-processing on device.
//
// plv_format_assignment: the assignment file of write_assignment
// (PL/engine.py:318-322): one "vertex community\n" line per vertex, decimal.
// Line lengths -> exclusive scan -> every thread prints its own line; the
// host then writes the buffer with one call.
//
// plv_pair_counts: the contingency counts of compare_partitions
// (PL/evaluation.py:68-86): tp = sum over (s, p) cells of C(cell, 2), and
// the same over the classes of s and of p.  Sorting replaces np.unique +
// np.bincount: runs of equal keys are the cells / classes.
#include "common.cuh"
#include <cub/cub.cuh>

namespace plv {

__device__ __forceinline__ int ndigits(uint64_t v) {
    int d = 1;
    while (v >= 10) {
        v /= 10;
        d++;
    }
    return d;
}

__device__ __forceinline__ int line_len(int64_t i, int64_t c) {
    return ndigits((uint64_t)i) + 1 + (c < 0 ? 1 + ndigits((uint64_t)(-c)) : ndigits((uint64_t)c)) + 1;
}

template <class T>
__global__ void k_line_lengths(const T *assign, int64_t n, int64_t *len) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        len[i] = line_len(i, (int64_t)assign[i]);
}

__device__ __forceinline__ uint8_t *put_uint(uint8_t *o, uint64_t v) {
    const int d = ndigits(v);
    for (int k = d - 1; k >= 0; k--) {
        o[k] = (uint8_t)('0' + v % 10);
        v /= 10;
    }
    return o + d;
}

template <class T>
__global__ void k_print_lines(const T *assign, int64_t n, const int64_t *pos, uint8_t *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint8_t *o = out + pos[i];
        o = put_uint(o, (uint64_t)i);
        *o++ = ' ';
        const int64_t c = (int64_t)assign[i];
        if (c < 0) {
            *o++ = '-';
            o = put_uint(o, (uint64_t)(-c));
        } else {
            o = put_uint(o, (uint64_t)c);
        }
        *o = '\n';
    }
}

template <class T>
static void format_assignment(const T *assign, int64_t n, uint8_t *out, int64_t cap,
                              int64_t *len_h, cudaStream_t s) {
    if (n <= 0) {
        *len_h = 0;
        return;
    }
    Buf<int64_t> len(n + 1, s), pos(n + 1, s);
    k_line_lengths<<<grid_for(n, 256), 256, 0, s>>>(assign, n, len.get());
    PLV_LAUNCH_CHECK();
    PLV_CUDA(cudaMemsetAsync(len.get() + n, 0, sizeof(int64_t), s));
    size_t tb = 0;
    PLV_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, len.get(), pos.get(), n + 1, s));
    Buf<char> tmp(tb, s);
    PLV_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, len.get(), pos.get(), n + 1, s));
    const int64_t total = d2h(pos.get() + n, s);
    *len_h = total;
    if (total > cap) return;  // caller retries with a larger buffer
    k_print_lines<<<grid_for(n, 256), 256, 0, s>>>(assign, n, pos.get(), out);
    PLV_LAUNCH_CHECK();
    PLV_CUDA(cudaStreamSynchronize(s));
}

// Sum over runs of equal keys of C(run, 2) = sum_i (i - start(i)), start(i)
// = the last run head at or before i (an inclusive max-scan of head indices).
__global__ void k_run_heads(const int64_t *a, const int64_t *b, int64_t n, int64_t *hp) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const bool head = i == 0 || a[i] != a[i - 1] || (b && b[i] != b[i - 1]);
        hp[i] = head ? i : 0;
    }
}

__global__ void k_rank_sum(const int64_t *start, int64_t n, unsigned long long *out) {
    unsigned long long acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        acc += (unsigned long long)(i - start[i]);
    typedef cub::BlockReduce<unsigned long long, 256> BR;
    __shared__ typename BR::TempStorage t;
    const unsigned long long tot = BR(t).Sum(acc);
    if (threadIdx.x == 0 && tot) atomicAdd(out, tot);
}

static void run_pairs(const int64_t *a, const int64_t *b, int64_t n, int64_t *hp, int64_t *st,
                      unsigned long long *out, cudaStream_t s) {
    const unsigned g = grid_for(n, 256, 148 * 8);
    k_run_heads<<<g, 256, 0, s>>>(a, b, n, hp);
    PLV_LAUNCH_CHECK();
    size_t tb = 0;
    PLV_CUDA(cub::DeviceScan::InclusiveScan(nullptr, tb, hp, st, cub::Max(), n, s));
    Buf<char> tmp(tb, s);
    PLV_CUDA(cub::DeviceScan::InclusiveScan(tmp.get(), tb, hp, st, cub::Max(), n, s));
    k_rank_sum<<<g, 256, 0, s>>>(st, n, out);
    PLV_LAUNCH_CHECK();
}

static void pair_counts(const int64_t *s_lab, const int64_t *p_lab, int64_t n, int64_t *out_h,
                        cudaStream_t st) {
    Buf<int64_t> sk(n, st), pk(n, st), k1(n, st), v1(n, st), k2(n, st), v2(n, st);
    Buf<unsigned long long> acc(3, st);
    PLV_CUDA(cudaMemsetAsync(acc.get(), 0, 3 * sizeof(unsigned long long), st));
    size_t b1 = 0, b2 = 0;
    PLV_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, b1, s_lab, sk.get(), n, 0, 64, st));
    PLV_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b2, p_lab, k1.get(), s_lab, v1.get(), n, 0,
                                             64, st));
    Buf<char> tmp(b1 > b2 ? b1 : b2, st);
    size_t b = tmp.n;
    // classes of s and of p
    PLV_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(), b, s_lab, sk.get(), n, 0, 64, st));
    b = tmp.n;
    PLV_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(), b, p_lab, pk.get(), n, 0, 64, st));
    // cells: by p, then stably by s -> (s, p) order
    b = tmp.n;
    PLV_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), b, p_lab, k1.get(), s_lab, v1.get(), n, 0,
                                             64, st));
    b = tmp.n;
    PLV_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), b, v1.get(), k2.get(), k1.get(), v2.get(),
                                             n, 0, 64, st));
    // k1 / v1 are free again: head positions and run starts
    run_pairs(k2.get(), v2.get(), n, k1.get(), v1.get(), acc.get(), st);       // cells
    run_pairs(sk.get(), nullptr, n, k1.get(), v1.get(), acc.get() + 1, st);    // classes of s
    run_pairs(pk.get(), nullptr, n, k1.get(), v1.get(), acc.get() + 2, st);    // classes of p
    unsigned long long h[3];
    PLV_CUDA(cudaMemcpyAsync(h, acc.get(), sizeof(h), cudaMemcpyDeviceToHost, st));
    PLV_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i < 3; i++) out_h[i] = (int64_t)h[i];
}

}  // namespace plv

extern "C" int plv_format_assignment(const void *assign, int elem_bytes, int64_t n, uint8_t *out,
                                     int64_t cap, int64_t *len_h, void *stream) {
    PLV_ENTRY
    if (elem_bytes == 4)
        plv::format_assignment((const int32_t *)assign, n, out, cap, len_h, plv::S(stream));
    else if (elem_bytes == 8)
        plv::format_assignment((const int64_t *)assign, n, out, cap, len_h, plv::S(stream));
    else
        PLV_FAIL(PLV_EINVAL, "assignment elements must be 4 or 8 bytes");
    PLV_EXIT
}

extern "C" int plv_pair_counts(const int64_t *s, const int64_t *p, int64_t n, int64_t *out_h,
                               void *stream) {
    PLV_ENTRY
    if (n < 0) PLV_FAIL(PLV_EINVAL, "negative length");
    out_h[0] = out_h[1] = out_h[2] = 0;
    if (n > 1) plv::pair_counts(s, p, n, out_h, plv::S(stream));
    PLV_EXIT
}
