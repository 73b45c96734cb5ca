// ingest.cu -- edge-list text -> device records (load_graph, PL/graph.py:245-288,
// edge-list branch).
//
// The file's bytes are copied to HBM once and parsed there:
//   1. line starts: a flag per byte (previous byte is '\n'), stable compaction;
//   2. one thread per line: strip, skip blank / '#' lines, split on ASCII
//      blanks, parse `u v [w]`;
//   3. stable compaction of the record lines (file order is the reference's
//      record order, which the duplicate merge depends on);
//   4. the reference's id rule (densify_ids, PL/graph.py:270-288): ids that
//      already form 0..n-1 are kept -- checked with a presence bitmap.
// Only lines the device can parse with exactly Python's result are accepted:
// ASCII digits / signs / '.', 'e' and blanks, ids of at most 18 digits, and
// weights on Clinger's fast path (an integer significand below 2^53 times
// 10^e with |e| <= 22: one correctly rounded multiply or divide, which is
// what float() returns).  Anything else -- other characters, a malformed
// line, a non-positive weight, non-dense ids, an empty file -- reports
// PLV_INGEST_HOST and the caller re-parses the file with the reference's
// host rules (which also raise the reference's errors with line numbers).
#include "common.cuh"
#include <cub/cub.cuh>

namespace plv {

__global__ void k_line_flags(const uint8_t *t, int64_t len, uint8_t *flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
         i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = (i == 0 || t[i - 1] == '\n') ? 1 : 0;
}

__device__ __forceinline__ bool is_blank(uint8_t c) {
    return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f';
}

// [+-]?[0-9]{1,18}
__device__ __forceinline__ bool parse_int(const uint8_t *p, int n, int64_t *out) {
    int i = 0;
    bool neg = false;
    if (i < n && (p[i] == '+' || p[i] == '-')) neg = p[i++] == '-';
    if (i == n || n - i > 18) return false;
    int64_t v = 0;
    for (; i < n; i++) {
        const uint8_t c = p[i];
        if (c < '0' || c > '9') return false;
        v = v * 10 + (c - '0');
    }
    *out = neg ? -v : v;
    return true;
}

// Python float() of a plain decimal, on Clinger's fast path only.
__device__ __forceinline__ bool parse_weight(const uint8_t *p, int n, double *out) {
    const double P10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                            1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
    int i = 0;
    bool neg = false;
    if (i < n && (p[i] == '+' || p[i] == '-')) neg = p[i++] == '-';
    uint64_t m = 0;
    int digits = 0, frac = 0, nd = 0;
    bool dot = false;
    for (; i < n; i++) {
        const uint8_t c = p[i];
        if (c >= '0' && c <= '9') {
            nd++;
            if (m == 0 && c == '0') {
                if (dot) frac++;
                continue;  // leading zeros carry no significant digit
            }
            if (++digits > 19) return false;
            m = m * 10 + (c - '0');
            if (dot) frac++;
        } else if (c == '.' && !dot) {
            dot = true;
        } else {
            break;
        }
    }
    if (nd == 0) return false;
    int e = 0;
    if (i < n) {
        if (p[i] != 'e' && p[i] != 'E') return false;
        i++;
        bool eneg = false;
        if (i < n && (p[i] == '+' || p[i] == '-')) eneg = p[i++] == '-';
        if (i == n || n - i > 4) return false;
        for (; i < n; i++) {
            if (p[i] < '0' || p[i] > '9') return false;
            e = e * 10 + (p[i] - '0');
        }
        if (eneg) e = -e;
    }
    e -= frac;
    if (m >= (1ull << 53)) return false;
    double x = (double)m;  // exact
    if (m != 0) {
        if (e > 22 || e < -22) return false;
        x = e >= 0 ? __dmul_rn(x, P10[e]) : __ddiv_rn(x, P10[-e]);
    }
    *out = neg ? -x : x;
    return true;
}

// kind: 0 skipped (blank / comment), 1 record; *host set on anything else.
__global__ void k_parse_lines(const uint8_t *t, int64_t len, const int64_t *starts,
                              const int *nlines_d, uint8_t *kind, int64_t *u, int64_t *v,
                              double *w, int *host) {
    const int64_t L = *nlines_d;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < L;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = starts[q], b = q + 1 < L ? starts[q + 1] : len;
        int64_t p = a;
        kind[q] = 0;
        while (p < b && is_blank(t[p])) p++;
        if (p == b || t[p] == '#') continue;
        int64_t ts[4], te[4];
        int nt = 0;
        bool ok = true;
        while (p < b) {
            const uint8_t c = t[p];
            if (c == '\r' && p + 1 < len && t[p + 1] != '\n') ok = false;  // lone CR: a line break to Python
            if (is_blank(c)) {
                p++;
                continue;
            }
            if (nt == 3) {
                ok = false;  // a fourth token: malformed
                break;
            }
            ts[nt] = p;
            while (p < b && !is_blank(t[p])) {
                if (t[p] >= 0x80 || t[p] < 0x20) ok = false;  // non-ASCII / control: host rules
                p++;
            }
            te[nt++] = p;
        }
        int64_t uu = 0, vv = 0;
        double ww = 1.0;
        if (ok && nt >= 2) {
            ok = parse_int(t + ts[0], (int)(te[0] - ts[0]), &uu) &&
                 parse_int(t + ts[1], (int)(te[1] - ts[1]), &vv);
            if (ok && nt == 3) ok = parse_weight(t + ts[2], (int)(te[2] - ts[2]), &ww) && ww > 0.0;
        } else {
            ok = false;
        }
        if (!ok || te[nt - 1] - ts[0] > 4096) {
            atomicOr(host, 1);
            continue;
        }
        kind[q] = 1;
        u[q] = uu;
        v[q] = vv;
        w[q] = ww;
    }
}

__global__ void k_id_range(const int64_t *u, const int64_t *v, const int *R_d,
                           unsigned long long *mn, unsigned long long *mx) {
    const int64_t R = *R_d;
    long long lo = INT64_MAX, hi = INT64_MIN;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
         r += (int64_t)gridDim.x * blockDim.x) {
        const long long a = u[r], b = v[r];
        lo = min(lo, min(a, b));
        hi = max(hi, max(a, b));
    }
    typedef cub::BlockReduce<long long, 256> BR;
    __shared__ typename BR::TempStorage tmp;
    const long long blo = BR(tmp).Reduce(lo, cub::Min());
    __syncthreads();
    const long long bhi = BR(tmp).Reduce(hi, cub::Max());
    if (threadIdx.x == 0) {
        atomicMin((long long *)mn, blo);
        atomicMax((long long *)mx, bhi);
    }
}

__global__ void k_presence(const int64_t *u, const int64_t *v, int64_t R, uint32_t *bits) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = u[r], b = v[r];
        atomicOr(bits + (a >> 5), 1u << (a & 31));
        atomicOr(bits + (b >> 5), 1u << (b & 31));
    }
}

__global__ void k_popc(const uint32_t *bits, int64_t nw, unsigned long long *cnt) {
    unsigned long long c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nw;
         i += (int64_t)gridDim.x * blockDim.x)
        c += __popc(bits[i]);
    typedef cub::BlockReduce<unsigned long long, 256> BR;
    __shared__ typename BR::TempStorage tmp;
    const unsigned long long b = BR(tmp).Sum(c);
    if (threadIdx.x == 0 && b) atomicAdd(cnt, b);
}

__global__ void k_to_i32(const int64_t *a, int64_t n, int32_t *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int32_t)a[i];
}

// Returns PLV_OK with records in u32/v32/w (capacity cap) and info_h =
// {records, n}, or PLV_INGEST_HOST when the host parser must take the file.
static int parse_edge_list(const uint8_t *text, int64_t len, int32_t *u32, int32_t *v32,
                           double *wout, int64_t cap, int64_t *info_h, cudaStream_t s) {
    if (len <= 0) return PLV_INGEST_HOST;
    // 1. line starts
    Buf<uint8_t> flag(len, s);
    k_line_flags<<<grid_for(len, 256), 256, 0, s>>>(text, len, flag);
    PLV_LAUNCH_CHECK();
    Buf<int> nl(1, s);
    Buf<int64_t> starts(len, s);
    cub::CountingInputIterator<int64_t> pos(0);
    size_t tb = 0;
    PLV_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, pos, flag.get(), starts.get(), nl.get(), len, s));
    Buf<char> tmp(tb, s);
    PLV_CUDA(cub::DeviceSelect::Flagged(tmp.get(), tb, pos, flag.get(), starts.get(), nl.get(), len, s));
    const int64_t L = d2h(nl.get(), s);
    // 2. lines
    Buf<uint8_t> kind(L, s);
    Buf<int64_t> lu(L, s), lv(L, s);
    Buf<double> lw(L, s);
    Buf<int> host(1, s);
    PLV_CUDA(cudaMemsetAsync(host.get(), 0, sizeof(int), s));
    k_parse_lines<<<grid_for(L, 256), 256, 0, s>>>(text, len, starts, nl, kind, lu, lv, lw, host);
    PLV_LAUNCH_CHECK();
    if (d2h(host.get(), s)) return PLV_INGEST_HOST;
    // 3. record lines in file order
    Buf<int64_t> ru(L, s), rv(L, s);
    Buf<double> rw(L, s);
    Buf<int> nr(1, s);
    size_t t2 = 0;
    PLV_CUDA(cub::DeviceSelect::Flagged(nullptr, t2, lu.get(), kind.get(), ru.get(), nr.get(), L, s));
    Buf<char> tmp2(t2, s);
    PLV_CUDA(cub::DeviceSelect::Flagged(tmp2.get(), t2, lu.get(), kind.get(), ru.get(), nr.get(), L, s));
    PLV_CUDA(cub::DeviceSelect::Flagged(tmp2.get(), t2, lv.get(), kind.get(), rv.get(), nr.get(), L, s));
    PLV_CUDA(cub::DeviceSelect::Flagged(tmp2.get(), t2, lw.get(), kind.get(), rw.get(), nr.get(), L, s));
    const int64_t R = d2h(nr.get(), s);
    if (R == 0) return PLV_INGEST_HOST;  // empty: the host raises the reference's error
    if (R > cap) PLV_FAIL(PLV_EINVAL, "record buffer too small (%lld records)", (long long)R);
    // 4. dense ids?
    Buf<unsigned long long> mm(2, s);
    const unsigned long long init[2] = {(unsigned long long)INT64_MAX,
                                        (unsigned long long)INT64_MIN};
    PLV_CUDA(cudaMemcpyAsync(mm.get(), init, sizeof(init), cudaMemcpyHostToDevice, s));
    k_id_range<<<grid_for(R, 256, 148 * 8), 256, 0, s>>>(ru, rv, nr, mm.get(), mm.get() + 1);
    PLV_LAUNCH_CHECK();
    long long lohi[2];
    PLV_CUDA(cudaMemcpyAsync(lohi, mm.get(), sizeof(lohi), cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    if (lohi[0] != 0 || lohi[1] >= INT32_MAX) return PLV_INGEST_HOST;
    const int64_t n = lohi[1] + 1, nw = (n + 31) / 32;
    Buf<uint32_t> bits(nw, s);
    PLV_CUDA(cudaMemsetAsync(bits.get(), 0, sizeof(uint32_t) * nw, s));
    k_presence<<<grid_for(R, 256), 256, 0, s>>>(ru, rv, R, bits);
    PLV_LAUNCH_CHECK();
    Buf<unsigned long long> cnt(1, s);
    PLV_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(unsigned long long), s));
    k_popc<<<grid_for(nw, 256, 148 * 8), 256, 0, s>>>(bits, nw, cnt);
    PLV_LAUNCH_CHECK();
    if ((int64_t)d2h(cnt.get(), s) != n) return PLV_INGEST_HOST;  // renumbering: host rule
    k_to_i32<<<grid_for(R, 256), 256, 0, s>>>(ru, R, u32);
    PLV_LAUNCH_CHECK();
    k_to_i32<<<grid_for(R, 256), 256, 0, s>>>(rv, R, v32);
    PLV_LAUNCH_CHECK();
    PLV_CUDA(cudaMemcpyAsync(wout, rw.get(), sizeof(double) * R, cudaMemcpyDeviceToDevice, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    info_h[0] = R;
    info_h[1] = n;
    return PLV_OK;
}

}  // namespace plv

extern "C" int plv_parse_edge_list(const uint8_t *text, int64_t len, int32_t *u, int32_t *v,
                                   double *w, int64_t cap, int64_t *info_h, void *stream) {
    PLV_ENTRY
    return plv::parse_edge_list(text, len, u, v, w, cap, info_h, plv::S(stream));
    PLV_EXIT
}
