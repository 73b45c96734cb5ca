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
// cmt: the comment character; a record line has tmin..tmax tokens.
__global__ void k_parse_lines(const uint8_t *t, int64_t len, const int64_t *starts,
                              const int *nlines_d, uint8_t *kind, int64_t *u, int64_t *v,
                              double *w, int *host, uint8_t cmt, int tmin, int tmax) {
    const int64_t L = *nlines_d;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < L;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = starts[q], b = q + 1 < L ? starts[q + 1] : len;
        int64_t p = a;
        kind[q] = 0;
        while (p < b && is_blank(t[p])) p++;
        if (p == b || t[p] == cmt) continue;
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
            if (nt == tmax) {
                ok = false;  // one token too many: malformed
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
        if (ok && nt >= tmin) {
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
    k_parse_lines<<<grid_for(L, 256), 256, 0, s>>>(text, len, starts, nl, kind, lu, lv, lw, host,
                                                    (uint8_t)'#', 2, 3);
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

// ------------------------------------------------------- Matrix Market

// 1-based (i, j) -> 0-based, every index in [0, rows); *bad otherwise.
__global__ void k_mm_ids(const int64_t *ru, const int64_t *rv, int64_t R, int64_t rows,
                         int32_t *u, int32_t *v, int *bad) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = ru[r] - 1, j = rv[r] - 1;
        if (i < 0 || i >= rows || j < 0 || j >= rows) {
            atomicOr(bad, 1);
            continue;
        }
        u[r] = (int32_t)i;
        v[r] = (int32_t)j;
    }
}

// The coordinate lines of a symmetric Matrix Market body (the text after the
// size line; PL/graph.py:412-478): '%' comments, exactly 2 (pattern) or 3
// tokens, 1-based indices.  PLV_INGEST_HOST on anything the host must judge.
static int parse_mm(const uint8_t *text, int64_t len, int64_t rows, int pattern, int32_t *u32,
                    int32_t *v32, double *wout, int64_t cap, int64_t *info_h, cudaStream_t s) {
    info_h[0] = 0;
    if (len <= 0) return PLV_INGEST_HOST;
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
    Buf<uint8_t> kind(L, s);
    Buf<int64_t> lu(L, s), lv(L, s);
    Buf<double> lw(L, s);
    Buf<int> host(1, s);
    PLV_CUDA(cudaMemsetAsync(host.get(), 0, sizeof(int), s));
    const int nt = pattern ? 2 : 3;
    k_parse_lines<<<grid_for(L, 256), 256, 0, s>>>(text, len, starts, nl, kind, lu, lv, lw, host,
                                                    (uint8_t)'%', nt, nt);
    PLV_LAUNCH_CHECK();
    if (d2h(host.get(), s)) return PLV_INGEST_HOST;
    Buf<int64_t> ru(L, s), rv(L, s);
    Buf<int> nr(1, s);
    size_t t2 = 0;
    PLV_CUDA(cub::DeviceSelect::Flagged(nullptr, t2, lu.get(), kind.get(), ru.get(), nr.get(), L, s));
    Buf<char> tmp2(t2, s);
    PLV_CUDA(cub::DeviceSelect::Flagged(tmp2.get(), t2, lu.get(), kind.get(), ru.get(), nr.get(), L, s));
    PLV_CUDA(cub::DeviceSelect::Flagged(tmp2.get(), t2, lv.get(), kind.get(), rv.get(), nr.get(), L, s));
    const int64_t R = d2h(nr.get(), s);
    if (R == 0) return PLV_INGEST_HOST;
    if (R > cap) PLV_FAIL(PLV_EINVAL, "record buffer too small (%lld records)", (long long)R);
    PLV_CUDA(cub::DeviceSelect::Flagged(tmp2.get(), t2, lw.get(), kind.get(), wout, nr.get(), L, s));
    PLV_CUDA(cudaMemsetAsync(host.get(), 0, sizeof(int), s));
    k_mm_ids<<<grid_for(R, 256), 256, 0, s>>>(ru, rv, R, rows, u32, v32, host);
    PLV_LAUNCH_CHECK();
    if (d2h(host.get(), s)) return PLV_INGEST_HOST;
    info_h[0] = R;
    return PLV_OK;
}

// --------------------------------------------------------------- METIS
//
// The adjacency lines after the header (PL/graph.py:326-411): every line that
// is not a '%' comment is the next vertex's list (blank = isolated); tokens
// are 1-based neighbours, or (neighbour, weight) pairs.  The device takes the
// files whose lists are clean -- no duplicate neighbour, every edge listed in
// both directions with bitwise-equal weights, the declared edge count -- and
// emits the upper entries (vertex <= neighbour) in file order, the
// reference's record order; every other file goes to the host rules.

__device__ __forceinline__ bool metis_comment(const uint8_t *t, int64_t a, int64_t b) {
    int64_t p = a;
    while (p < b && is_blank(t[p]) && t[p] != '\n') p++;
    return p < b && t[p] == '%';
}

// per line: 1 if it is an adjacency line (not a comment)
__global__ void k_metis_lines(const uint8_t *t, int64_t len, const int64_t *starts,
                              const int *nl_d, int32_t *adj, int *bad) {
    const int64_t L = *nl_d;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < L;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = starts[q], b = q + 1 < L ? starts[q + 1] : len;
        adj[q] = metis_comment(t, a, b) ? 0 : 1;
        for (int64_t p = a; p < b; p++) {
            const uint8_t c = t[p];
            if (c >= 0x80 || (c < 0x20 && !is_blank(c))) atomicOr(bad, 1);
            if (c == '\r' && p + 1 < len && t[p + 1] != '\n') atomicOr(bad, 1);  // lone CR
        }
    }
}

// token starts: a non-blank byte after a blank one (or at a line start)
__global__ void k_tok_flags(const uint8_t *t, int64_t len, uint8_t *flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
         i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = !is_blank(t[i]) && (i == 0 || is_blank(t[i - 1])) ? 1 : 0;
}

__device__ __forceinline__ int64_t last_le(const int64_t *a, int64_t n, int64_t x) {
    int64_t lo = 0, hi = n;  // largest q with a[q] <= x
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] <= x)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

// token k -> its line, the line's vertex (adjacency rank), its index in the
// line (first token of the line found by a binary search in the token list)
__global__ void k_metis_tokens(const uint8_t *t, int64_t len, const int64_t *starts, int64_t L,
                               const int32_t *vrank, const int32_t *adj, const int64_t *tok,
                               int64_t T, int64_t n, int weighted, int64_t *tline, int32_t *tvert,
                               int64_t *tval, double *twt, int *bad) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < T;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = tok[k];
        const int64_t q = last_le(starts, L, p);
        tline[k] = q;
        if (!adj[q]) {  // a comment line's token
            tvert[k] = -1;
            continue;
        }
        const int32_t vert = vrank[q];
        tvert[k] = vert;
        if (vert >= n) {  // text past the declared vertices
            atomicOr(bad, 1);
            continue;
        }
        int64_t e = p;
        while (e < len && !is_blank(t[e])) e++;
        // index of this token within its line: tokens of the line start at
        // the first token position >= starts[q]
        const int64_t first = [&] {
            int64_t lo = 0, hi = k;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (tok[mid] < starts[q])
                    lo = mid + 1;
                else
                    hi = mid;
            }
            return lo;
        }();
        const bool wtok = weighted && ((k - first) & 1);
        if (wtok) {
            double w;
            if (!parse_weight(t + p, (int)(e - p), &w) || !(w > 0.0) || e - p > 64) atomicOr(bad, 1);
            else twt[k] = w;
        } else {
            int64_t x;
            if (e - p > 18 || !parse_int(t + p, (int)(e - p), &x) || x < 1 || x > n) atomicOr(bad, 1);
            else tval[k] = x - 1;
        }
    }
}

// entries: the neighbour tokens with their weight (the next token when weighted)
__global__ void k_metis_entries(const int64_t *tline, const int32_t *tvert, const int64_t *tval,
                                const double *twt, const int64_t *tok, const int64_t *starts,
                                int64_t T, int weighted, uint8_t *isnbr, int *bad) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < T;
         k += (int64_t)gridDim.x * blockDim.x) {
        isnbr[k] = 0;
        if (tvert[k] < 0) continue;
        const int64_t q = tline[k];
        int64_t lo = 0, hi = k;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (tok[mid] < starts[q])
                lo = mid + 1;
            else
                hi = mid;
        }
        const int64_t idx = k - lo;
        if (!weighted) {
            isnbr[k] = 1;
        } else if (!(idx & 1)) {
            if (k + 1 >= T || tline[k + 1] != q) atomicOr(bad, 1);  // odd token count
            else isnbr[k] = 1;
        }
    }
}

__global__ void k_metis_emit(const int64_t *sel, int64_t E, const int32_t *tvert,
                             const int64_t *tval, const double *twt, int weighted,
                             uint64_t *ukey, uint64_t *lkey, uint8_t *upper, double *ew,
                             int32_t *ea, int32_t *eb) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < E;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = sel[r];
        const int64_t a = tvert[k], b = tval[k];
        const double w = weighted ? twt[k + 1] : 1.0;
        const int64_t lo = a < b ? a : b, hi = a < b ? b : a;
        const uint64_t key = ((uint64_t)lo << 32) | (uint64_t)hi;
        const bool up = a <= b;
        upper[r] = up;
        ukey[r] = up ? key : ~0ull;
        lkey[r] = up ? ~0ull : key;
        ew[r] = w;
        ea[r] = (int32_t)a;
        eb[r] = (int32_t)b;
    }
}

// sorted keys: duplicates (equal neighbours) -> bad; count real keys
__global__ void k_metis_dups(const uint64_t *k, int64_t E, unsigned long long *cnt, int *bad) {
    unsigned long long c = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < E;
         r += (int64_t)gridDim.x * blockDim.x) {
        if (k[r] == ~0ull) continue;
        c++;
        if (r > 0 && k[r - 1] == k[r]) atomicOr(bad, 1);
    }
    if (c) atomicAdd(cnt, c);
}

// the sorted upper non-self keys / weights equal the sorted lower ones
__global__ void k_metis_sym(const uint64_t *uk, const double *uw, const uint64_t *lk,
                            const double *lw, int64_t cnt, int *bad) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < cnt;
         r += (int64_t)gridDim.x * blockDim.x)
        if (uk[r] != lk[r] || uw[r] != lw[r]) atomicOr(bad, 1);
}

__global__ void k_nonself_flags(const uint64_t *k, int64_t E, uint8_t *f) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < E;
         r += (int64_t)gridDim.x * blockDim.x)
        f[r] = k[r] != ~0ull && (uint32_t)(k[r] >> 32) != (uint32_t)k[r];
}

static int parse_metis(const uint8_t *text, int64_t len, int64_t n, int64_t m_declared,
                       int weighted, int32_t *u32, int32_t *v32, double *wout, int64_t cap,
                       int64_t *info_h, cudaStream_t s) {
    info_h[0] = 0;
    if (len <= 0 || n <= 0) return PLV_INGEST_HOST;
    Buf<int> bad(1, s);
    PLV_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
    // lines and their adjacency ranks
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
    Buf<int32_t> adj(L + 1, s), vrank(L + 1, s);
    k_metis_lines<<<grid_for(L, 256), 256, 0, s>>>(text, len, starts, nl, adj, bad);
    PLV_LAUNCH_CHECK();
    PLV_CUDA(cudaMemsetAsync(adj.get() + L, 0, sizeof(int32_t), s));
    size_t ts = 0;
    PLV_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, ts, adj.get(), vrank.get(), L + 1, s));
    Buf<char> tmp3(ts, s);
    PLV_CUDA(cub::DeviceScan::ExclusiveSum(tmp3.get(), ts, adj.get(), vrank.get(), L + 1, s));
    // a missing final newline leaves no empty last line; fewer than n lines -> host
    if (d2h(vrank.get() + L, s) < n) return PLV_INGEST_HOST;
    // tokens
    PLV_CUDA(cudaMemsetAsync(flag.get(), 0, len, s));
    k_tok_flags<<<grid_for(len, 256), 256, 0, s>>>(text, len, flag);
    PLV_LAUNCH_CHECK();
    Buf<int64_t> tok(len, s);
    Buf<int> ntk(1, s);
    PLV_CUDA(cub::DeviceSelect::Flagged(tmp.get(), tb, pos, flag.get(), tok.get(), ntk.get(), len, s));
    const int64_t T = d2h(ntk.get(), s);
    if (T == 0) return PLV_INGEST_HOST;
    Buf<int64_t> tline(T, s), tval(T, s);
    Buf<int32_t> tvert(T, s);
    Buf<double> twt(T, s);
    k_metis_tokens<<<grid_for(T, 256), 256, 0, s>>>(text, len, starts, L, vrank, adj, tok, T, n,
                                                    weighted, tline, tvert, tval, twt, bad);
    PLV_LAUNCH_CHECK();
    Buf<uint8_t> isnbr(T, s);
    k_metis_entries<<<grid_for(T, 256), 256, 0, s>>>(tline, tvert, tval, twt, tok, starts, T,
                                                     weighted, isnbr, bad);
    PLV_LAUNCH_CHECK();
    if (d2h(bad.get(), s)) return PLV_INGEST_HOST;
    Buf<int64_t> sel(T, s);
    Buf<int> ne(1, s);
    size_t t4 = 0;
    PLV_CUDA(cub::DeviceSelect::Flagged(nullptr, t4, pos, isnbr.get(), sel.get(), ne.get(), T, s));
    Buf<char> tmp4(t4, s);
    PLV_CUDA(cub::DeviceSelect::Flagged(tmp4.get(), t4, pos, isnbr.get(), sel.get(), ne.get(), T, s));
    const int64_t E = d2h(ne.get(), s);
    if (E == 0) return PLV_INGEST_HOST;
    Buf<uint64_t> ukey(E, s), lkey(E, s), uks(E, s), lks(E, s);
    Buf<uint8_t> up(E, s);
    Buf<double> ew(E, s), uws(E, s), lws(E, s);
    Buf<int32_t> ea(E, s), eb(E, s);
    k_metis_emit<<<grid_for(E, 256), 256, 0, s>>>(sel, E, tvert, tval, twt, weighted, ukey, lkey,
                                                  up, ew, ea, eb);
    PLV_LAUNCH_CHECK();
    size_t t5 = 0;
    PLV_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t5, ukey.get(), uks.get(), ew.get(), uws.get(), E, 0, 64, s));
    Buf<char> tmp5(t5, s);
    PLV_CUDA(cub::DeviceRadixSort::SortPairs(tmp5.get(), t5, ukey.get(), uks.get(), ew.get(), uws.get(), E, 0, 64, s));
    PLV_CUDA(cub::DeviceRadixSort::SortPairs(tmp5.get(), t5, lkey.get(), lks.get(), ew.get(), lws.get(), E, 0, 64, s));
    Buf<unsigned long long> cnt(2, s);
    PLV_CUDA(cudaMemsetAsync(cnt.get(), 0, 2 * sizeof(unsigned long long), s));
    k_metis_dups<<<grid_for(E, 256), 256, 0, s>>>(uks, E, cnt.get(), bad);
    PLV_LAUNCH_CHECK();
    k_metis_dups<<<grid_for(E, 256), 256, 0, s>>>(lks, E, cnt.get() + 1, bad);
    PLV_LAUNCH_CHECK();
    unsigned long long c[2];
    PLV_CUDA(cudaMemcpyAsync(c, cnt.get(), sizeof(c), cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    if (d2h(bad.get(), s) || (int64_t)c[0] != m_declared) return PLV_INGEST_HOST;
    // symmetry: the upper non-self keys (sorted) are exactly the lower keys
    Buf<uint8_t> nsf(E, s);
    k_nonself_flags<<<grid_for(E, 256), 256, 0, s>>>(uks, E, nsf);
    PLV_LAUNCH_CHECK();
    Buf<uint64_t> unk(E, s);
    Buf<double> unw(E, s);
    Buf<int> nns(1, s);
    size_t t6 = 0;
    PLV_CUDA(cub::DeviceSelect::Flagged(nullptr, t6, uks.get(), nsf.get(), unk.get(), nns.get(), E, s));
    Buf<char> tmp6(t6, s);
    PLV_CUDA(cub::DeviceSelect::Flagged(tmp6.get(), t6, uks.get(), nsf.get(), unk.get(), nns.get(), E, s));
    PLV_CUDA(cub::DeviceSelect::Flagged(tmp6.get(), t6, uws.get(), nsf.get(), unw.get(), nns.get(), E, s));
    const int64_t nsu = d2h(nns.get(), s);
    if (nsu != (int64_t)c[1]) return PLV_INGEST_HOST;
    if (nsu) {
        k_metis_sym<<<grid_for(nsu, 256), 256, 0, s>>>(unk, unw, lks, lws, nsu, bad);
        PLV_LAUNCH_CHECK();
    }
    if (d2h(bad.get(), s)) return PLV_INGEST_HOST;
    // the upper entries in file order
    if ((int64_t)c[0] > cap) PLV_FAIL(PLV_EINVAL, "record buffer too small");
    Buf<int> nu(1, s);
    size_t t7 = 0, t8 = 0;
    PLV_CUDA(cub::DeviceSelect::Flagged(nullptr, t7, ea.get(), up.get(), u32, nu.get(), E, s));
    PLV_CUDA(cub::DeviceSelect::Flagged(nullptr, t8, ew.get(), up.get(), wout, nu.get(), E, s));
    t7 = t7 > t8 ? t7 : t8;
    Buf<char> tmp7(t7, s);
    PLV_CUDA(cub::DeviceSelect::Flagged(tmp7.get(), t7, ea.get(), up.get(), u32, nu.get(), E, s));
    PLV_CUDA(cub::DeviceSelect::Flagged(tmp7.get(), t7, eb.get(), up.get(), v32, nu.get(), E, s));
    PLV_CUDA(cub::DeviceSelect::Flagged(tmp7.get(), t7, ew.get(), up.get(), wout, nu.get(), E, s));
    info_h[0] = (int64_t)c[0];
    return PLV_OK;
}

}  // namespace plv

extern "C" int plv_parse_edge_list(const uint8_t *text, int64_t len, int32_t *u, int32_t *v,
                                   double *w, int64_t cap, int64_t *info_h, void *stream) {
    PLV_ENTRY
    return plv::parse_edge_list(text, len, u, v, w, cap, info_h, plv::S(stream));
    PLV_EXIT
}

extern "C" int plv_parse_mm(const uint8_t *text, int64_t len, int64_t rows, int pattern,
                            int32_t *u, int32_t *v, double *w, int64_t cap, int64_t *info_h,
                            void *stream) {
    PLV_ENTRY
    return plv::parse_mm(text, len, rows, pattern, u, v, w, cap, info_h, plv::S(stream));
    PLV_EXIT
}

extern "C" int plv_parse_metis(const uint8_t *text, int64_t len, int64_t n, int64_t m_declared,
                               int weighted, int32_t *u, int32_t *v, double *w, int64_t cap,
                               int64_t *info_h, void *stream) {
    PLV_ENTRY
    return plv::parse_metis(text, len, n, m_declared, weighted, u, v, w, cap, info_h,
                            plv::S(stream));
    PLV_EXIT
}
