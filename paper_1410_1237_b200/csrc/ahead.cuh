// ahead.cuh -- small colour classes of an integral phase decided from tables
// accumulated AHEAD of their stage (included by decide.cu only).
//
// A coloured iteration (PL/engine.py:140-163) ends in a long tail of colour
// classes that hold a handful of high-degree vertices each: stage k + 1 reads
// the state stage k wrote, so every such stage used to pay its own chain of
// dependent launches -- accumulate e_{i->C} over the rows (gather the
// assignment, atomics), pass over the sums (gains, argmax), apply.  On an
// integral graph (PLV_F_INTEGRAL: every sum exact in any order) the
// accumulation does not have to wait for its stage:
//
//  * a WINDOW is a run of consecutive small stages.  When the window starts,
//    ONE launch accumulates e_{i->C} for every vertex of every stage of the
//    window into per-vertex hash tables, from the assignment of that moment
//    (bandwidth-bound work over the whole GPU instead of one short
//    latency-bound launch per stage);
//  * a vertex j that moves from a to b in a window stage changes e_{i->a} and
//    e_{i->b} of its neighbours i in LATER stages of the window, and nothing
//    else.  The pairs (j, i) are static, so they are listed at plan time;
//    the apply of j's stage pushes w_ij from a's slot to b's slot of i's
//    table (exact integer arithmetic), beside its own state updates;
//  * the stage itself is then one pass over its vertices' tables -- the gains
//    of PL/_kernels.pyx:86-87 on the exact sums, the (gain desc, label asc)
//    argmax and the singleton-pair guard, as in the hub tier -- followed by
//    the apply.  A slot whose sum fell to zero is no neighbour community and
//    is skipped.
//
// The tables are clean (key -1, sum 0) outside their window: every pass
// clears what it read.
#pragma once

namespace plv {

constexpr int AH_NT = 256;             // threads per pass block
#ifndef AH_UU
#define AH_UU 4                        // (8 measured slower: 86 registers, 2 blocks per SM)
#endif
constexpr int AH_U = AH_UU;            // table slots per pass thread
constexpr int AH_SL = AH_NT * AH_U;    // table slots per pass block
constexpr int AH_CH = 1024;            // row entries per accumulate block (256 threads x 4)
#ifndef AH_MAX_NS
#define AH_MAX_NS 2048                 // vertices of an ahead stage
#endif
#ifndef AH_MAX_ENTRIES
#define AH_MAX_ENTRIES (3 << 20)       // row entries of an ahead stage
#endif
constexpr int64_t AH_MAX_SLOTS = (int64_t)1 << 28;  // 4 GB of slots per window
#ifndef AH_CAP8
#define AH_CAP8 14  // table slots: (deg + pushes + 2) * AH_CAP8 / 8
#endif
#ifndef AH_TRIGGER
#define AH_TRIGGER 1  // early programmatic launch of the next kernel of an ahead stage
#endif
#ifndef AH_MINB
#define AH_MINB 4     // pass blocks per SM (64 registers)
#endif

struct AheadDev {
    AheadRec *tab;
    const int64_t *tbase;   // per ahead vertex: first slot (window-relative)
    const uint32_t *tcap;   // slots: (deg + pushes into it + 2) x AH_CAP8 / 8
    const int32_t *vid;
    const int64_t *row;
    const int32_t *deg;
    int32_t *cold;  // community at the window start (= at its stage: it moves only there)
    int32_t *sold;  // slot of c_old, -1 when no neighbour has been there
    int32_t *tick;  // pass tickets
    int2 *amove;    // (c_old, c_new) of the stage's move, (-1, -1) when it stays
    const int64_t *poff;  // first pass partial
    Best *part;
};

struct AheadWin {
    int64_t s0 = 0;                 // first stage
    int64_t nacc = 0, acc_base = 0;  // accumulate blocks
    int64_t slots = 0;
};

struct Ahead {
    AheadDev d{};
    int64_t *acc_blk = nullptr, *pass_blk = nullptr;  // (vertex << 32) | chunk or slice
    int32_t *fx_src = nullptr, *fx_dst = nullptr;
    double *fx_w = nullptr;
    std::vector<int64_t> g0;        // per stage: its first ahead vertex (nst + 1)
    std::vector<int> win_of;        // per stage: window, -1 when not ahead
    std::vector<AheadWin> wins;
    std::vector<int64_t> pb_base, pb_cnt;  // per stage: pass blocks
    std::vector<int64_t> fx_base, fx_cnt;  // per stage: fix entries
    int64_t nvert = 0, nfix = 0, nslots = 0;
    void release() {
        void *ps[] = {d.tab, (void *)d.tbase, (void *)d.tcap, (void *)d.vid, (void *)d.row,
                      (void *)d.deg, d.cold, d.sold, d.tick, d.amove, (void *)d.poff, d.part,
                      acc_blk, pass_blk, fx_src, fx_dst, fx_w};
        for (void *p : ps) pool_free(p);
        d = AheadDev{};
        acc_blk = pass_blk = nullptr;
        fx_src = fx_dst = nullptr;
        fx_w = nullptr;
    }
};

// ------------------------------------------------------------------ kernels

// Window start: every row entry of every ahead vertex of the window into its
// table (a block per 1024-entry chunk of one row).
__global__ void __launch_bounds__(256) k_ah_accum(DecideArgs A, AheadDev D, const int64_t *blk) {
    const int64_t pk = blk[blockIdx.x];
    const int64_t g = pk >> 32, ch = pk & 0xffffffffll;
    const int32_t i = D.vid[g];
    const int64_t row = D.row[g];
    const int deg = D.deg[g];
    const int tid = threadIdx.x, lane = tid & 31;
    constexpr int U = AH_CH / 256;
    int32_t jj[U], cc[U];
    double ww[U];
#pragma unroll
    for (int u = 0; u < U; u++) {  // the static part of the entries (graph, plan)
        const int64_t t = ch * AH_CH + u * 256 + tid;
        jj[u] = t < deg ? ld_row(A.nbr + (row + t)) : i;
        ww[u] = t < deg ? ld_row(A.wts + (row + t)) : 0.0;
    }
    AheadRec *tab = D.tab + D.tbase[g];
    const uint32_t cap = D.tcap[g];
    pdl_wait();  // the previous stage's apply: the assignment
    const int32_t c_old = ld_state(A.assign + i);
    if (ch == 0 && tid == 0) D.cold[g] = c_old;
#pragma unroll
    for (int u = 0; u < U; u++) cc[u] = jj[u] != i ? ld_state(A.assign + jj[u]) : -1;
#pragma unroll
    for (int u = 0; u < U; u++) {
        // one claim per (warp, community); every lane adds its own entry
        const int32_t c = cc[u];
        const unsigned grp = __match_any_sync(FULL, c);
        const int leader = __ffs(grp) - 1;
        uint32_t s = 0;
        if (c >= 0 && lane == leader) {
            bool fresh;
            s = ahead_claim(tab, c, cap, &fresh);
            if (fresh && c == c_old) D.sold[g] = (int32_t)s;
        }
        s = __shfl_sync(FULL, s, leader);
        if (c >= 0) atomicAdd(&tab[s].val, ww[u]);
    }
}

__device__ __forceinline__ AheadRec ldcg_rec(const AheadRec *p) {
    const int4 v = __ldcg(reinterpret_cast<const int4 *>(p));
    AheadRec r;
    r.key = v.x;
    r.pad = 0;
    r.val = __hiloint2double(v.w, v.z);
    return r;
}
__device__ __forceinline__ void clear_rec(AheadRec *p) {
    *reinterpret_cast<int4 *>(p) = make_int4(-1, 0, 0, 0);
}

// Warp argmax under (gain desc, label asc) with three warp reductions instead
// of five rounds of whole-record shuffles: the lane holding the best (any of
// them when equal records tie).  The gain's bits are mapped to an unsigned
// key of the same order (-0.0 first folded into +0.0, which compares equal);
// labels are int32 values.
__device__ __forceinline__ int ah_warp_argmax(const Best &b) {
    const long long bits = __double_as_longlong(b.g + 0.0);
    const unsigned long long key =
        (unsigned long long)bits ^ (bits < 0 ? ~0ull : 0x8000000000000000ull);
    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
    const unsigned mh = __reduce_max_sync(FULL, hi);
    bool c = hi == mh;
    const unsigned ml = __reduce_max_sync(FULL, c ? lo : 0u);
    c = c && lo == ml;
    const unsigned lb = (unsigned)(int32_t)b.l ^ 0x80000000u;
    const unsigned mb = __reduce_min_sync(FULL, c ? lb : 0xffffffffu);
    c = c && lb == mb;
    return __ffs(__ballot_sync(FULL, c)) - 1;
}

__device__ __forceinline__ Best ah_shfl_best(const Best &b, int src) {
    Best r;
    r.g = __shfl_sync(FULL, b.g, src);
    r.l = __shfl_sync(FULL, b.l, src);
    r.c = __shfl_sync(FULL, b.c, src);
    r.e = __shfl_sync(FULL, b.e, src);
    r.n = __shfl_sync(FULL, b.n, src);
    return r;
}

// Block argmax; the result is valid in warp 0 (one block barrier).
__device__ __forceinline__ Best ah_block_best(BestSmem<AH_NT> &S, const Best &b) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == ah_warp_argmax(b)) S.w[wid] = b;
    __syncthreads();
    if (wid != 0) return b;
    const Best c = lane < AH_NT / 32 ? S.w[lane] : Best{-INFINITY, INT32_MAX, -1, 0.0, 0};
    return ah_shfl_best(c, ah_warp_argmax(c));
}

// Pass block (ahead vertex g, table slice y): the gains of the slice's
// communities on the exact sums, the slice's best; the block that completes
// the vertex's last slice decides it (PL/_kernels.pyx:92-98), records its move
// for the apply's pushes and returns the vertex's state to idle.  Every slot
// read is cleared (c_old's by the deciding block, which reads it last).
__global__ void __launch_bounds__(AH_NT, AH_MINB) k_ah_pass(DecideArgs A, AheadDev D,
                                                            const int64_t *blk, int64_t g_first) {
#if AH_TRIGGER
    pdl_trigger();
#endif
    __shared__ BestSmem<AH_NT> S;
    __shared__ int s_last;
    // plv_debug_trace(2): begin, wait over, gains done, block best, ticket, end
    const bool tr_on = g_tr_on == 2 && threadIdx.x == 0;
    Trace tr;
    tr.n = 0;
    if (tr_on) tr.mark();
    const int tid = threadIdx.x;
    const int64_t pk = blk[blockIdx.x];
    const int64_t g = pk >> 32, y = pk & 0xffffffffll;
    const int32_t i = D.vid[g];
    AheadRec *tab = D.tab + D.tbase[g];
    const int64_t cap = (int64_t)D.tcap[g];
    const double ki = A.k[i];
    const int nsl = (int)(D.poff[g + 1] - D.poff[g]);
    pdl_wait();  // the window's accumulation / the previous stage's apply and pushes
    TR_MARK
    const int32_t c_old = __ldcg(D.cold + g);
    const int32_t so = __ldcg(D.sold + g);
    AheadRec r[AH_U];
#pragma unroll
    for (int u = 0; u < AH_U; u++) {
        const int64_t s = y * AH_SL + u * AH_NT + tid;
        r[u] = s < cap ? ldcg_rec(tab + s) : AheadRec{-1, 0, 0.0};
    }
    const double f_old = so >= 0 ? __ldcg(&tab[so].val) : 0.0;
    const double a_old_excl = dsub(ld_state(A.a_tot + c_old), ki);
    double at[AH_U];
    unsigned long long nc = 0;
#pragma unroll
    for (int u = 0; u < AH_U; u++) {  // every gather in flight before any store
        const bool live = r[u].key >= 0 && r[u].val != 0.0;
        nc += live;
        at[u] = live && r[u].key != c_old ? ld_state(A.a_tot + r[u].key) : 0.0;
    }
    Best b{0.0, LBL(A.labels, c_old), c_old, 0.0, 0};
#pragma unroll
    for (int u = 0; u < AH_U; u++) {
        if (r[u].key < 0 || r[u].key == c_old) continue;
        const int64_t s = y * AH_SL + u * AH_NT + tid;
        clear_rec(tab + s);
        if (r[u].val == 0.0) continue;  // its neighbours all left: not a candidate
        const double g1 = gain_of(r[u].val, f_old, A.m, ki, a_old_excl, at[u], A.four_m_sq);
        consider(b, g1, LBL(A.labels, r[u].key), r[u].key, r[u].val, 0);
    }
    if (A.cand) {  // candidate statistic: one atomic per warp
        unsigned long long w = nc;
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(FULL, w, o);
        if ((tid & 31) == 0 && w) atomicAdd(A.cand, w);
    }
    if (tr_on && b.g != -1.0) tr.mark();  // (the gains are computed)
    if (nsl > 1) {
        b = ah_block_best(S, b);
        TR_MARK
        if (tid == 0) {
            D.part[D.poff[g] + y] = b;
            __threadfence();
            s_last = atomicAdd(D.tick + g, 1) == nsl - 1;
            if (s_last) __threadfence();
        }
        __syncthreads();
        TR_MARK
        if (!s_last) {
            TR_END(8)
            return;
        }
        if (tid >= 32) return;
        Best bw{0.0, LBL(A.labels, c_old), c_old, 0.0, 0};
        for (int64_t t = D.poff[g] + tid; t < D.poff[g + 1]; t += 32) {
            const Best o = ldcg_best(D.part + t);
            consider(bw, o.g, o.l, o.c, o.e, o.n);
        }
        b = ah_shfl_best(bw, ah_warp_argmax(bw));
    } else {
        b = ah_block_best(S, b);
    }
    if (tid == 0) {
        const int64_t x = g - g_first;
        bool moved = b.g > 0.0 && b.c != c_old;
        if (moved && ld_state(A.sizes + c_old) == 1 && ld_state(A.sizes + b.c) == 1 &&
            LBL(A.labels, b.c) > LBL(A.labels, c_old))
            moved = false;  // singleton-pair guard
        A.out_target[x] = moved ? b.c : c_old;
        A.out_moved[x] = moved ? 1 : 0;
        A.out_e_old[x] = f_old;
        A.out_e_best[x] = moved ? b.e : f_old;
        D.amove[g] = moved ? make_int2(c_old, b.c) : make_int2(-1, -1);
        if (so >= 0) clear_rec(tab + so);
        D.sold[g] = -1;
        D.tick[g] = 0;
    }
    TR_END(9)
}

// ------------------------------------------------------------------ planning

// Row entries of every stage of at most AH_MAX_NS vertices (a block per stage).
__global__ void k_ah_stage_entries(const int64_t *off, const int32_t *vtx, const int64_t *soff,
                                   int64_t nst, unsigned long long *out) {
    typedef cub::BlockReduce<unsigned long long, 256> BR;
    __shared__ typename BR::TempStorage tmp;
    for (int64_t a = blockIdx.x; a < nst; a += gridDim.x) {
        const int64_t b0 = soff[a], b1 = soff[a + 1];
        unsigned long long v = 0;
        if (b1 - b0 <= AH_MAX_NS)
            for (int64_t p = b0 + threadIdx.x; p < b1; p += 256) {
                const int32_t i = vtx[p];
                v += (unsigned long long)(off[i + 1] - off[i]);
            }
        const unsigned long long tot = BR(tmp).Sum(v);
        if (threadIdx.x == 0) out[a] = tot;
        __syncthreads();
    }
}

__global__ void k_ah_vertices(const int64_t *off, const int32_t *vtx, const int64_t *gpos,
                              int64_t G, int32_t *vid, int64_t *row, int32_t *deg,
                              int32_t *hubidx) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < G;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = vtx[gpos[g]];
        vid[g] = i;
        row[g] = off[i];
        deg[g] = (int32_t)(off[i + 1] - off[i]);
        hubidx[i] = (int32_t)g;
    }
}

__global__ void k_ah_fill_tab(AheadRec *t, int64_t n) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
         s += (int64_t)gridDim.x * blockDim.x)
        clear_rec(t + s);
}

__global__ void k_ah_fill_move(int2 *m, int64_t n) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
         s += (int64_t)gridDim.x * blockDim.x)
        m[s] = make_int2(-1, -1);
}

// The static pairs (j -> i): i an ahead vertex, j a neighbour in an EARLIER
// stage of i's window.  FILL = false counts them per j, true writes them at
// fx_off[j] (any order: the pushes are exact integer updates).
template <bool FILL>
__global__ void __launch_bounds__(256) k_ah_fix(const int32_t *nbr, const double *wts,
                                                const int64_t *blk, const int32_t *vid,
                                                const int64_t *row, const int32_t *deg,
                                                const int32_t *hubidx, const int32_t *gstage,
                                                const int32_t *gwin, unsigned long long *cnt,
                                                unsigned long long *cin,
                                                const unsigned long long *fx_off, int32_t *fx_src,
                                                int32_t *fx_dst, double *fx_w) {
    const int64_t pk = blk[blockIdx.x];
    const int64_t g = pk >> 32, ch = pk & 0xffffffffll;
    const int64_t r0 = row[g];
    const int d = deg[g];
    const int32_t st = gstage[g], wn = gwin[g];
    for (int u = 0; u < AH_CH / 256; u++) {
        const int64_t t = ch * AH_CH + u * 256 + threadIdx.x;
        if (t >= d) break;
        const int32_t j = nbr[r0 + t];
        const int32_t gj = hubidx[j];
        if (gj < 0 || gwin[gj] != wn || gstage[gj] >= st) continue;
        const unsigned long long k = atomicAdd(cnt + gj, 1ull);
        if (!FILL) atomicAdd(cin + g, 1ull);
        if (FILL) {
            const unsigned long long p = fx_off[gj] + k;
            fx_src[p] = gj;
            fx_dst[p] = (int32_t)g;
            fx_w[p] = wts[r0 + t];
        }
    }
}

static bool ahead_env_off() {
    const char *e = getenv("PLV_AHEAD");
    return e && e[0] == '0';
}
static bool ahead_env_lowdeg() {  // tests: low-degree stages qualify too
    const char *e = getenv("PLV_AHEAD_LOWDEG");
    return e && e[0] == '1';
}

// Choose the ahead stages (clearing their tiers), group them into windows and
// build the tables, block lists and fix lists.  h: the (stage, tier) histogram.
static int64_t ahead_env(const char *name, int64_t dflt) {  // experiments
    const char *e = getenv(name);
    const int64_t v = e ? atoll(e) : 0;
    return v > 0 ? v : dflt;
}
static int64_t ahead_env_slots() { return ahead_env("PLV_AHEAD_SLOTS", AH_MAX_SLOTS); }

static void ahead_plan(Plan &P, const int64_t *off, const int32_t *nbr, const double *wts,
                       const int32_t *vtx, const int64_t *soff_h, const int64_t *d_soff,
                       int64_t nst, int64_t n, cudaStream_t s) {
    if (ahead_env_off() || nst < 2 || n >= ((int64_t)1 << 31)) return;
    const int64_t max_win_slots = ahead_env_slots();
    const bool lowdeg = ahead_env_lowdeg();
    Buf<unsigned long long> d_ent(nst, s);
    k_ah_stage_entries<<<grid_for(nst, 1, 148 * 8), 256, 0, s>>>(off, vtx, d_soff, nst, d_ent);
    PLV_LAUNCH_CHECK();
    std::vector<unsigned long long> ent(nst);
    PLV_CUDA(cudaMemcpyAsync(ent.data(), d_ent.get(), sizeof(unsigned long long) * nst,
                             cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    int64_t first = -1;
    for (int64_t a = 0; a < nst && first < 0; a++)
        if (P.st[a].ns) first = a;
    std::vector<char> is_ah(nst, 0);
    int64_t G = 0;
    for (int64_t a = 0; a < nst; a++) {
        const StagePlan &sp = P.st[a];
        if (!sp.ns || a == first || sp.ns > AH_MAX_NS || (int64_t)ent[a] > AH_MAX_ENTRIES) continue;
        if (!lowdeg && (sp.tcount[0] + sp.tcount[1]) * 8 > sp.ns) continue;
        is_ah[a] = 1;
        G += sp.ns;
    }
    if (!G) return;
    Ahead *H = new Ahead();
    P.ah = H;
    H->g0.assign(nst + 1, 0);
    H->win_of.assign(nst, -1);
    H->pb_base.assign(nst, 0);
    H->pb_cnt.assign(nst, 0);
    H->fx_base.assign(nst, 0);
    H->fx_cnt.assign(nst, 0);
    std::vector<int64_t> gpos(G);
    std::vector<int32_t> gstage(G), gwin(G);
    {
        int64_t g = 0;
        for (int64_t a = 0; a < nst; a++) {
            H->g0[a] = g;
            if (is_ah[a])
                for (int64_t x = 0; x < P.st[a].ns; x++) {
                    gpos[g] = soff_h[a] + x;
                    gstage[g] = (int32_t)a;
                    g++;
                }
        }
        H->g0[nst] = g;
    }
    H->nvert = G;
    AheadDev &D = H->d;
    int32_t *vid = dalloc<int32_t>(G);
    int64_t *row = dalloc<int64_t>(G);
    int32_t *deg = dalloc<int32_t>(G);
    D.vid = vid;
    D.row = row;
    D.deg = deg;
    Buf<int64_t> d_gpos(G, s);
    Buf<int32_t> hubidx(n, s);
    PLV_CUDA(cudaMemcpyAsync(d_gpos.get(), gpos.data(), sizeof(int64_t) * G, cudaMemcpyHostToDevice,
                             s));
    PLV_CUDA(cudaMemsetAsync(hubidx.get(), 0xff, sizeof(int32_t) * n, s));
    k_ah_vertices<<<grid_for(G, 256), 256, 0, s>>>(off, vtx, d_gpos, G, vid, row, deg, hubidx);
    PLV_LAUNCH_CHECK();
    std::vector<int32_t> hdeg(G);
    PLV_CUDA(cudaMemcpyAsync(hdeg.data(), deg, sizeof(int32_t) * G, cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    // windows (runs of consecutive ahead stages, cut where a window's tables
    // could exceed the slot budget) and the accumulation blocks
    std::vector<int64_t> acc;
    int64_t cur = -1, wslots = 0;
    for (int64_t a = 0; a < nst; a++) {
        if (!P.st[a].ns) continue;  // an empty stage does not end a window
        if (!is_ah[a]) {
            cur = -1;
            continue;
        }
        int64_t sslots = 0;  // (an upper bound: a table has at most 2.25 deg + 36 slots)
        for (int64_t g = H->g0[a]; g < H->g0[a + 1]; g++) sslots += 3 * (int64_t)hdeg[g] + 64;
        if (cur < 0 || wslots + sslots > max_win_slots) {
            AheadWin w;
            w.s0 = a;
            w.acc_base = (int64_t)acc.size();
            H->wins.push_back(w);
            cur = (int64_t)H->wins.size() - 1;
            wslots = 0;
        }
        wslots += sslots;
        H->win_of[a] = (int)cur;
        for (int64_t g = H->g0[a]; g < H->g0[a + 1]; g++) {
            gwin[g] = (int32_t)cur;
            const int64_t nch = ((int64_t)hdeg[g] + AH_CH - 1) / AH_CH;
            for (int64_t c = 0; c < nch; c++) acc.push_back((g << 32) | c);
        }
        H->wins[cur].nacc = (int64_t)acc.size() - H->wins[cur].acc_base;
    }
    H->acc_blk = dalloc<int64_t>(acc.size());
    if (!acc.empty())
        PLV_CUDA(cudaMemcpyAsync(H->acc_blk, acc.data(), sizeof(int64_t) * acc.size(),
                                 cudaMemcpyHostToDevice, s));
    // fix lists: counts per source (the list offsets) and per destination (the
    // table sizes)
    Buf<int32_t> d_gstage(G, s), d_gwin(G, s);
    Buf<unsigned long long> cnt(G + 1, s), cin(G, s), fx_off(G + 1, s);
    PLV_CUDA(cudaMemcpyAsync(d_gstage.get(), gstage.data(), sizeof(int32_t) * G,
                             cudaMemcpyHostToDevice, s));
    PLV_CUDA(cudaMemcpyAsync(d_gwin.get(), gwin.data(), sizeof(int32_t) * G, cudaMemcpyHostToDevice,
                             s));
    PLV_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(unsigned long long) * (G + 1), s));
    PLV_CUDA(cudaMemsetAsync(cin.get(), 0, sizeof(unsigned long long) * G, s));
    const unsigned na = (unsigned)acc.size();
    if (na) {
        k_ah_fix<false><<<na, 256, 0, s>>>(nbr, wts, H->acc_blk, vid, row, deg, hubidx, d_gstage,
                                           d_gwin, cnt, cin, nullptr, nullptr, nullptr, nullptr);
        PLV_LAUNCH_CHECK();
    }
    size_t tb = 0;
    PLV_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.get(), fx_off.get(), G + 1, s));
    Buf<char> tmp(tb, s);
    PLV_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, cnt.get(), fx_off.get(), G + 1, s));
    std::vector<unsigned long long> foff(G + 1), hin(G);
    PLV_CUDA(cudaMemcpyAsync(foff.data(), fx_off.get(), sizeof(unsigned long long) * (G + 1),
                             cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaMemcpyAsync(hin.data(), cin.get(), sizeof(unsigned long long) * G,
                             cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    // table slices and pass blocks.  A table holds at most one community per
    // row entry plus one per push into it, so deg + pushes + 2 slots can never
    // fill up (the claim loops end); an eighth more keeps the probe runs short.
    // (Power-of-two tables of >= 2 deg + 2 slots measured ~2x the pass and
    // accumulation traffic.)
    std::vector<int64_t> tbase(G), poff(G + 1, 0), pass;
    std::vector<uint32_t> tcap(G);
    const int64_t cap8 = ahead_env("PLV_AHEAD_CAP8", AH_CAP8) < 9 ? 9 : ahead_env("PLV_AHEAD_CAP8", AH_CAP8);
    int64_t max_slots = 0;
    cur = -1;
    wslots = 0;
    for (int64_t a = 0; a < nst; a++) {
        if (!is_ah[a]) continue;
        if (H->win_of[a] != cur) {
            cur = H->win_of[a];
            wslots = 0;
        }
        H->pb_base[a] = (int64_t)pass.size();
        for (int64_t g = H->g0[a]; g < H->g0[a + 1]; g++) {
            const int64_t need = (int64_t)hdeg[g] + (int64_t)hin[g] + 2;
            int64_t cap = need * cap8 / 8;
            cap = (cap + 3) / 4 * 4;
            if (cap < 32) cap = 32;
            tbase[g] = wslots;
            tcap[g] = (uint32_t)cap;
            wslots += cap;
            const int64_t nsl = (cap + AH_SL - 1) / AH_SL;
            for (int64_t y = 0; y < nsl; y++) pass.push_back((g << 32) | y);
            poff[g + 1] = poff[g] + nsl;
        }
        H->pb_cnt[a] = (int64_t)pass.size() - H->pb_base[a];
        H->wins[cur].slots = wslots;
        max_slots = wslots > max_slots ? wslots : max_slots;
    }
    H->nslots = max_slots;
    int64_t *d_tbase = dalloc<int64_t>(G), *d_poff = dalloc<int64_t>(G + 1);
    uint32_t *d_tcap = dalloc<uint32_t>(G);
    D.tbase = d_tbase;
    D.tcap = d_tcap;
    D.poff = d_poff;
    PLV_CUDA(cudaMemcpyAsync(d_tbase, tbase.data(), sizeof(int64_t) * G, cudaMemcpyHostToDevice, s));
    PLV_CUDA(cudaMemcpyAsync(d_tcap, tcap.data(), sizeof(uint32_t) * G, cudaMemcpyHostToDevice, s));
    PLV_CUDA(cudaMemcpyAsync(d_poff, poff.data(), sizeof(int64_t) * (G + 1), cudaMemcpyHostToDevice,
                             s));
    H->pass_blk = dalloc<int64_t>(pass.size());
    PLV_CUDA(cudaMemcpyAsync(H->pass_blk, pass.data(), sizeof(int64_t) * pass.size(),
                             cudaMemcpyHostToDevice, s));
    D.tab = dalloc<AheadRec>(max_slots);
    k_ah_fill_tab<<<grid_for(max_slots, 256), 256, 0, s>>>(D.tab, max_slots);
    PLV_LAUNCH_CHECK();
    D.cold = dalloc<int32_t>(G);
    D.sold = dalloc<int32_t>(G);
    D.tick = dalloc<int32_t>(G);
    D.amove = dalloc<int2>(G);
    D.part = dalloc<Best>(poff[G]);
    PLV_CUDA(cudaMemsetAsync(D.cold, 0xff, sizeof(int32_t) * G, s));
    PLV_CUDA(cudaMemsetAsync(D.sold, 0xff, sizeof(int32_t) * G, s));
    PLV_CUDA(cudaMemsetAsync(D.tick, 0, sizeof(int32_t) * G, s));
    k_ah_fill_move<<<grid_for(G, 256), 256, 0, s>>>(D.amove, G);
    PLV_LAUNCH_CHECK();
    H->nfix = (int64_t)foff[G];
    H->fx_src = dalloc<int32_t>(H->nfix);
    H->fx_dst = dalloc<int32_t>(H->nfix);
    H->fx_w = dalloc<double>(H->nfix);
    if (H->nfix) {
        PLV_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(unsigned long long) * (G + 1), s));
        k_ah_fix<true><<<na, 256, 0, s>>>(nbr, wts, H->acc_blk, vid, row, deg, hubidx, d_gstage,
                                          d_gwin, cnt, nullptr, fx_off, H->fx_src, H->fx_dst,
                                          H->fx_w);
        PLV_LAUNCH_CHECK();
    }
    for (int64_t a = 0; a < nst; a++) {
        H->fx_base[a] = (int64_t)foff[H->g0[a]];
        H->fx_cnt[a] = (int64_t)(foff[H->g0[a + 1]] - foff[H->g0[a]]);
    }
    // the ahead stages leave the tiers
    for (int64_t a = 0; a < nst; a++)
        if (is_ah[a]) P.st[a].ahead = true;
    PLV_CUDA(cudaStreamSynchronize(s));
}

// Stage a's decide from its ahead tables; the window's accumulation first
// when a opens its window.
static void ahead_launch_decide(const Plan &P, int64_t a, const DecideArgs &A, cudaStream_t st) {
    const Ahead &H = *P.ah;
    const AheadWin &w = H.wins[H.win_of[a]];
    if (w.s0 == a && w.nacc)
        launch_pdl(k_ah_accum, (unsigned)w.nacc, 256, 0, st, A, H.d,
                   (const int64_t *)(H.acc_blk + w.acc_base));
    launch_pdl(k_ah_pass, (unsigned)H.pb_cnt[a], AH_NT, 0, st, A, H.d,
               (const int64_t *)(H.pass_blk + H.pb_base[a]), H.g0[a]);
}

void ahead_stage_args(const Plan &P, int64_t a, StageArgs &S) {
    if (!P.ah || !P.st[a].ahead) return;
    const Ahead &H = *P.ah;
    S.fx.n = H.fx_cnt[a];
    S.fx.src = H.fx_src + H.fx_base[a];
    S.fx.dst = H.fx_dst + H.fx_base[a];
    S.fx.w = H.fx_w + H.fx_base[a];
    S.fx.amove = H.d.amove;
    S.fx.tab = H.d.tab;
    S.fx.tbase = H.d.tbase;
    S.fx.tcap = H.d.tcap;
    S.fx.cold = H.d.cold;
    S.fx.sold = H.d.sold;
}

}  // namespace plv
