// phase.cu -- the phase engine: run_phase (PL/engine.py:166-216) on device.
//
// A phase iterates sweeps over a fixed stage list (the colour classes in
// ascending colour, or all of V) until the reference's stopping rule fires.
// Everything static within a phase is planned once -- decide tiers per stage,
// hub entry layout, event / sort buffers -- and one iteration (every stage's
// decide + exact apply, the move counter, the modularity reduction and a
// 24-byte read-back) is captured into a CUDA graph.  An iteration is then one
// graph launch plus one host synchronisation for the theta test.
//
// Partitioned mode (multi-GPU): rank r of W owns the vertex
// range [bounds[r], bounds[r+1]).  Stages list their vertices in ascending
// id, so a rank's share of a stage is one contiguous slice and rank order is
// subset order.  Per stage, every rank decides its slice only (the decide
// plan covers the rank's slices, and a rank may hold only its own rows), the
// slices' (target, moved, e_old, e_best) are packed into 24-byte records and
// exchanged by ONE in-place NCCL all-gather (slices padded to the stage's
// largest), and every rank replays the whole stage's exact apply -- the
// replicated assignment / a_tot / w_internal / sizes stay bit-identical on
// every rank and to the single-GPU run.  An uncoloured stage needs the movers'
// LIVE e_a / e_b, which only a row's owner can fold: after the first exchange
// each rank folds its own movers' (launch_live), a second all-gather carries
// them, and the apply runs on them as on a colour class.  The collectives are
// captured into the iteration's graph with the kernels.  Without a
// communicator (world > 1, comm NULL) the stages are stepped from the host
// (plv_phase_step: decide, live, apply) and the caller moves the slices
// (gloo in the tests).
#include "localmove.cuh"
#include "nccl_dyn.cuh"
#include "pairwise.cuh"
#include <cub/cub.cuh>
#include <chrono>
#include <cmath>
#include <cstring>

namespace plv {

// Device state of the phase loop (PL/engine.py:203-212 on device).
constexpr int CYC_K = 32;  // ring of recent state hashes (periods 1..CYC_K-1)
struct RunCtl {
    double theta;
    int64_t max_iters;
    int64_t it, total, hit;
    double q_prev;
    int64_t have_prev;
    unsigned long long t0;
    // exact cycle skipping (integral one-stage phases; see k_run_ctl)
    int64_t cyc_on, cyc_mode, cyc_t0, cyc_p, cyc_stop, cyc_done;
    int32_t cyc_cmd, cyc_mismatch;  // k_cycle: 1 snapshot, 2 compare
    unsigned long long ring[CYC_K];
};

struct Phase {
    const int64_t *off;
    const int32_t *nbr;
    const double *wts;
    const double *k;
    const double *selfw;
    const int32_t *labels;
    int64_t n;
    double m;
    int flags;
    int32_t *assign;
    double *a_tot;
    double *w_int;
    int32_t *sizes;
    const int32_t *vtx;       // all stages' active vertices (apply)
    int32_t *fvtx = nullptr;  // the filtered stage lists when some vertex was inactive
    int32_t *pos = nullptr;   // filtered uncoloured stage: subset position per vertex
    int32_t *lvtx = nullptr;  // this rank's slices, stage after stage (decide plan)
    std::vector<int64_t> goff;  // global stage offsets into vtx (nst + 1)
    std::vector<int64_t> slo;   // per stage: W + 1 slice bounds, relative to the stage
    int64_t rank = 0, world = 1;
    void *comm = nullptr;       // ncclComm_t (partitioned, captured exchange)
    const int32_t *deg = nullptr;  // replicated degrees (partitioned rows: activity)
    int *single_bad = nullptr;     // 0: the iteration starts from the singleton state
    unsigned char *xbuf = nullptr;  // exchange records: world x (largest slice) x 24 B
    std::vector<int64_t> xmax;      // per stage: largest slice
    int64_t xcap = 0;               // largest slice of any stage
    bool own_out = true;        // decide outputs allocated here (else the caller's)
    Plan plan;
    ApplyBuffers ab;
    int32_t *target = nullptr;
    uint8_t *moved = nullptr;
    double *e_old = nullptr, *e_best = nullptr;
    unsigned long long *counters = nullptr;  // [0] moves, [1] cand
    double *q = nullptr;
    double *mod_scratch = nullptr;
    double *h_out = nullptr;  // pinned: q, moves, cand
    bool timing = false;
    std::vector<cudaEvent_t> ev;
    cudaStream_t side[NTIER - 1] = {};  // decide tiers in parallel branches
    cudaEvent_t fork = nullptr, join[NTIER - 1] = {};
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    // whole-phase graph: the iteration inside a device-side WHILE loop
    cudaGraph_t rgraph = nullptr;
    cudaGraphExec_t rexec = nullptr;
    RunCtl *ctl = nullptr;         // device loop state
    double *tr_q = nullptr;        // per-iteration trace (capacity tr_cap)
    unsigned long long *tr_mv = nullptr, *tr_t = nullptr;
    int64_t tr_cap = 0;
    bool run_graph_failed = false;
    int64_t graph_kernels = 0;  // kernel nodes in the single-iteration graph
    uint8_t *dirty = nullptr;  // incremental modularity in the device loop (one stage)
    int mod_d0 = 0;
    // exact cycle skipping: XOR hash of the assignment (updated by apply), and
    // the state snapshot the candidate cycle is verified against
    unsigned long long *chash = nullptr;
    int32_t *snap_i = nullptr;  // assign, sizes
    double *snap_d = nullptr;   // a_tot, w_int

    void release_run() {
        cudaDeviceSynchronize();  // buffers go back to the pool idle
        if (rexec) cudaGraphExecDestroy(rexec);
        if (rgraph) cudaGraphDestroy(rgraph);
        rexec = nullptr;
        rgraph = nullptr;
        void *pr[] = {ctl, tr_q, tr_mv, tr_t, dirty, chash, snap_i, snap_d};
        for (void *p : pr)
            pool_free(p);
        ctl = nullptr;
        dirty = nullptr;
        chash = nullptr;
        snap_i = nullptr;
        snap_d = nullptr;
        tr_q = nullptr;
        tr_mv = tr_t = nullptr;
        tr_cap = 0;
    }
    void release() {
        release_run();
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        exec = nullptr;
        graph = nullptr;
        for (auto e : ev) cudaEventDestroy(e);
        ev.clear();
        for (int t = 0; t < NTIER - 1; t++) {
            if (side[t]) cudaStreamDestroy(side[t]);
            if (join[t]) cudaEventDestroy(join[t]);
            side[t] = nullptr;
            join[t] = nullptr;
        }
        if (fork) cudaEventDestroy(fork);
        fork = nullptr;
        plan.release();
        ab.release();
        void *ps[] = {counters, q, mod_scratch, lvtx, fvtx, pos, xbuf, single_bad};
        for (void *p : ps)
            pool_free(p);
        if (own_out) {
            void *po[] = {target, moved, e_old, e_best};
            for (void *p : po)
                pool_free(p);
        }
        lvtx = fvtx = pos = nullptr;
        xbuf = nullptr;
        single_bad = nullptr;
        target = nullptr;
        moved = nullptr;
        e_old = e_best = nullptr;
        counters = nullptr;
        q = mod_scratch = nullptr;
        if (h_out) cudaFreeHost(h_out);
        h_out = nullptr;
    }
};

// Stage a's decide over this rank's slice (outputs at their global positions).
// first: the iteration's first stage, which may see the singleton state
// (*P.single_bad == 0: decided by the k_single_* kernels, decide.cu).
static void record_decide(Phase &P, size_t a, cudaStream_t st, bool first = false) {
    const StagePlan &sp = P.plan.st[a];
    if (!sp.ns) return;
    const int64_t o = P.goff[a] + P.slo[a * (P.world + 1) + P.rank];
    DecideArgs A = make_decide_args(P.off, P.nbr, P.wts, P.k, P.labels, P.lvtx + sp.off, P.assign,
                                    P.a_tot, P.sizes, P.m, (P.flags & PLV_F_INTEGRAL) ? 1 : 0,
                                    P.target + o, P.moved + o, P.e_old + o, P.e_best + o,
                                    P.counters + 1);
    if (first) A.notsingle = P.single_bad;
    if (P.timing) PLV_CUDA(cudaEventRecordWithFlags(P.ev[2 * a], st, cudaEventRecordExternal));
    if (P.timing)
        launch_decide(P.plan, (int64_t)a, A, st);  // serial, so the events bracket all tiers
    else
        launch_decide_par(P.plan, (int64_t)a, A, st, P.side, P.fork, P.join);
    if (P.timing)
        PLV_CUDA(cudaEventRecordWithFlags(P.ev[2 * a + 1], st, cudaEventRecordExternal));
}

// Exchange record of one decided (or live-folded) stage position.
struct XRec {
    int32_t target;
    int32_t moved;
    double e_old, e_best;
};

__global__ void k_xpack(const int32_t *target, const uint8_t *moved, const double *e_old,
                        const double *e_best, int64_t cnt, XRec *out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt;
         t += (int64_t)gridDim.x * blockDim.x)
        out[t] = XRec{target[t], (int32_t)moved[t], e_old[t], e_best[t]};
}

// every other rank's slice back to stage positions (sl: W + 1 slice bounds)
__global__ void k_xunpack(const XRec *in, const int64_t *sl, int W, int rank, int64_t cmax,
                          int32_t *target, uint8_t *moved, double *e_old, double *e_best) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < (int64_t)W * cmax;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(g / cmax);
        const int64_t t = g - (int64_t)r * cmax;
        if (r == rank || t >= sl[r + 1] - sl[r]) continue;
        const XRec x = in[g];
        const int64_t p = sl[r] + t;
        target[p] = x.target;
        moved[p] = (uint8_t)x.moved;
        e_old[p] = x.e_old;
        e_best[p] = x.e_best;
    }
}

// Every rank's slice of stage a to every rank: pack this rank's slice, one
// in-place all-gather of the padded slices, unpack the others.
static void record_exchange(Phase &P, size_t a, cudaStream_t st) {
    if (!P.comm) return;  // (a 1-rank communicator still runs: the capture path)
    const int64_t *sl = P.slo.data() + a * (P.world + 1);
    const int64_t g = P.goff[a], cmax = P.xmax[a];
    if (!cmax) return;
    XRec *xb = (XRec *)P.xbuf;
    const int64_t mine = sl[P.rank + 1] - sl[P.rank];
    const int64_t o = g + sl[P.rank];
    if (mine) {
        k_xpack<<<grid_for(mine, 256), 256, 0, st>>>(P.target + o, P.moved + o, P.e_old + o,
                                                     P.e_best + o, mine, xb + P.rank * cmax);
        PLV_LAUNCH_CHECK();
    }
    nccl_allgather_inplace(xb, sizeof(XRec) * (size_t)cmax, (int)P.rank, P.comm, st);
    if (P.world > 1) {
        // slice bounds of this stage, relative to the stage, on device: kept
        // in the tail of the exchange buffer (written once at creation)
        const int64_t *dsl = (const int64_t *)(P.xbuf + sizeof(XRec) * P.world * P.xcap) + a * (P.world + 1);
        k_xunpack<<<grid_for(P.world * cmax, 256), 256, 0, st>>>(
            xb, dsl, (int)P.world, (int)P.rank, cmax, P.target + g, P.moved + g, P.e_old + g,
            P.e_best + g);
        PLV_LAUNCH_CHECK();
    }
}

// Partitioned uncoloured stage: the live e_a / e_b of this rank's movers.
static void record_live(Phase &P, size_t a, cudaStream_t st);

// Stage a's exact apply over the whole stage (replicated on every rank).
static StageArgs stage_args(const Phase &P, size_t a, uint8_t *dirty, unsigned long long *chash) {
    const int64_t g = P.goff[a], ns = P.goff[a + 1] - g;
    StageArgs S{P.off, P.nbr, P.wts, P.k, P.selfw, P.vtx + g, ns, P.target + g,
                P.moved + g, P.e_old + g, P.e_best + g, P.pos, P.flags,
                P.assign, P.a_tot, P.w_int, P.sizes, P.ab.ta + g, P.ab.tb + g,
                nullptr, nullptr, P.counters};
    S.dirty = dirty;
    S.chash = chash;
    S.tree_n = P.n;
    S.tree_d0 = P.mod_d0;
    return S;
}

// A partitioned uncoloured stage runs decide -> exchange -> live -> exchange
// -> apply: its apply then uses the exchanged live e_a / e_b like a colour
// class does its decide values.
static bool live_mode(const Phase &P) {
    return (P.world > 1 || P.comm) && !(P.flags & PLV_F_INDEPENDENT);
}

static void record_apply(Phase &P, size_t a, cudaStream_t st, uint8_t *dirty = nullptr,
                         unsigned long long *chash = nullptr) {
    StageArgs S = stage_args(P, a, dirty, chash);
    if (live_mode(P)) S.flags = (S.flags | PLV_F_INDEPENDENT) & ~PLV_F_IDENTITY;
    ahead_stage_args(P.plan, (int64_t)a, S);
    launch_apply(S, P.ab, st);
}

static void record_live(Phase &P, size_t a, cudaStream_t st) {
    StageArgs S = stage_args(P, a, nullptr, nullptr);
    const int64_t *sl = P.slo.data() + a * (P.world + 1);
    S.xlo = sl[P.rank];
    S.xhi = sl[P.rank + 1];
    S.live_a = P.e_old + P.goff[a];
    S.live_b = P.e_best + P.goff[a];
    launch_live(S, P.ab, st);
}

static void record_finish(Phase &P, cudaStream_t st) {
    modularity_async(P.w_int, P.a_tot, P.n, P.m, P.q, P.mod_scratch, st);
    PLV_CUDA(cudaMemcpyAsync(P.h_out, P.q, sizeof(double), cudaMemcpyDeviceToHost, st));
    PLV_CUDA(cudaMemcpyAsync(P.h_out + 1, P.counters, 2 * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, st));
}

static void record_iteration(Phase &P, cudaStream_t st) {
    PLV_CUDA(cudaMemsetAsync(P.counters, 0, sizeof(unsigned long long) * 2, st));
    if (P.single_bad) launch_single_check(P.assign, P.sizes, P.n, P.single_bad, st);
    bool first = true;
    for (size_t a = 0; a + 1 < P.goff.size(); a++) {
        if (P.goff[a + 1] == P.goff[a]) continue;
        record_decide(P, a, st, first);
        first = false;
        record_exchange(P, a, st);
        if (live_mode(P)) {
            record_live(P, a, st);
            record_exchange(P, a, st);
        }
        record_apply(P, a, st);
    }
    record_finish(P, st);
}

// Slice bounds of every stage for every rank boundary: sl[a * (W + 1) + r] =
// lower_bound(stage a, bounds[r]) - stage start (stages ascending).
__global__ void k_stage_slices(const int32_t *vtx, const int64_t *goff, int64_t nst,
                               const int64_t *bounds, int64_t W, int64_t *sl) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nst * (W + 1);
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = t / (W + 1), r = t % (W + 1);
        const int64_t b0 = goff[a], b1 = goff[a + 1];
        const int64_t key = bounds[r];
        int64_t lo = b0, hi = b1;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)vtx[mid] < key)
                lo = mid + 1;
            else
                hi = mid;
        }
        sl[t] = lo - b0;
    }
}

// A vertex whose row holds nothing but (at most) its self loop has no
// candidate community: decide keeps it (PL/_kernels.pyx:77-95 with an empty
// e_to) and apply has nothing to do, so stage lists keep only the others.
__global__ void k_active_flags(const int64_t *off, const int32_t *deg, const double *selfw,
                               const int32_t *vtx, int64_t total, int32_t *flag) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = vtx[g];
        const int64_t d = (deg ? (int64_t)deg[i] : off[i + 1] - off[i]) - (selfw[i] != 0.0 ? 1 : 0);
        flag[g] = d > 0 ? 1 : 0;
    }
}

__global__ void k_active_compact(const int32_t *vtx, const int32_t *flag, const int32_t *scan,
                                 int64_t total, int32_t *out) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x)
        if (flag[g]) out[scan[g]] = vtx[g];
}

__global__ void k_gather_offsets(const int32_t *scan, const int32_t *flag, const int64_t *goff,
                                 int64_t nst, int64_t total, int64_t *out) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a <= nst;
         a += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = goff[a];
        out[a] = g < total ? (int64_t)scan[g] : (int64_t)scan[total - 1] + flag[total - 1];
    }
}

__global__ void k_positions(const int32_t *sub, int64_t ns, int32_t *pos) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < ns;
         x += (int64_t)gridDim.x * blockDim.x)
        pos[sub[x]] = (int32_t)x;
}

// Drop inactive vertices from the stage lists (order kept); updates P.vtx,
// P.goff and, for an uncoloured stage, the flags and the position table.
static void filter_active(Phase &P, const int32_t *vtx, int64_t nst, cudaStream_t s) {
    P.vtx = vtx;
    const int64_t total = P.goff[nst];
    if (!total) return;
    Buf<int32_t> flag(total, s), scan(total, s);
    k_active_flags<<<grid_for(total, 256), 256, 0, s>>>(P.off, P.deg, P.selfw, vtx, total, flag);
    PLV_LAUNCH_CHECK();
    size_t tb = 0;
    PLV_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag.get(), scan.get(), total, s));
    Buf<char> tmp(tb, s);
    PLV_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, flag.get(), scan.get(), total, s));
    Buf<int64_t> d_goff(nst + 1, s), d_new(nst + 1, s);
    PLV_CUDA(cudaMemcpyAsync(d_goff.get(), P.goff.data(), sizeof(int64_t) * (nst + 1),
                             cudaMemcpyHostToDevice, s));
    k_gather_offsets<<<grid_for(nst + 1, 256), 256, 0, s>>>(scan, flag, d_goff, nst, total, d_new);
    PLV_LAUNCH_CHECK();
    std::vector<int64_t> nw(nst + 1);
    PLV_CUDA(cudaMemcpyAsync(nw.data(), d_new.get(), sizeof(int64_t) * (nst + 1),
                             cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    if (nw[nst] == total) return;  // every listed vertex is active
    P.fvtx = dalloc<int32_t>(nw[nst]);
    k_active_compact<<<grid_for(total, 256), 256, 0, s>>>(vtx, flag, scan, total, P.fvtx);
    PLV_LAUNCH_CHECK();
    P.vtx = P.fvtx;
    P.goff = nw;
    if (P.flags & PLV_F_IDENTITY) {
        // the stage is no longer arange(n): apply's live rule looks positions up
        P.flags &= ~PLV_F_IDENTITY;
        P.pos = dalloc<int32_t>(P.n);
        PLV_CUDA(cudaMemsetAsync(P.pos, 0xff, sizeof(int32_t) * P.n, s));
        k_positions<<<grid_for(nw[nst], 256), 256, 0, s>>>(P.fvtx, nw[nst], P.pos);
        PLV_LAUNCH_CHECK();
    }
    PLV_CUDA(cudaStreamSynchronize(s));
}

static void capture_iteration(Phase &P) {
    int prio_lo = 0, prio_hi = 0;
    PLV_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    cudaStream_t cs;
    PLV_CUDA(cudaStreamCreateWithPriority(&cs, cudaStreamNonBlocking, prio_hi));
    PLV_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    try {
        record_iteration(P, cs);
    } catch (...) {
        cudaGraph_t g2 = nullptr;
        cudaStreamEndCapture(cs, &g2);
        if (g2) cudaGraphDestroy(g2);
        cudaStreamDestroy(cs);
        throw;
    }
    PLV_CUDA(cudaStreamEndCapture(cs, &P.graph));
    PLV_CUDA(cudaStreamDestroy(cs));
    PLV_CUDA(cudaGraphInstantiate(&P.exec, P.graph, cudaGraphInstantiateFlagUseNodePriority));
    // kernel nodes of one iteration (evidence of the native path for bench.py)
    size_t nn = 0;
    PLV_CUDA(cudaGraphGetNodes(P.graph, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    PLV_CUDA(cudaGraphGetNodes(P.graph, nodes.data(), &nn));
    P.graph_kernels = 0;
    for (auto nd : nodes) {
        cudaGraphNodeType t;
        PLV_CUDA(cudaGraphNodeGetType(nd, &t));
        P.graph_kernels += t == cudaGraphNodeTypeKernel;
    }
}

static Phase *phase_create(const int64_t *off, const int32_t *nbr, const double *wts,
                           const double *k, const double *selfw, int64_t n, double m, int flags,
                           const int32_t *labels, const int64_t *stage_off_h, const int32_t *vtx,
                           int64_t nst, int32_t *assign, double *a_tot, double *w_int,
                           int32_t *sizes, int timing, int64_t rank, int64_t world,
                           const int64_t *bounds_h, void *comm, const int32_t *deg,
                           int32_t *out_target, uint8_t *out_moved, double *out_e_old,
                           double *out_e_best, cudaStream_t s) {
    Phase *P = new Phase();
    try {
        P->off = off;
        P->nbr = nbr;
        P->wts = wts;
        P->k = k;
        P->selfw = selfw;
        P->labels = labels;
        P->n = n;
        P->m = m;
        P->flags = flags;
        P->assign = assign;
        P->a_tot = a_tot;
        P->w_int = w_int;
        P->sizes = sizes;
        P->timing = timing != 0;
        P->rank = rank;
        P->world = world;
        P->comm = comm;
        P->deg = deg;
#ifndef PLV_SINGLE
#define PLV_SINGLE 1  // the singleton-state decide of a phase's first stage (decide.cu)
#endif
        if (PLV_SINGLE) P->single_bad = dalloc<int>(1);
        P->goff.assign(stage_off_h, stage_off_h + nst + 1);
        ensure_decide_attrs();
        filter_active(*P, vtx, nst, s);
        vtx = P->vtx;
        flags = P->flags;
        stage_off_h = P->goff.data();
        int64_t total = stage_off_h[nst];
        // this rank's slice of every stage
        P->slo.assign(nst * (world + 1), 0);
        std::vector<int64_t> loff(nst + 1, 0);
        if (world == 1) {
            for (int64_t a = 0; a < nst; a++) P->slo[2 * a + 1] = stage_off_h[a + 1] - stage_off_h[a];
            loff = P->goff;
            P->lvtx = dalloc<int32_t>(total);
            if (total)
                PLV_CUDA(cudaMemcpyAsync(P->lvtx, vtx, sizeof(int32_t) * total,
                                         cudaMemcpyDeviceToDevice, s));
        } else {
            Buf<int64_t> d_goff(nst + 1, s), d_bounds(world + 1, s), d_sl(nst * (world + 1), s);
            PLV_CUDA(cudaMemcpyAsync(d_goff.get(), stage_off_h, sizeof(int64_t) * (nst + 1),
                                     cudaMemcpyHostToDevice, s));
            PLV_CUDA(cudaMemcpyAsync(d_bounds.get(), bounds_h, sizeof(int64_t) * (world + 1),
                                     cudaMemcpyHostToDevice, s));
            if (nst) {
                k_stage_slices<<<grid_for(nst * (world + 1), 256), 256, 0, s>>>(
                    vtx, d_goff, nst, d_bounds, world, d_sl);
                PLV_LAUNCH_CHECK();
                PLV_CUDA(cudaMemcpyAsync(P->slo.data(), d_sl.get(),
                                         sizeof(int64_t) * nst * (world + 1),
                                         cudaMemcpyDeviceToHost, s));
            }
            PLV_CUDA(cudaStreamSynchronize(s));
            for (int64_t a = 0; a < nst; a++) {
                const int64_t *sl = P->slo.data() + a * (world + 1);
                loff[a + 1] = loff[a] + (sl[rank + 1] - sl[rank]);
            }
            P->lvtx = dalloc<int32_t>(loff[nst]);
            for (int64_t a = 0; a < nst; a++) {
                const int64_t c = loff[a + 1] - loff[a];
                if (c)
                    PLV_CUDA(cudaMemcpyAsync(P->lvtx + loff[a],
                                             vtx + stage_off_h[a] + P->slo[a * (world + 1) + rank],
                                             sizeof(int32_t) * c, cudaMemcpyDeviceToDevice, s));
            }
        }
        // small colour classes of an integral single-rank phase are decided from
        // tables accumulated ahead (ahead.cuh)
        const bool ahead_ok = (flags & PLV_F_INTEGRAL) && (flags & PLV_F_INDEPENDENT) &&
                              world == 1 && !comm;
        plan_build(P->plan, off, P->lvtx, loff.data(), nst, n, s, nbr, wts, ahead_ok);
        if (comm) {  // exchange records + the slice table on device
            P->xmax.assign(nst, 0);
            for (int64_t a = 0; a < nst; a++)
                for (int64_t r = 0; r < world; r++) {
                    const int64_t c = P->slo[a * (world + 1) + r + 1] - P->slo[a * (world + 1) + r];
                    P->xmax[a] = c > P->xmax[a] ? c : P->xmax[a];
                }
            for (int64_t a = 0; a < nst; a++) P->xcap = P->xmax[a] > P->xcap ? P->xmax[a] : P->xcap;
            const size_t rec = sizeof(XRec) * (size_t)world * (size_t)P->xcap;
            P->xbuf = (unsigned char *)pool_alloc(rec + sizeof(int64_t) * P->slo.size());
            if (!P->slo.empty())
                PLV_CUDA(cudaMemcpyAsync(P->xbuf + rec, P->slo.data(), sizeof(int64_t) * P->slo.size(),
                                         cudaMemcpyHostToDevice, s));
        }
        int64_t max_large = 0;
        for (int64_t a = 0; a < nst; a++) {
            const int64_t ns = stage_off_h[a + 1] - stage_off_h[a];
            if (!((flags & PLV_F_INDEPENDENT) && ns <= SMALL_APPLY_MAX))
                max_large = ns > max_large ? ns : max_large;
        }
        P->ab.alloc(total, max_large, n, s);
        P->own_out = !out_target;
        if (P->own_out) {
            P->target = dalloc<int32_t>(total);
            P->moved = dalloc<uint8_t>(total);
            P->e_old = dalloc<double>(total);
            P->e_best = dalloc<double>(total);
        } else {
            P->target = out_target;
            P->moved = out_moved;
            P->e_old = out_e_old;
            P->e_best = out_e_best;
        }
        P->counters = dalloc<unsigned long long>(2);
        PLV_CUDA(cudaMemsetAsync(P->counters, 0, 2 * sizeof(unsigned long long), s));
        P->q = dalloc<double>(1);
        P->mod_scratch = dalloc<double>(modularity_scratch_doubles(n));
        modularity_scratch_init(P->mod_scratch, s);
        PLV_CUDA(cudaMallocHost((void **)&P->h_out, 4 * sizeof(double)));
        if (P->timing) {
            P->ev.resize(2 * nst);
            for (auto &e : P->ev) PLV_CUDA(cudaEventCreate(&e));
        }
        int prio_lo = 0, prio_hi = 0;
        PLV_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        for (int t = 0; t < NTIER - 1; t++) {
            // the hub chain (capture stream) first, then the block tiers (their
            // per-vertex latency is long), the warp / thread tiers last
            int pr = prio_hi + (NTIER - 1 - t);
            if (pr > prio_lo) pr = prio_lo;
            PLV_CUDA(cudaStreamCreateWithPriority(&P->side[t], cudaStreamNonBlocking, pr));
            PLV_CUDA(cudaEventCreateWithFlags(&P->join[t], cudaEventDisableTiming));
        }
        PLV_CUDA(cudaEventCreateWithFlags(&P->fork, cudaEventDisableTiming));
        PLV_CUDA(cudaStreamSynchronize(s));
        // the single-iteration graph is captured on the first plv_phase_iterate
        // (run() only needs the whole-phase graph; comm engines capture now)
        if (comm) capture_iteration(*P);
    } catch (...) {
        cudaStreamSynchronize(s);
        P->release();
        delete P;
        throw;
    }
    return P;
}

static void phase_iterate(Phase *P, cudaStream_t s, double *q, int64_t *moves, int64_t *cand) {
    if (!P->exec) {
        if (P->world > 1 && !P->comm) PLV_FAIL(PLV_EINVAL, "host-stepped partition: use plv_phase_step");
        capture_iteration(*P);
    }
    PLV_CUDA(cudaGraphLaunch(P->exec, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    *q = P->h_out[0];
    unsigned long long c[2];
    memcpy(c, P->h_out + 1, sizeof(c));
    *moves = (int64_t)c[0];
    if (cand) *cand = (int64_t)c[1];
}

static const double ZERO_GUARD = 1e-15;  // PL/engine.py:28

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_run_start(RunCtl *c) { c->t0 = gtimer(); }

// End of one loop iteration: trace row, the reference's stopping rule
// (PL/engine.py:203-212, _iteration_converged :134-137), loop condition.
__global__ void k_run_ctl(RunCtl *c, const double *q, const unsigned long long *counters,
                          double *tr_q, unsigned long long *tr_mv, unsigned long long *tr_t,
                          const unsigned long long *chash, int *single_bad,
                          cudaGraphConditionalHandle h) {
    pdl_wait();  // Q and the move counter
    // a further iteration follows only after moves: no longer the singleton state
    if (single_bad) *single_bad = 1;
    const double q_cur = *q;
    const unsigned long long moves = counters[0];
    const int64_t it = c->it;
    tr_q[it] = q_cur;
    tr_mv[it] = moves;
    tr_t[it] = gtimer();
    c->it = it + 1;
    c->total += (int64_t)moves;
    bool stop = false;
    if (moves == 0) {
        stop = true;
    } else if (c->have_prev) {
        const double qp = c->q_prev;
        const bool conv = fabs(qp) < ZERO_GUARD ? fabs(q_cur - qp) < c->theta
                                                : fabs(q_cur - qp) / fabs(qp) < c->theta;
        stop = conv;
    }
    if (!stop && it + 1 >= c->max_iters) {
        c->hit = 1;
        stop = true;
    }
    c->q_prev = q_cur;
    c->have_prev = 1;
    // Exact cycle skipping.  In an integral graph a_tot / w_int / sizes are
    // exact functions of the assignment, and an iteration is a function of
    // the state, so once the state after iteration done equals the state
    // after done - p, everything repeats with period p: the state after the
    // cap is the state after any iteration congruent to it (mod p), and the
    // trace rows repeat.  A hash match (ring of recent assignment hashes) is
    // a candidate; the state is snapshotted and compared bit for bit p
    // iterations later (k_cycle); once verified -- by then every consecutive
    // pair of Q values in the cycle has passed the stopping test -- the loop
    // runs on only to the next iteration congruent to the cap and the host
    // fills in the remaining trace rows.
    c->cyc_cmd = 0;
    if (c->cyc_on && !stop) {
        const int64_t done = it + 1;
        const unsigned long long H = *chash;
        if (c->cyc_mode == 0) {
            for (int64_t p = 1; p < CYC_K && p < done; p++)
                if (c->ring[(done - p) % CYC_K] == H) {
                    c->cyc_mode = 1;
                    c->cyc_t0 = done;
                    c->cyc_p = p;
                    c->cyc_cmd = 1;  // snapshot the state after iteration done
                    break;
                }
        } else if (c->cyc_mode == 1 && done == c->cyc_t0 + c->cyc_p) {
            c->cyc_mode = 2;
            c->cyc_mismatch = 0;
            c->cyc_cmd = 2;  // compare with the snapshot
        } else if (c->cyc_mode == 2) {
            if (c->cyc_mismatch) {
                c->cyc_mode = 0;  // hash collision
            } else {
                const int64_t t0 = c->cyc_t0, p = c->cyc_p, cap = c->max_iters;
                const int64_t want = (cap - t0) % p;
                int64_t stop_at = done + (((want - (done - t0)) % p) + p) % p;
                c->cyc_mode = 3;
                c->cyc_stop = stop_at;
            }
        }
        if (c->cyc_mode == 3 && done == c->cyc_stop) {
            c->cyc_done = 1;
            c->hit = 1;
            stop = true;
        }
        c->ring[done % CYC_K] = H;
    }
    cudaGraphSetConditional(h, stop ? 0u : 1u);
}

// The cycle check's data side: snapshot (cmd 1) or compare (cmd 2) the state.
__global__ void k_cycle(RunCtl *c, const int32_t *assign, const int32_t *sizes,
                        const double *a_tot, const double *w_int, int64_t n, int32_t *snap_i,
                        double *snap_d) {
    const int cmd = c->cyc_cmd;
    if (!cmd) return;
    bool diff = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (cmd == 1) {
            snap_i[i] = assign[i];
            snap_i[n + i] = sizes[i];
            snap_d[i] = a_tot[i];
            snap_d[n + i] = w_int[i];
        } else {
            // bitwise: -0.0 vs 0.0 or NaN payloads would differ
            diff |= snap_i[i] != assign[i] || snap_i[n + i] != sizes[i] ||
                    __double_as_longlong(snap_d[i]) != __double_as_longlong(a_tot[i]) ||
                    __double_as_longlong(snap_d[n + i]) != __double_as_longlong(w_int[i]);
        }
    }
    if (diff) c->cyc_mismatch = 1;
}

__device__ __forceinline__ unsigned long long vhash(int64_t i, int32_t comm) {
    return mix64(((unsigned long long)i << 32) ^ (unsigned int)comm ^ 0x9E3779B97F4A7C15ull);
}

__global__ void k_hash_assign(const int32_t *assign, int64_t n, unsigned long long *h) {
    unsigned long long x = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x ^= vhash(i, assign[i]);
    for (int o = 16; o > 0; o >>= 1) x ^= __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0 && x) atomicXor(h, x);
}

// Capture the whole phase: k_run_start, then WHILE (condition) { iteration;
// k_run_ctl }.  The per-iteration read-back of the single-iteration graph is
// replaced by the device trace; the host synchronises once per phase.
static void build_run_graph(Phase &P, int64_t cap, cudaStream_t s) {
    P.release_run();
    P.ctl = dalloc<RunCtl>(1);
    P.tr_q = dalloc<double>(cap);
    P.tr_mv = dalloc<unsigned long long>(cap);
    P.tr_t = dalloc<unsigned long long>(cap);
    P.tr_cap = cap;
    // one uncoloured stage (the long, capped phases): the apply marks the tree
    // nodes its movers touch and Q recomputes only those (full on iteration 0);
    // the apply of a one-stage phase always runs k_stage_prep (non-independent)
    int64_t nonempty = 0;
    for (size_t a = 0; a + 1 < P.goff.size(); a++) nonempty += P.goff[a + 1] > P.goff[a];
    if (nonempty == 1 && !(P.flags & PLV_F_INDEPENDENT) &&
        modularity_inc_supported(P.n, &P.mod_d0)) {
        P.dirty = dalloc<uint8_t>((size_t)1 << P.mod_d0);
        PLV_CUDA(cudaMemsetAsync(P.dirty, 0, (size_t)1 << P.mod_d0, s));
    }
#ifndef PLV_CYCLE_FLOAT
#define PLV_CYCLE_FLOAT 0
#endif
    if (nonempty == 1 && !(P.flags & PLV_F_INDEPENDENT) &&
        ((P.flags & PLV_F_INTEGRAL) || PLV_CYCLE_FLOAT)) {
        P.chash = dalloc<unsigned long long>(1);
        P.snap_i = dalloc<int32_t>(2 * P.n);
        P.snap_d = dalloc<double>(2 * P.n);
    }
    PLV_CUDA(cudaGraphCreate(&P.rgraph, 0));
    cudaGraphConditionalHandle h;
    PLV_CUDA(cudaGraphConditionalHandleCreate(&h, P.rgraph, 1, cudaGraphCondAssignDefault));
    cudaGraphNode_t start;
    {
        cudaKernelNodeParams kp = {};
        void *args[] = {(void *)&P.ctl};
        kp.func = (void *)k_run_start;
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(1);
        kp.kernelParams = args;
        PLV_CUDA(cudaGraphAddKernelNode(&start, P.rgraph, nullptr, 0, &kp));
        count_launch();
    }
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t loop;
    cudaGraphNode_t before = start;
    if (P.single_bad)  // iteration 0 may start from the singleton state
        before = add_single_check_nodes(P.rgraph, start, P.assign, P.sizes, P.n, P.single_bad);
    PLV_CUDA(cudaGraphAddNode(&loop, P.rgraph, &before, 1, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    int prio_lo = 0, prio_hi = 0;
    PLV_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    cudaStream_t cs;
    PLV_CUDA(cudaStreamCreateWithPriority(&cs, cudaStreamNonBlocking, prio_hi));
    PLV_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
    try {
        PLV_CUDA(cudaMemsetAsync(P.counters, 0, sizeof(unsigned long long) * 2, cs));
        bool first = true;
        for (size_t a = 0; a + 1 < P.goff.size(); a++) {
            if (P.goff[a + 1] == P.goff[a]) continue;
            record_decide(P, a, cs, first);
            first = false;
            record_apply(P, a, cs, P.dirty, P.chash);
        }
        if (P.dirty)
            modularity_async_inc(P.w_int, P.a_tot, P.n, P.m, P.q, P.mod_scratch, P.dirty,
                                 &P.ctl->it, cs);
        else
            modularity_async(P.w_int, P.a_tot, P.n, P.m, P.q, P.mod_scratch, cs);
        launch_pdl(k_run_ctl, 1, 1, 0, cs, P.ctl, (const double *)P.q,
                   (const unsigned long long *)P.counters, P.tr_q, P.tr_mv, P.tr_t,
                   (const unsigned long long *)P.chash, P.single_bad, h);
        if (P.chash) {
            k_cycle<<<grid_for(P.n, 256, 148 * 8), 256, 0, cs>>>(P.ctl, P.assign, P.sizes, P.a_tot,
                                                                P.w_int, P.n, P.snap_i, P.snap_d);
            PLV_LAUNCH_CHECK();
        }
    } catch (...) {
        cudaGraph_t g2 = nullptr;
        cudaStreamEndCapture(cs, &g2);
        cudaStreamDestroy(cs);
        throw;
    }
    cudaGraph_t got = nullptr;
    PLV_CUDA(cudaStreamEndCapture(cs, &got));
    PLV_CUDA(cudaStreamDestroy(cs));
    PLV_CUDA(cudaGraphInstantiate(&P.rexec, P.rgraph, cudaGraphInstantiateFlagUseNodePriority));
}

// The phase loop on device: returns false when the loop graph is unavailable
// (then the caller runs the host loop).
static bool phase_run_device(Phase &P, double theta, int64_t max_iters, double *q_h,
                             int64_t *mv_h, double *ms_h, int64_t *res_h, cudaStream_t s) {
    if (P.world > 1 || P.comm || P.timing || P.run_graph_failed) return false;
    if (!P.rexec || P.tr_cap < max_iters) {
        try {
            build_run_graph(P, max_iters, s);
        } catch (Fail &) {
            cudaGetLastError();
            P.release_run();
            P.run_graph_failed = true;
            return false;
        }
    }
    RunCtl c0;
    memset(&c0, 0, sizeof(c0));
    c0.theta = theta;
    c0.max_iters = max_iters;
    c0.cyc_on = P.chash ? 1 : 0;
    PLV_CUDA(cudaMemcpyAsync(P.ctl, &c0, sizeof(c0), cudaMemcpyHostToDevice, s));
    if (P.chash) {
        PLV_CUDA(cudaMemsetAsync(P.chash, 0, sizeof(unsigned long long), s));
        k_hash_assign<<<grid_for(P.n, 256, 148 * 8), 256, 0, s>>>(P.assign, P.n, P.chash);
        PLV_LAUNCH_CHECK();
    }
    PLV_CUDA(cudaGraphLaunch(P.rexec, s));
    RunCtl c;
    PLV_CUDA(cudaMemcpyAsync(&c, P.ctl, sizeof(c), cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    const int64_t it = c.it;
    std::vector<unsigned long long> mv(it), tt(it);
    PLV_CUDA(cudaMemcpyAsync(q_h, P.tr_q, sizeof(double) * it, cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaMemcpyAsync(mv.data(), P.tr_mv, sizeof(unsigned long long) * it,
                             cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaMemcpyAsync(tt.data(), P.tr_t, sizeof(unsigned long long) * it,
                             cudaMemcpyDeviceToHost, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    unsigned long long prev = c.t0;
    for (int64_t i = 0; i < it; i++) {
        mv_h[i] = (int64_t)mv[i];
        ms_h[i] = (double)(tt[i] - prev) / 1e6;
        prev = tt[i];
    }
    int64_t iters = it, total = c.total;
    if (c.cyc_done) {
        // rows it+1 .. cap repeat rows t0+1 .. t0+p (1-based iteration numbers)
        const int64_t t0 = c.cyc_t0, p = c.cyc_p;
        for (int64_t x = it + 1; x <= max_iters; x++) {
            const int64_t src = t0 + 1 + ((x - t0 - 1) % p);
            q_h[x - 1] = q_h[src - 1];
            mv_h[x - 1] = mv_h[src - 1];
            ms_h[x - 1] = 0.0;  // not executed
            total += mv_h[x - 1];
        }
        iters = max_iters;
    }
    res_h[0] = iters;
    res_h[1] = total;
    res_h[2] = c.hit;
    res_h[3] = 1;
    res_h[4] = c.cyc_done ? c.cyc_p : 0;
    res_h[5] = c.cyc_done ? it : 0;
    return true;
}


static bool converged(double q_cur, double q_prev, double theta) {  // PL/engine.py:134-137
    if (fabs(q_prev) < ZERO_GUARD) return fabs(q_cur - q_prev) < theta;
    return fabs(q_cur - q_prev) / fabs(q_prev) < theta;
}

}  // namespace plv

extern "C" int plv_phase_create(const int64_t *off, const int32_t *nbr, const double *wts,
                                const double *k, const double *selfw, int64_t n, double m,
                                int flags, const int32_t *labels, const int64_t *stage_off_h,
                                const int32_t *stage_vtx, int64_t nstages, int32_t *assign,
                                double *a_tot, double *w_int, int32_t *sizes, int timing,
                                void **handle_h, void *stream) {
    PLV_ENTRY
    if (!(m > 0.0)) PLV_FAIL(PLV_EINVAL, "modularity undefined for edgeless graph");
    int64_t b[2] = {0, n};
    *handle_h = plv::phase_create(off, nbr, wts, k, selfw, n, m, flags, labels, stage_off_h,
                                  stage_vtx, nstages, assign, a_tot, w_int, sizes, timing, 0, 1, b,
                                  nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                                  plv::S(stream));
    PLV_EXIT
}

static int phase_create_part(const int64_t *off, const int32_t *nbr, const double *wts,
                             const double *k, const double *selfw, int64_t n, double m, int flags,
                             const int32_t *labels, const int64_t *stage_off_h,
                             const int32_t *stage_vtx, int64_t nstages, int32_t *assign,
                             double *a_tot, double *w_int, int32_t *sizes, int64_t rank,
                             int64_t world, const int64_t *bounds_h, void *comm,
                             const int32_t *deg, int32_t *out_target, uint8_t *out_moved,
                             double *out_e_old, double *out_e_best, void **handle_h,
                             void *stream) {
    PLV_ENTRY
    if (!(m > 0.0)) PLV_FAIL(PLV_EINVAL, "modularity undefined for edgeless graph");
    if (world < 1 || rank < 0 || rank >= world) PLV_FAIL(PLV_EINVAL, "bad rank/world");
    if (bounds_h[0] != 0 || bounds_h[world] != n)
        PLV_FAIL(PLV_EINVAL, "partition bounds must run from 0 to n");
    for (int64_t r = 0; r < world; r++)
        if (bounds_h[r + 1] < bounds_h[r]) PLV_FAIL(PLV_EINVAL, "partition bounds must ascend");
    if ((out_target == nullptr) != (out_e_best == nullptr) ||
        (out_target == nullptr) != (out_moved == nullptr) ||
        (out_target == nullptr) != (out_e_old == nullptr))
        PLV_FAIL(PLV_EINVAL, "decide outputs: all four or none");
    *handle_h = plv::phase_create(off, nbr, wts, k, selfw, n, m, flags, labels, stage_off_h,
                                  stage_vtx, nstages, assign, a_tot, w_int, sizes, 0, rank, world,
                                  bounds_h, comm, deg, out_target, out_moved, out_e_old, out_e_best,
                                  plv::S(stream));
    PLV_EXIT
}

extern "C" int plv_phase_create_part(const int64_t *off, const int32_t *nbr, const double *wts,
                                     const double *k, const double *selfw, int64_t n, double m,
                                     int flags, const int32_t *labels, const int64_t *stage_off_h,
                                     const int32_t *stage_vtx, int64_t nstages, int32_t *assign,
                                     double *a_tot, double *w_int, int32_t *sizes, int64_t rank,
                                     int64_t world, const int64_t *bounds_h, void *comm,
                                     int32_t *out_target, uint8_t *out_moved, double *out_e_old,
                                     double *out_e_best, void **handle_h, void *stream) {
    return phase_create_part(off, nbr, wts, k, selfw, n, m, flags, labels, stage_off_h,
                             stage_vtx, nstages, assign, a_tot, w_int, sizes, rank, world,
                             bounds_h, comm, nullptr, out_target, out_moved, out_e_old,
                             out_e_best, handle_h, stream);
}

extern "C" int plv_phase_create_part2(const int64_t *off, const int32_t *nbr, const double *wts,
                                      const double *k, const double *selfw, int64_t n, double m,
                                      int flags, const int32_t *labels, const int64_t *stage_off_h,
                                      const int32_t *stage_vtx, int64_t nstages, int32_t *assign,
                                      double *a_tot, double *w_int, int32_t *sizes, int64_t rank,
                                      int64_t world, const int64_t *bounds_h, void *comm,
                                      const int32_t *deg, int32_t *out_target,
                                      uint8_t *out_moved, double *out_e_old, double *out_e_best,
                                      void **handle_h, void *stream) {
    return phase_create_part(off, nbr, wts, k, selfw, n, m, flags, labels, stage_off_h,
                             stage_vtx, nstages, assign, a_tot, w_int, sizes, rank, world,
                             bounds_h, comm, deg, out_target, out_moved, out_e_old, out_e_best,
                             handle_h, stream);
}

extern "C" int plv_phase_step(void *handle, int64_t stage, int op, double *q_h, int64_t *moves_h,
                              void *stream) {
    PLV_ENTRY
    plv::Phase *P = (plv::Phase *)handle;
    cudaStream_t s = plv::S(stream);
    const int64_t nst = (int64_t)P->goff.size() - 1;
    if (op == PLV_STEP_FINISH) {
        plv::record_finish(*P, s);
        PLV_CUDA(cudaStreamSynchronize(s));
        *q_h = P->h_out[0];
        unsigned long long c[2];
        memcpy(c, P->h_out + 1, sizeof(c));
        *moves_h = (int64_t)c[0];
        PLV_CUDA(cudaMemsetAsync(P->counters, 0, sizeof(unsigned long long) * 2, s));
    } else {
        if (stage < 0 || stage >= nst) PLV_FAIL(PLV_ERANGE, "stage out of range");
        if (P->goff[stage + 1] > P->goff[stage]) {
            if (op == PLV_STEP_DECIDE)
                plv::record_decide(*P, (size_t)stage, s);
            else if (op == PLV_STEP_APPLY)
                plv::record_apply(*P, (size_t)stage, s);
            else if (op == PLV_STEP_LIVE) {
                if (plv::live_mode(*P)) plv::record_live(*P, (size_t)stage, s);
            }
            else
                PLV_FAIL(PLV_EINVAL, "unknown step op");
        }
    }
    PLV_EXIT
}

extern "C" int plv_phase_slices(void *handle, int64_t *stage_off_h, int64_t *slices_h) {
    PLV_ENTRY
    plv::Phase *P = (plv::Phase *)handle;
    memcpy(stage_off_h, P->goff.data(), sizeof(int64_t) * P->goff.size());
    memcpy(slices_h, P->slo.data(), sizeof(int64_t) * P->slo.size());
    PLV_EXIT
}

extern "C" int plv_phase_iterate(void *handle, double *q_h, int64_t *moves_h, int64_t *cand_h,
                                 void *stream) {
    PLV_ENTRY
    plv::phase_iterate((plv::Phase *)handle, plv::S(stream), q_h, moves_h, cand_h);
    PLV_EXIT
}

extern "C" int plv_phase_run(void *handle, double theta, int64_t max_iters, double *q_trace_h,
                             int64_t *moves_trace_h, double *ms_trace_h, int64_t *result_h,
                             void *stream) {
    PLV_ENTRY
    plv::Phase *P = (plv::Phase *)handle;
    cudaStream_t s = plv::S(stream);
    if (max_iters < 1) PLV_FAIL(PLV_EINVAL, "max_iters must be >= 1");
    if (plv::phase_run_device(*P, theta, max_iters, q_trace_h, moves_trace_h, ms_trace_h,
                              result_h, s))
        return PLV_OK;
    int64_t it = 0, total = 0, hit = 0;
    bool have_prev = false;
    double q_prev = 0.0, q_cur = 0.0;
    while (true) {
        auto t0 = std::chrono::steady_clock::now();
        int64_t moves = 0;
        plv::phase_iterate(P, s, &q_cur, &moves, nullptr);
        auto t1 = std::chrono::steady_clock::now();
        q_trace_h[it] = q_cur;
        moves_trace_h[it] = moves;
        ms_trace_h[it] = std::chrono::duration<double, std::milli>(t1 - t0).count();
        it++;
        total += moves;
        if (moves == 0) break;
        if (have_prev && plv::converged(q_cur, q_prev, theta)) break;
        if (it >= max_iters) {
            hit = 1;
            break;
        }
        q_prev = q_cur;
        have_prev = true;
    }
    result_h[0] = it;
    result_h[1] = total;
    result_h[2] = hit;
    result_h[3] = 0;
    result_h[4] = 0;
    result_h[5] = 0;
    PLV_EXIT
}

extern "C" int plv_phase_graph_kernels(void *handle, int64_t *n_h) {
    PLV_ENTRY
    plv::Phase *P = (plv::Phase *)handle;
    if (!P->exec) {
        if (P->world > 1 && !P->comm) PLV_FAIL(PLV_EINVAL, "host-stepped partition has no graph");
        plv::capture_iteration(*P);
    }
    *n_h = P->graph_kernels;
    PLV_EXIT
}

extern "C" int plv_phase_ahead_stats(void *handle, int64_t *out_h) {
    PLV_ENTRY
    plv::Phase *P = (plv::Phase *)handle;
    plv::ahead_stats(P->plan, out_h);
    PLV_EXIT
}

extern "C" int plv_phase_decide_ms(void *handle, double *ms_h) {
    PLV_ENTRY
    plv::Phase *P = (plv::Phase *)handle;
    if (!P->timing) PLV_FAIL(PLV_EINVAL, "phase created without timing");
    double tot = 0.0;
    for (size_t a = 0; a < P->plan.st.size(); a++) {
        if (!P->plan.st[a].ns) continue;
        float ms = 0.f;
        PLV_CUDA(cudaEventElapsedTime(&ms, P->ev[2 * a], P->ev[2 * a + 1]));
        tot += ms;
    }
    *ms_h = tot;
    PLV_EXIT
}

extern "C" int plv_phase_destroy(void *handle) {
    PLV_ENTRY
    plv::Phase *P = (plv::Phase *)handle;
    if (P) {
        const unsigned long long f0 = plv::pool_free_failures();
        P->release();
        delete P;
        if (plv::pool_free_failures() != f0) throw plv::Fail{PLV_ECUDA};  // message set by pool_free
    }
    PLV_EXIT
}
