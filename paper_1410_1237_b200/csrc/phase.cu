// phase.cu -- the phase engine: run_phase (PL/engine.py:166-216) on device.
//
// A phase iterates sweeps over a fixed stage list (the colour classes in
// ascending colour, or all of V) until the reference's stopping rule fires.
// Everything static within a phase is planned once -- decide tiers per stage,
// hub entry layout, event / sort buffers -- and one iteration (every stage's
// decide + exact apply, the move counter, the modularity reduction and a
// 24-byte read-back) is captured into a CUDA graph.  An iteration is then one
// graph launch plus one host synchronisation for the theta test.
#include "localmove.cuh"
#include "pairwise.cuh"
#include <chrono>
#include <cmath>
#include <cstring>

namespace plv {

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
    const int32_t *vtx;
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

    void release() {
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
        void *ps[] = {target, moved, e_old, e_best, counters, q, mod_scratch};
        for (void *p : ps)
            if (p) cudaFree(p);
        if (h_out) cudaFreeHost(h_out);
        h_out = nullptr;
    }
};

static void record_iteration(Phase &P, cudaStream_t st) {
    PLV_CUDA(cudaMemsetAsync(P.counters, 0, sizeof(unsigned long long) * 2, st));
    for (size_t a = 0; a < P.plan.st.size(); a++) {
        const StagePlan &sp = P.plan.st[a];
        if (!sp.ns) continue;
        DecideArgs A = make_decide_args(P.off, P.nbr, P.wts, P.k, P.labels, P.vtx + sp.off,
                                        P.assign, P.a_tot, P.sizes, P.m,
                                        (P.flags & PLV_F_INTEGRAL) ? 1 : 0, P.target + sp.off,
                                        P.moved + sp.off, P.e_old + sp.off, P.e_best + sp.off,
                                        P.counters + 1);
        if (P.timing)
            PLV_CUDA(cudaEventRecordWithFlags(P.ev[2 * a], st, cudaEventRecordExternal));
        if (P.timing)
            launch_decide(P.plan, (int64_t)a, A, st);  // serial, so the events bracket all tiers
        else
            launch_decide_par(P.plan, (int64_t)a, A, st, P.side, P.fork, P.join);
        if (P.timing)
            PLV_CUDA(cudaEventRecordWithFlags(P.ev[2 * a + 1], st, cudaEventRecordExternal));
        StageArgs S{P.off, P.nbr, P.wts, P.k, P.selfw, P.vtx + sp.off, sp.ns, P.target + sp.off,
                    P.moved + sp.off, P.e_old + sp.off, P.e_best + sp.off, nullptr, P.flags,
                    P.assign, P.a_tot, P.w_int, P.sizes, P.ab.ta + sp.off, P.ab.tb + sp.off,
                    nullptr, nullptr, P.counters};
        launch_apply(S, P.ab, st);
    }
    modularity_async(P.w_int, P.a_tot, P.n, P.m, P.q, P.mod_scratch, st);
    PLV_CUDA(cudaMemcpyAsync(P.h_out, P.q, sizeof(double), cudaMemcpyDeviceToHost, st));
    PLV_CUDA(cudaMemcpyAsync(P.h_out + 1, P.counters, 2 * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, st));
}

static Phase *phase_create(const int64_t *off, const int32_t *nbr, const double *wts,
                           const double *k, const double *selfw, int64_t n, double m, int flags,
                           const int32_t *labels, const int64_t *stage_off_h, const int32_t *vtx,
                           int64_t nst, int32_t *assign, double *a_tot, double *w_int,
                           int32_t *sizes, int timing, cudaStream_t s) {
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
        P->vtx = vtx;
        P->timing = timing != 0;
        ensure_decide_attrs();
        plan_build(P->plan, off, vtx, stage_off_h, nst, n, s);
        int64_t total = stage_off_h[nst];
        int64_t max_large = 0;
        for (auto &sp : P->plan.st)
            if (!((flags & PLV_F_INDEPENDENT) && sp.ns <= SMALL_APPLY_MAX))
                max_large = sp.ns > max_large ? sp.ns : max_large;
        P->ab.alloc(total, max_large, n, s);
        P->target = dalloc<int32_t>(total);
        P->moved = dalloc<uint8_t>(total);
        P->e_old = dalloc<double>(total);
        P->e_best = dalloc<double>(total);
        P->counters = dalloc<unsigned long long>(2);
        P->q = dalloc<double>(1);
        P->mod_scratch = dalloc<double>(modularity_scratch_doubles(n));
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
        cudaStream_t cs;
        PLV_CUDA(cudaStreamCreateWithPriority(&cs, cudaStreamNonBlocking, prio_hi));
        PLV_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        try {
            record_iteration(*P, cs);
        } catch (...) {
            cudaGraph_t g2 = nullptr;
            cudaStreamEndCapture(cs, &g2);
            if (g2) cudaGraphDestroy(g2);
            cudaStreamDestroy(cs);
            throw;
        }
        PLV_CUDA(cudaStreamEndCapture(cs, &P->graph));
        PLV_CUDA(cudaStreamDestroy(cs));
        PLV_CUDA(cudaGraphInstantiate(&P->exec, P->graph, cudaGraphInstantiateFlagUseNodePriority));
    } catch (...) {
        cudaStreamSynchronize(s);
        P->release();
        delete P;
        throw;
    }
    return P;
}

static void phase_iterate(Phase *P, cudaStream_t s, double *q, int64_t *moves, int64_t *cand) {
    PLV_CUDA(cudaGraphLaunch(P->exec, s));
    PLV_CUDA(cudaStreamSynchronize(s));
    *q = P->h_out[0];
    unsigned long long c[2];
    memcpy(c, P->h_out + 1, sizeof(c));
    *moves = (int64_t)c[0];
    if (cand) *cand = (int64_t)c[1];
}

static const double ZERO_GUARD = 1e-15;  // PL/engine.py:28

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
    *handle_h = plv::phase_create(off, nbr, wts, k, selfw, n, m, flags, labels, stage_off_h,
                                  stage_vtx, nstages, assign, a_tot, w_int, sizes, timing,
                                  plv::S(stream));
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
        P->release();
        delete P;
    }
    PLV_EXIT
}
