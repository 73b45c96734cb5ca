// localmove.cuh -- shared declarations of the local-moving hot path
// (decide.cu, apply.cu, phase.cu).
//
// decide (PL/_kernels.pyx:21-101): every subset vertex i aggregates
// e_{i->C} over its neighbours j != i by snapshot community, summed in
// adjacency order per community (fp64, bit-exact with the reference's
// sequential hash accumulation), then takes the argmax of the Eq. 4 gain
// under (gain desc, label asc) with the singleton-pair guard.
//
// apply (PL/_kernels.pyx:104-145) is restated in parallel, bit-exactly:
// e_a / e_b of a mover use the *live* assignment (the target of an
// earlier-moved subset vertex, else the snapshot) and the per-community
// a_tot / w_internal updates are folded in subset order, one thread per
// community, after a stable sort of (community, subset position) events.
#pragma once
#include "common.cuh"
#include <vector>

namespace plv {

constexpr unsigned FULL = 0xffffffffu;
constexpr int T0_MAXD = 12;
constexpr int T1_MAXD = 128;
constexpr int T2A_MAXD = 680;  // tier 2: 1024-slot tables (>= 1.5 * (680 + 1))
constexpr int T2_MAXD = 2048;   // tier 3: 4096-slot tables
constexpr int T1_WARPS = 2;   // warps per block in tier 1 (8, 4, 2, 1 measured; 2 best)
constexpr int T1_TS = 256;    // slots per warp table (>= 1.5 * (128 + 1))
constexpr int BLK = 512;      // threads per block in tier 3 (128/256/1024 measured slower)
constexpr int T2_TS = 4096;   // smem slots for tier 2 (>= 1.5 * (2048 + 1))
constexpr int T2A_TS = 1024;
constexpr int NTIER = 5;  // t0, t1, t2 (block, small table), t3 (block), t4 (hubs)

constexpr int SMALL_APPLY_MAX = 1024;  // stage size handled by the one-CTA apply (2048 measured slower)
constexpr int SA_THREADS = 256;
constexpr int SA_ITEMS = 8;   // 256 * 8 = 2048 events = 2 * SMALL_APPLY_MAX
constexpr uint32_t SENTINEL = 0xFFFFFFFFu;

struct DecideArgs {
    const int64_t *off;
    const int32_t *nbr;
    const double *wts;
    const double *k;
    const int32_t *labels;  // NULL: labels[c] == c
    const int32_t *subset;  // stage vertices
    const int32_t *assign;
    const double *a_tot;
    const int32_t *sizes;
    double m, four_m_sq;
    double inv_m, inv_f;  // 1 / m, 1 / four_m_sq: approximate gains only (never in a result)
    int integral;
    int32_t *out_target;  // per stage index
    uint8_t *out_moved;
    double *out_e_old;
    double *out_e_best;
    unsigned long long *cand;  // nullable: += distinct candidate communities
    // First stage of an iteration: *notsingle == 0 when the state is the
    // singleton state (assign[v] == v for all v) -- then the k_single_* kernels
    // decide and the general tier kernels return at once; nullptr otherwise.
    const int *notsingle = nullptr;
};

DecideArgs make_decide_args(const int64_t *off, const int32_t *nbr, const double *wts,
                            const double *k, const int32_t *labels, const int32_t *subset,
                            const int32_t *assign, const double *a_tot, const int32_t *sizes,
                            double m, int integral, int32_t *out_target, uint8_t *out_moved,
                            double *out_e_old, double *out_e_best, unsigned long long *cand);

struct StagePlan {
    int64_t off = 0, ns = 0;
    int64_t tcount[NTIER] = {0, 0, 0, 0, 0};
    int64_t tstart[NTIER] = {0, 0, 0, 0, 0};  // into the tier list
    int64_t hub_base = 0;              // this stage's first hub_eoff / hub_toff entry
    int64_t hub_entries = 0;
    int64_t hub_nblk = 0;      // hub pass blocks (one per candidate slice)
    int64_t hub_blk_base = 0;  // first of them in hub_blk
    bool hub_dense = false;    // hub tier on dense per-hub community arrays
    bool ahead = false;        // decided from tables accumulated ahead (ahead.cuh)
};

struct Best;  // decide.cu
struct Ahead;  // ahead.cuh: tables of small colour classes accumulated ahead

// A slot of an ahead table: community and its exact integer-valued sum.
struct __align__(16) AheadRec {
    int32_t key;  // -1: empty
    int32_t pad;
    double val;
};

// What a stage's apply needs to push its movers' changes into the ahead tables
// of later stages of the same window (ahead.cuh).
struct AheadFix {
    int64_t n = 0;    // fix entries of this stage (0: none)
    unsigned pb = 0;  // first fix block of the apply launch
    const int32_t *src = nullptr, *dst = nullptr;  // ahead vertex that may move -> later one
    const double *w = nullptr;
    const int2 *amove = nullptr;  // per ahead vertex: (c_old, c_new) of its move, or (-1, -1)
    AheadRec *tab = nullptr;
    const int64_t *tbase = nullptr;
    const uint32_t *tcap = nullptr;
    const int32_t *cold = nullptr;
    int32_t *sold = nullptr;
};

// A dense hub-array entry (hub, community): any-order sum, term count, first
// row position.  16-byte aligned, so one record never spans two sectors.
struct __align__(16) DenseRec {
    double val;
    int32_t cnt;
    int32_t mk;
};

constexpr int MAXS = 32;  // overlapping candidates resolved exactly per vertex

// Static per-phase decide plan: each stage's vertices split into the five
// degree tiers; hubs (tier 4) get entry offsets and a slice of a global hash
// table.
struct Plan {
    std::vector<StagePlan> st;
    int32_t *tier_list = nullptr;  // stage-local indices grouped by (stage, tier)
    int32_t *tier_vid = nullptr;   // the vertex of each tier-list entry
    int64_t *tier_row = nullptr;   // its row [row, end)
    int64_t *tier_end = nullptr;
    int64_t *hub_eoff = nullptr;   // per stage: nh+1 entry offsets (from 0)
    int64_t *hub_toff = nullptr;   // per stage: nh+1 table offsets (from 0, pow2 sizes)
    int64_t *hub_poff = nullptr;   // per stage: nh+1 partial-best offsets (slices)
    int64_t *hub_blk = nullptr;    // pass blocks, (hub << 32) | slice, stage after stage
    int64_t *hub_row = nullptr;    // per stage: nh (+1 pad) row starts
    int32_t *hub_vid = nullptr;    // per stage: nh (+1 pad) hub vertices
    int64_t max_hub_entries = 0, max_hubs = 0, max_table = 0;
    int32_t *hkeys = nullptr;  // hub tables: key -1 / val 0 / cnt 0 when clean
    double *hvals = nullptr;
    int32_t *hcnt = nullptr;
    int32_t *hsold = nullptr;   // per hub: table slot of c_old (-1 idle)
    int32_t *hncnt = nullptr;   // per hub: near-candidate counters (0 idle)
    void *hnear = nullptr;      // per hub: 2 * MAXS near candidates
    Best *hpart = nullptr;      // pass partial bests
    DenseRec *drec = nullptr;   // dense hub records [dense_k * n] (idle: 0 / 0 / INT_MAX)
    int32_t *cbuf = nullptr;    // communities of a dense stage's hub entries
    int64_t dn = 0, max_dense_entries = 0, dense_k = 0;
    int64_t max_slices = 1;
    Ahead *ah = nullptr;  // ahead tables (integral coloured phases; ahead.cuh)
    void release();
};


// nbr / wts / ahead_ok: stages of at most AH_MAX_NS high-degree vertices of an
// integral, single-rank, coloured phase are planned for the ahead tables.
void plan_build(Plan &P, const int64_t *off, const int32_t *vtx, const int64_t *stage_off_h,
                int64_t nst, int64_t n, cudaStream_t s, const int32_t *nbr = nullptr,
                const double *wts = nullptr, bool ahead_ok = false);
void ensure_decide_attrs();
// *bad = 1 unless assign[v] == v and sizes[v] == 1 for every v (the singleton state of
// PL/modularity.py:47-56); *bad must be 0 on entry.
void launch_single_check(const int32_t *assign, const int32_t *sizes, int64_t n, int *bad,
                         cudaStream_t st);
// The same as graph nodes after `dep` (memset, scan); returns the last node.
cudaGraphNode_t add_single_check_nodes(cudaGraph_t g, cudaGraphNode_t dep, const int32_t *assign,
                                       const int32_t *sizes, int64_t n, int *bad);
// Launch stage `a`'s decide kernels (no host synchronisation; capturable).
void launch_decide(const Plan &P, int64_t a, DecideArgs A, cudaStream_t st);
// Tier t on stream ts[t].
void launch_decide_tiers(const Plan &P, int64_t a, DecideArgs A, const cudaStream_t *ts);
// The stage's non-empty tiers as parallel branches (NTIER - 1 side streams, a
// fork event and NTIER - 1 join events), joined back into `st`.
void launch_decide_par(const Plan &P, int64_t a, DecideArgs A, cudaStream_t st,
                       const cudaStream_t *side, cudaEvent_t fork, const cudaEvent_t *join);

struct StageArgs {
    const int64_t *off;
    const int32_t *nbr;
    const double *wts;
    const double *k;
    const double *selfw;
    const int32_t *subset;
    int64_t ns;
    const int32_t *target;
    const uint8_t *moved;
    const double *e_old;
    const double *e_best;
    const int32_t *pos;  // general subsets: subset position per vertex, -1 if absent
    int flags;
    int32_t *assign;
    double *a_tot;
    double *w_int;
    int32_t *sizes;
    double *ta;  // per stage index: 2 e_a + 2 sw (leaving), 2 e_b + 2 sw (joining)
    double *tb;
    uint32_t *ekey;
    int32_t *eval;
    unsigned long long *moves;
    int32_t *ccnt = nullptr;  // small graphs: events per community (counting sort, apply.cu)
    int32_t *big = nullptr;  // high-degree movers (live folds by whole warps)
    unsigned long long *nbig = nullptr;
    int32_t *huge = nullptr;  // huge movers (live folds by whole blocks)
    unsigned long long *nhuge = nullptr;
    unsigned long long *lcnt = nullptr;  // long community runs of the fold (reset by prep)
    // incremental modularity (pairwise.cuh): mark the depth-d0 tree nodes of
    // both communities of every mover (nullptr: off)
    uint8_t *dirty = nullptr;
    unsigned long long *chash = nullptr;  // cycle skipping: XOR hash of the assignment
    int64_t tree_n = 0;
    int tree_d0 = 0;
    // live-only pass of a partitioned uncoloured stage (phase.cu): the live
    // e_a / e_b of the movers at positions [xlo, xhi) go to live_a / live_b
    // and nothing else is written (the replicated apply follows)
    double *live_a = nullptr, *live_b = nullptr;
    int64_t xlo = 0, xhi = 0;
    AheadFix fx;  // an ahead stage's pushes into later ahead tables
};

// Event / sort scratch for stages of up to max_ns vertices.
struct ApplyBuffers {
    double *ta = nullptr, *tb = nullptr;
    uint32_t *ekey = nullptr, *ekey2 = nullptr;
    int32_t *eval = nullptr, *eval2 = nullptr;
    void *tmp = nullptr;
    size_t bytes = 0;
    double *dW = nullptr, *dA = nullptr;  // sorted event deltas (long-run folds)
    int64_t *lrun = nullptr;              // heads of long community runs
    unsigned long long *lcnt = nullptr;
    int32_t *big = nullptr;               // high-degree movers, then huge movers
    unsigned long long *nbig = nullptr;   // [0] big, [1] huge
    int64_t big_cap = 0;
    int nb = 1;
    int64_t n = 0;  // communities (= vertices of the phase's graph)
    int32_t *ccnt = nullptr, *ccur = nullptr;  // counting sort of a small graph's events (n each)
    void alloc(int64_t ta_len, int64_t max_ns, int64_t n, cudaStream_t s);
    void release();
};

// out[0..4]: ahead stages, vertices, windows, fix entries, table slots.
void ahead_stats(const Plan &P, int64_t *out);
// Stage a's ahead fix entries into S.fx (nothing for other stages).
void ahead_stage_args(const Plan &P, int64_t a, StageArgs &S);
// Launch one stage's apply (no host synchronisation; capturable).
void launch_apply(StageArgs S, const ApplyBuffers &B, cudaStream_t st);
// Live e_a / e_b of the movers at positions [S.xlo, S.xhi) into S.live_a / S.live_b
// (a partitioned uncoloured stage; the rows of those movers must be present).
void launch_live(StageArgs S, const ApplyBuffers &B, cudaStream_t st);

template <class T>
T *dalloc(size_t count) {
    T *p = nullptr;
    p = (T *)pool_alloc(sizeof(T) * (count ? count : 1));
    return p;
}

}  // namespace plv
