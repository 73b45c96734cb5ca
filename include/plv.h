/*
 * plv.h -- C ABI of libplv.so, the B200 (sm_100a) parallel-Louvain hot path.
 *
 * Drop-in boundary for the reference package `parlouvain` (arXiv 1410.1237).
 * The reference crosses into native code only through its kernel seam
 * PL/backend.py:13-22 (decide_moves / apply_moves / color_assign /
 * color_conflicts, PL/_kernels.pyx) and otherwise runs numpy on the host
 * (Graph.from_edges, vf_compact, rebuild, modularity).  Each entry point below
 * replaces one of those, cited as PL/<file>:<line>
 * (PL/ = /root/reference/pkg/src/parlouvain/).
 *
 * Conventions
 *  - Every array argument is a DEVICE pointer unless its name ends in `_h`
 *    (host).  Vertex / community ids are int32 (n < 2^31), CSR offsets int64,
 *    weights and aggregates float64.  The caller owns every buffer; the
 *    library allocates only private, stream-ordered scratch.
 *  - `stream` is a cudaStream_t passed as void*.  Work is stream-ordered;
 *    entry points that return sizes through `_h` arguments synchronise the
 *    stream before returning.
 *  - Return value: PLV_OK (0) or a negative PLV_E* code; plv_last_error()
 *    gives a message for the calling thread.  The Python host maps codes to
 *    the reference's exception classes (PL/errors.py).
 *  - No CPU fallback: without a usable sm_100 device every call returns
 *    PLV_ENODEV.
 */
#ifndef PLV_H
#define PLV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PLV_OK 0
#define PLV_EINVAL -1     /* bad argument (ValueError)                        */
#define PLV_EWEIGHT -2    /* non-finite / non-positive weight (GraphParseError) */
#define PLV_ERANGE -3     /* vertex id out of range (ValueError)              */
#define PLV_ECUDA -4      /* CUDA runtime error                               */
#define PLV_ENODEV -5     /* no usable sm_100 device                          */
#define PLV_EDUP -6       /* subset lists a vertex twice (ValueError)         */

int plv_abi_version(void);
const char *plv_last_error(void);
/* 1 when a compute-capability-10.x device is visible, else 0. */
int plv_device_ok(void);
/* Kernels this library has launched so far in this process (CUB's internal
 * sort/scan kernels not included). */
unsigned long long plv_launch_count(void);

/* ---------------------------------------------------------------- sums */

/* ndarray.sum() of a float64 array with numpy's pairwise tree, bit-exact
 * (used by PL/graph.py:80 and PL/modularity.py:64).  out: 1 double. */
int plv_sum(const double *a, int64_t n, double *out, void *stream);

/* modularity (PL/modularity.py:59-64): q = sum(w_int)/2m - sum((a_tot/2m)^2)
 * with both sums as numpy pairwise trees.  out: 1 double. */
int plv_modularity(const double *w_int, const double *a_tot, int64_t n, double m,
                   double *out, void *stream);

/* ------------------------------------------------------------ CSR build */

/*
 * Graph.from_edges (PL/graph.py:88-147) + Graph.__init__ (PL/graph.py:64-86).
 * Records u, v (int32) and w (float64), R of them, in input order.
 * Outputs: off[n+1]; nbr/wts with room for 2*R entries; selfw[n]; k[n].
 * info_h[0..5] = {nnz, merged, num_edges, max_degree, integral, num_self};
 * m_h = total_weight.  `integral` = every merged weight is an integer and the
 * total is < 2^52 (then every downstream sum is exact in any order).
 */
int plv_csr_build(const int32_t *u, const int32_t *v, const double *w, int64_t R, int64_t n,
                  int64_t *off, int32_t *nbr, double *wts, double *selfw, double *k,
                  int64_t *info_h, double *m_h, void *stream);

/* Graph.edge_records (PL/graph.py:169-174): the a <= b half, row-major.
 * ra/rb/rw need room for nnz entries; count_h = records written. */
int plv_edge_records(const int64_t *off, const int32_t *nbr, const double *wts, int64_t n,
                     int32_t *ra, int32_t *rb, double *rw, int64_t *count_h, void *stream);

/* ----------------------------------------------------- vertex following */

/*
 * vf_compact (PL/heuristics.py:46-89): vertex_map[n] (int32) plus the
 * compacted graph's records (kept edge_records, then (t,t,w) per folded
 * vertex in ascending id); rec_* need room for nnz + n entries.
 * info_h = {n_new, merged_count, num_records}.  Feed the records to
 * plv_csr_build to finish the compaction (PL/heuristics.py:85-87).
 */
int plv_vf_records(const int64_t *off, const int32_t *nbr, const double *wts,
                   const double *selfw, int64_t n, int32_t *vertex_map, int32_t *rec_u,
                   int32_t *rec_v, double *rec_w, int64_t *info_h, void *stream);

/* ------------------------------------------------------------- coloring */

/*
 * color_graph (PL/heuristics.py:92-118): speculative rounds of color_assign
 * (PL/_kernels.pyx:148-174) and color_conflicts (PL/_kernels.pyx:177-195)
 * until no vertex is rejected; rejects keep ascending order.
 * colors[n] (int32).  info_h = {num_colors, rounds}.
 */
int plv_color(const int64_t *off, const int32_t *nbr, int64_t n, int64_t max_degree,
              int32_t *colors, int64_t *info_h, void *stream);

/* Kernel-granular seam twins (PL/_kernels.pyx:148-195); `colors` may hold -1. */
int plv_color_assign(const int64_t *off, const int32_t *nbr, const int32_t *active, int64_t na,
                     const int32_t *colors, int32_t *out_colors, void *stream);
int plv_color_conflicts(const int64_t *off, const int32_t *nbr, const int32_t *active,
                        int64_t na, const int32_t *colors, uint8_t *out_keep, void *stream);

/* Coloring.classes (PL/heuristics.py:34-38): class_off[num_colors+1] and the
 * vertices of every class in ascending id (stable sort by colour). */
int plv_color_classes(const int32_t *colors, int64_t n, int64_t num_colors, int64_t *class_off,
                      int32_t *class_vtx, void *stream);

/* ----------------------------------------------------------- local move */

/* Flags for plv_apply / plv_iteration. */
#define PLV_F_INDEPENDENT 1  /* no two subset vertices are adjacent (colour class) */
#define PLV_F_INTEGRAL 2     /* graph weights integral: aggregate in any order   */
#define PLV_F_IDENTITY 4     /* subset == arange(n)                              */

/*
 * decide_moves (PL/_kernels.pyx:21-101) for every subset vertex against the
 * state at entry (the reference's snapshot, PL/engine.py:150-152).
 * labels may be NULL (labels[c] == c, the case for every state the engine
 * builds, PL/modularity.py:52).  Outputs per subset index: target, moved,
 * e_old (= e_{i->c_old}), e_best (= e_{i->target}).  cand_h (nullable) receives
 * sum over the subset of distinct neighbour communities (roofline bytes).
 */
int plv_decide(const int64_t *off, const int32_t *nbr, const double *wts, const double *k,
               const int32_t *labels, const int32_t *subset, int64_t ns, const int32_t *assign,
               const double *a_tot, const int32_t *sizes, double m, int32_t *out_target,
               uint8_t *out_moved, double *out_e_old, double *out_e_best, int64_t *cand_h,
               void *stream);

/* plv_decide with flags (PLV_F_INTEGRAL selects order-free accumulation, exact
 * for integral graphs). */
int plv_decide_ex(const int64_t *off, const int32_t *nbr, const double *wts, const double *k,
                  const int32_t *labels, const int32_t *subset, int64_t ns,
                  const int32_t *assign, const double *a_tot, const int32_t *sizes, double m,
                  int flags, int32_t *out_target, uint8_t *out_moved, double *out_e_old,
                  double *out_e_best, int64_t *cand_h, void *stream);

/*
 * apply_moves (PL/_kernels.pyx:104-145): applies the decided moves as if
 * sequentially in subset order against the live assignment, bit-exactly
 * (parallel restatement: live e_a/e_b from the decide snapshot plus the
 * targets of earlier subset vertices, then one ordered fold per community).
 * moves_h = number of moves (PL/_kernels.pyx:145).
 */
int plv_apply(const int64_t *off, const int32_t *nbr, const double *wts, const double *k,
              const double *selfw, int64_t n, const int32_t *subset, int64_t ns,
              const int32_t *target, const uint8_t *moved, const double *e_old,
              const double *e_best, int flags, int32_t *assign, double *a_tot, double *w_int,
              int32_t *sizes, int64_t *moves_h, void *stream);

/* ----------------------------------------------------------- phase engine */

/*
 * run_phase (PL/engine.py:166-216) on a fixed stage list: the colour classes
 * in ascending colour (PLV_F_INDEPENDENT) or all of V (PLV_F_IDENTITY), plus
 * PLV_F_INTEGRAL for integral graphs.  stage_off_h (host, nstages+1) indexes
 * stage_vtx (device, concatenated stage vertices, ascending within a stage).
 * The state buffers (assign/a_tot/w_int/sizes) are updated in place by every
 * iteration.  Creation plans the decide tiers per stage and captures one
 * iteration (all stages' decide + exact apply, move counter, modularity) into
 * a CUDA graph; `timing` adds event records around every stage's decide.
 */
int plv_phase_create(const int64_t *off, const int32_t *nbr, const double *wts, const double *k,
                     const double *selfw, int64_t n, double m, int flags, const int32_t *labels,
                     const int64_t *stage_off_h, const int32_t *stage_vtx, int64_t nstages,
                     int32_t *assign, double *a_tot, double *w_int, int32_t *sizes, int timing,
                     void **handle_h, void *stream);
/* One iteration (PL/engine.py:187-197): q_h = Q after it, moves_h = moves,
 * cand_h (nullable) = sum of distinct candidate communities over all deciders. */
int plv_phase_iterate(void *handle, double *q_h, int64_t *moves_h, int64_t *cand_h, void *stream);
/* The phase loop with the reference's stopping rule (PL/engine.py:203-212):
 * per-iteration Q / moves / milliseconds into the *_trace_h arrays (capacity
 * max_iters); result_h (6 values) = {iterations, total_moves, hit_cap,
 * device_loop, cycle_period, iterations_executed}.
 * Single-GPU engines run the loop on the device (one CUDA graph: the
 * iteration inside a WHILE conditional node, stopping rule and trace in a
 * control kernel; milliseconds from the GPU global timer, device_loop = 1);
 * otherwise one graph launch + host test per iteration (device_loop = 0).
 * Integral graphs with one (uncoloured) stage skip exact cycles: when the
 * state after an iteration equals the state p iterations earlier (hash
 * candidate, then a bitwise comparison), the loop stops at the next
 * iteration congruent to the cap and the remaining trace rows are the
 * cycle's (milliseconds 0): same final state, same trace as running to the
 * cap (cycle_period = p, else 0). */
int plv_phase_run(void *handle, double theta, int64_t max_iters, double *q_trace_h,
                  int64_t *moves_trace_h, double *ms_trace_h, int64_t *result_h, void *stream);
/*
 * Partitioned phase (multi-GPU; the reference has no distributed mode -- new
 * design of SURVEY.md 8e, no reference interface replaced).  Rank `rank` of
 * `world` owns vertices [bounds_h[rank], bounds_h[rank+1]) (bounds_h: world+1
 * ascending host values from 0 to n) and decides only its slice of every
 * stage; the decided slices are exchanged with NCCL in-place broadcasts over
 * `comm` (an ncclComm_t from plv_nccl_comm_init), captured in the iteration
 * graph, and every rank applies whole stages, so the replicated state stays
 * bit-identical to plv_phase_create's.  comm NULL with world > 1: no graph;
 * the caller steps the stages (plv_phase_step) and moves the slices between
 * ranks' decide outputs itself.  out_* (device, capacity stage_off_h[nstages];
 * all four or none) are the decide outputs at global stage positions; NULL =
 * allocated by the library.
 */
int plv_phase_create_part(const int64_t *off, const int32_t *nbr, const double *wts,
                          const double *k, const double *selfw, int64_t n, double m, int flags,
                          const int32_t *labels, const int64_t *stage_off_h,
                          const int32_t *stage_vtx, int64_t nstages, int32_t *assign,
                          double *a_tot, double *w_int, int32_t *sizes, int64_t rank,
                          int64_t world, const int64_t *bounds_h, void *comm, int32_t *out_target,
                          uint8_t *out_moved, double *out_e_old, double *out_e_best,
                          void **handle_h, void *stream);
#define PLV_STEP_DECIDE 0 /* decide this rank's slice of `stage`              */
#define PLV_STEP_APPLY 1  /* exact apply of the whole of `stage`               */
#define PLV_STEP_FINISH 2 /* modularity; q_h / moves_h of the stepped iteration */
#define PLV_STEP_LIVE 3   /* uncoloured stage: live e_a / e_b of this rank's movers (the
                             reference's apply folds, PL/_kernels.pyx:116-136) into
                             the slice's e_old / e_best, to be exchanged before APPLY */
int plv_phase_step(void *handle, int64_t stage, int op, double *q_h, int64_t *moves_h,
                   void *stream);
/* The engine's stage offsets (nstages+1; stage lists keep only vertices with
 * a non-self neighbour -- the others never move) and the slice bounds of
 * every stage (nstages * (world+1), relative to the stage). */
int plv_phase_slices(void *handle, int64_t *stage_off_h, int64_t *slices_h);

/* plv_phase_create_part on a graph holding only the rows of this rank's
 * vertices (off / nbr / wts with empty rows elsewhere; k / selfw replicated):
 * deg (n, replicated) gives every vertex's degree for the stage lists'
 * activity rule.  In this mode an uncoloured stage folds its movers' live
 * e_a / e_b on their owner (PLV_STEP_LIVE) and exchanges them; with a
 * communicator the exchange is one in-place ncclAllGather of 24-byte records
 * per stage (and per live step), captured in the iteration graph. */
int plv_phase_create_part2(const int64_t *off, const int32_t *nbr, const double *wts,
                           const double *k, const double *selfw, int64_t n, double m, int flags,
                           const int32_t *labels, const int64_t *stage_off_h,
                           const int32_t *stage_vtx, int64_t nstages, int32_t *assign,
                           double *a_tot, double *w_int, int32_t *sizes, int64_t rank,
                           int64_t world, const int64_t *bounds_h, void *comm,
                           const int32_t *deg, int32_t *out_target, uint8_t *out_moved,
                           double *out_e_old, double *out_e_best, void **handle_h, void *stream);

/* NCCL communicator for plv_phase_create_part (NCCL is bound at run time). */
#define PLV_NCCL_ID_BYTES 128
int plv_nccl_unique_id(uint8_t *id_h);
int plv_nccl_comm_init(int64_t rank, int64_t world, const uint8_t *id_h, void **comm_h);
int plv_nccl_comm_destroy(void *comm);

/* Kernel nodes in the engine's single-iteration CUDA graph (captured now if
 * needed): the kernels one plv_phase_iterate launches. */
int plv_phase_graph_kernels(void *handle, int64_t *n_h);
/* Ahead tables of the engine's plan (integral coloured single-rank phases:
 * small high-degree colour classes are decided from per-vertex tables
 * accumulated at the start of their window of stages, csrc/ahead.cuh):
 * out_h[0] stages, [1] vertices, [2] windows, [3] static fix entries,
 * [4] table slots.  All zero when the plan has none. */
int plv_phase_ahead_stats(void *handle, int64_t *out_h);
/* Sum over stages of the decide time of the last iteration (timing handles). */
int plv_phase_decide_ms(void *handle, double *ms_h);
int plv_phase_destroy(void *handle);

/* ---------------------------------------------------------------- rebuild */

/*
 * rebuild (PL/engine.py:229-256) up to the from_edges call: renumber[n]
 * (int32, -1 for empty community ids, dense in ascending id), and the merged,
 * (lo, hi)-sorted coarse records lo/hi/w (room for nnz entries).
 * info_h = {n_new, num_records}.  Finish with plv_csr_from_sorted.
 */
int plv_rebuild_records(const int64_t *off, const int32_t *nbr, const double *wts, int64_t n,
                        const int32_t *assign, int32_t *renumber, int32_t *lo, int32_t *hi,
                        double *w, int64_t *info_h, void *stream);

/* Graph.from_edges on records already sorted by (a, b) with a <= b and no
 * duplicates (sorting and merging are then the identity); same outputs as
 * plv_csr_build. */
int plv_csr_from_sorted(const int32_t *a, const int32_t *b, const double *w, int64_t M,
                        int64_t n, int64_t *off, int32_t *nbr, double *wts, double *selfw,
                        double *k, int64_t *info_h, double *m_h, void *stream);

/* Hierarchy.flatten step (PL/engine.py:115): out[i] = renumber[assign[map[i]]]
 * (map may be NULL = identity). */
int plv_compose(const int32_t *map, const int32_t *assign, const int32_t *renumber, int64_t n,
                int32_t *out, void *stream);

/* ---------------------------------------------------------------- ingest */

/*
 * load_graph's edge-list branch (PL/graph.py:245-288) on
 * device: `text` (device, len bytes) is the file; record lines `u v [w]`
 * become u / v (int32, dense ids kept as in the file) and w (f64) in file
 * order, capacity cap.  info_h = {records, n}.  Returns PLV_INGEST_HOST
 * (> 0) when the file needs the host parser's rules: characters other than
 * ASCII digits, signs, '.', 'e' and blanks; a malformed line; a weight that
 * is not a plain decimal on Clinger's exact fast path or is not positive; ids
 * that do not already form 0..n-1 (renumbering by first appearance); an
 * empty file.  The host parser then reproduces the reference's result or its
 * error with the line number.
 */
#define PLV_INGEST_HOST 1
int plv_parse_edge_list(const uint8_t *text, int64_t len, int32_t *u, int32_t *v, double *w,
                        int64_t cap, int64_t *info_h, void *stream);

/* load_graph's Matrix Market branch (PL/graph.py:412-478) on device: `text`
 * is the file after its size line (the banner and size line are read on the
 * host); symmetric coordinate lines `i j [w]` (pattern: no w), '%' comments,
 * 1-based indices in [1, rows].  u / v (0-based int32), w in file order;
 * info_h[0] = records.  PLV_INGEST_HOST when the host rules must decide. */
int plv_parse_mm(const uint8_t *text, int64_t len, int64_t rows, int pattern, int32_t *u,
                 int32_t *v, double *w, int64_t cap, int64_t *info_h, void *stream);
/* load_graph's METIS branch (PL/graph.py:326-411) on device: `text` is the
 * file after its header line (n, m_declared and the edge-weight flag read on
 * the host).  Every non-comment line is the next vertex's adjacency list.
 * Accepted: no repeated neighbour, every edge in both directions with
 * bitwise-equal weights, exactly m_declared edges; out: the upper entries
 * (vertex <= neighbour) in file order, the reference's records.
 * PLV_INGEST_HOST otherwise (the host rules merge, tolerate or raise). */
int plv_parse_metis(const uint8_t *text, int64_t len, int64_t n, int64_t m_declared,
                    int weighted, int32_t *u, int32_t *v, double *w, int64_t cap,
                    int64_t *info_h, void *stream);

/* ------------------------------------------------------- post-processing */

/* write_assignment's file body (PL/engine.py:318-322): "i c\n" per vertex,
 * decimal, from a device assignment of int32 (elem_bytes 4) or int64 (8).
 * len_h = the byte length; the text is written to out (device) only when it
 * fits cap. */
int plv_format_assignment(const void *assign, int elem_bytes, int64_t n, uint8_t *out,
                          int64_t cap, int64_t *len_h, void *stream);
/* compare_partitions' contingency counts (PL/evaluation.py:68-86) for int64
 * labelings s, p of n vertices: out_h = {sum over (s,p) cells of C(cell,2),
 * sum over classes of s of C(class,2), same for p}. */
int plv_pair_counts(const int64_t *s, const int64_t *p, int64_t n, int64_t *out_h, void *stream);

/* ------------------------------------------------------------ generators */

/* Counter-based synthetic graphs (BASELINE.json configs), identical to the
 * numpy generators in paper_1410_1237_b200/synthetic.py.  Each writes records
 * (u, v, w) into caller buffers of capacity `cap` and returns the count in
 * count_h. */
int plv_gen_rmat(uint64_t seed, int scale, int64_t edge_factor, double a, double b, double c,
                 double w_lo, double w_hi, int32_t *u, int32_t *v, double *w, int64_t cap,
                 int64_t *count_h, void *stream);
int plv_gen_sbm(uint64_t seed, int64_t n, int64_t block, double p_in, double p_out, int32_t *u,
                int32_t *v, double *w, int64_t cap, int64_t *count_h, void *stream);
int plv_gen_grid(uint64_t seed, int64_t side, double keep, int64_t pendants, double w_lo,
                 int32_t *u, int32_t *v, double *w, int64_t cap, int64_t *count_h,
                 void *stream);
/* Chung-Lu: endpoints drawn by searchsorted(cdf, U * cdf[n-1], 'right'). */
int plv_gen_chung_lu(uint64_t seed, const double *cdf, int64_t n, int64_t records, int32_t *u,
                     int32_t *v, double *w, int64_t cap, int64_t *count_h, void *stream);

/* ---------------------------------------------------- 1D vertex partition
 * (new design -- the reference has no distributed mode).  Rank
 * r owns vertices [bounds[r], bounds[r+1]) and holds only their rows; the
 * host driver (paper_1410_1237_b200/partition.py) moves data between ranks.
 */

/* R-MAT records of draws [r_begin, r_end) (plv_gen_rmat restricted: the
 * ranges of all ranks concatenate to plv_gen_rmat's output). */
int plv_gen_rmat_range(uint64_t seed, int scale, int64_t edge_factor, double a, double b,
                       double c, double w_lo, double w_hi, int64_t r_begin, int64_t r_end,
                       int32_t *u, int32_t *v, double *w, int64_t cap, int64_t *count_h,
                       void *stream);
/* Route records to the owners of both endpoints (Graph.from_edges,
 * PL/graph.py:88-147, split by rows): every record once per distinct owner,
 * grouped by destination rank, input order kept within a group.  bounds:
 * device, world+1.  send_counts_h[world].  R < 2^31 per call. */
int plv_route_records(const int32_t *u, const int32_t *v, const double *w, int64_t R,
                      const int64_t *bounds, int world, int32_t *ou, int32_t *ov, double *ow,
                      int64_t cap, int64_t *send_counts_h, void *stream);
/* Keep rows [lo, hi) of a CSR (off n+1): out_off (n+1, empty rows outside),
 * out_nbr / out_wts (the rows' entries), deg[n] (zero outside).  info_h =
 * {entries, self loops, unique pairs (nbr >= row), max degree, non-integral}. */
int plv_part_own_rows(const int64_t *off, const int32_t *nbr, const double *wts, int64_t n,
                      int64_t lo, int64_t hi, int64_t *out_off, int32_t *out_nbr,
                      double *out_wts, int32_t *deg, int64_t *info_h, void *stream);
/* vf_compact (PL/heuristics.py:46-89) on owned rows: only_p1[v] = the single
 * neighbour + 1 of owned candidates, 0 elsewhere (to be summed over ranks). */
int plv_part_vf_only(const int64_t *off, const int32_t *nbr, const int32_t *deg,
                     const double *selfw, int64_t n, int64_t lo, int64_t hi, int32_t *only_p1,
                     void *stream);
/* ... from the replicated only_p1: merged flags, new_id (n+1, exclusive scan
 * of the survivors) and vertex_map; info_h = {n_new, merged_count}. */
int plv_part_vf_map(const int32_t *only_p1, int64_t n, uint8_t *merged, int32_t *new_id,
                    int32_t *vertex_map, int64_t *info_h, void *stream);
/* ... the owned rows' compacted records: kept (a <= b, row-major) and folded
 * (t, t, w) per owned merged vertex in ascending id; counts_h = {kept, folded}. */
int plv_part_vf_records(const int64_t *off, const int32_t *nbr, const double *wts, int64_t n,
                        int64_t lo, int64_t hi, const uint8_t *merged, const int32_t *new_id,
                        const int32_t *only_p1, int32_t *ku, int32_t *kv, double *kw,
                        int32_t *fu, int32_t *fv, double *fw, int64_t *counts_h, void *stream);
/* out[idx[t]] = val ? val[t] : fill (colour rounds, PL/heuristics.py:109-113). */
int plv_scatter_i32(const int32_t *idx, const int32_t *val, int32_t fill, int64_t cnt,
                    int32_t *out, void *stream);
/* active[t] for every keep[t] == 0, in order (PL/heuristics.py:114). */
int plv_select_rejected(const int32_t *active, const uint8_t *keep, int64_t na, int32_t *out,
                        int64_t *count_h, void *stream);
/* rebuild's renumbering (PL/engine.py:237-239): renumber[n] dense in ascending
 * community id, -1 for empty ids. */
int plv_renumber(const int32_t *assign, int64_t n, int32_t *renumber, int64_t *n_new_h,
                 void *stream);
/* rebuild's records (PL/engine.py:240-243) of the owned rows, row-major:
 * (renumber[assign[a]], renumber[assign[b]], w) for every entry b >= a. */
int plv_part_rebuild_records(const int64_t *off, const int32_t *nbr, const double *wts,
                             int64_t n, int64_t lo, int64_t hi, const int32_t *assign,
                             const int32_t *renumber, int32_t *ou, int32_t *ov, double *ow,
                             int64_t *count_h, void *stream);

/* ------------------------------------------------------------ diagnostics */

/* Per-block timeline of the decide kernels (tools/ktrace.py): plv_debug_trace(1)
 * starts recording globaltimer stamps (thread 0 of each block) and clears the
 * buffer, plv_debug_trace(0) stops (and clears); plv_debug_trace_read copies up
 * to max_records records of 8 u64 [kernel id << 32 | block, stamps t0..t5,
 * number of stamps] and returns their count in n_h.  No reference counterpart
 * (profiling aid). */
int plv_debug_trace(int on);
int plv_debug_trace_read(unsigned long long *out_h, int64_t max_records, int64_t *n_h);

#ifdef __cplusplus
}
#endif
#endif /* PLV_H */
