/*
 * plv_oracle.c -- CPU restatement of the parallel-Louvain hot path of the
 * reference package `parlouvain` (arXiv 1410.1237), used ONLY as a checker.
 *
 * TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and there only
 * as the oracle (never as the thing measured for the GPU product, never as a
 * fallback).  The product path lives in paper_1410_1237_b200/csrc/ and fails
 * loudly when its CUDA library is missing.
 *
 * Every function restates one reference function; citations are relative to
 * /root/reference/pkg/src/parlouvain/ (PL/).  numpy arithmetic the reference
 * relies on is restated explicitly (see SURVEY.md 8(a) "parity rules"):
 *   - ndarray.sum()            -> 0.0 + numpy pairwise tree   (orc_pairwise)
 *   - np.add.reduceat segment  -> w[s] + pairwise(w[s+1:e])    (reduceat_seg)
 *   - weighted np.bincount     -> sequential fold in input order
 *   - np.lexsort               -> stable sort (LSD radix here)
 * Parity is pinned against the compiled reference (oracle/_ref) by
 * tests/test_oracle_pins.py and the fixtures in tests/golden/.
 *
 * Built by oracle/Makefile with -O2 -ffp-contract=off (mirrors the reference
 * build flags, pkg/setup.py:32) so no FMA contraction changes rounding.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ---------------------------------------------------------------- numpy sums */

/* numpy pairwise_sum for float64 (leaves < 8 sequential, <= 128 eight-way
 * unrolled, otherwise split at n/2 rounded down to a multiple of 8). */
static double pairwise(const double *a, int64_t n)
{
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise(a, n2) + pairwise(a + n2, n - n2);
    }
}

/* ndarray.sum() of a contiguous float64 array. */
double orc_sum(const double *a, int64_t n) { return 0.0 + pairwise(a, n); }

/* np.add.reduceat value of one segment [s, e). */
static double reduceat_seg(const double *w, int64_t s, int64_t e)
{
    if (e - s <= 1) return w[s];
    return w[s] + pairwise(w + s + 1, e - s - 1);
}

/* ------------------------------------------------------- stable radix sort */

/* Stable LSD radix sort of `idx` by 64-bit `key[idx]` (only the low `bits`
 * bits are examined).  Equivalent to np.lexsort on the composite key. */
static void radix_sort_idx(const uint64_t *key, int64_t *idx, int64_t n, int bits)
{
    if (n <= 1) return;
    int64_t *tmp = (int64_t *)malloc(sizeof(int64_t) * n);
    uint64_t *k0 = (uint64_t *)malloc(sizeof(uint64_t) * n);
    uint64_t *k1 = (uint64_t *)malloc(sizeof(uint64_t) * n);
    for (int64_t i = 0; i < n; i++) k0[i] = key[idx[i]];
    int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * 65536);
    for (int shift = 0; shift < bits; shift += 16) {
        memset(cnt, 0, sizeof(int64_t) * 65536);
        for (int64_t i = 0; i < n; i++) cnt[(k0[i] >> shift) & 0xFFFF]++;
        int64_t run = 0;
        for (int d = 0; d < 65536; d++) { int64_t c = cnt[d]; cnt[d] = run; run += c; }
        for (int64_t i = 0; i < n; i++) {
            int64_t p = cnt[(k0[i] >> shift) & 0xFFFF]++;
            tmp[p] = idx[i];
            k1[p] = k0[i];
        }
        memcpy(idx, tmp, sizeof(int64_t) * n);
        uint64_t *t = k0; k0 = k1; k1 = t;
    }
    free(cnt); free(tmp); free(k0); free(k1);
}

static int bits_for(int64_t n)
{
    int b = 1;
    while (b < 63 && ((int64_t)1 << b) < n) b++;
    return b;
}

/* ------------------------------------------------------------ CSR building */

/*
 * Graph.from_edges (PL/graph.py:88-147) followed by Graph.__init__
 * (PL/graph.py:64-86).  Validation (weights finite > 0, ids in range) is done
 * by the Python caller exactly as the reference does before this point.
 *
 * Outputs: off[n+1]; nbr/wts sized >= 2R; selfw[n]; k[n];
 * info = {nnz, merged, num_edges, max_degree}; *m_out = total_weight.
 */
int orc_from_edges(const int64_t *u, const int64_t *v, const double *w, int64_t R,
                   int64_t n, int64_t *off, int64_t *nbr, double *wts, double *selfw,
                   double *k, int64_t *info, double *m_out)
{
    int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * (R ? R : 1));
    uint64_t *key = (uint64_t *)malloc(sizeof(uint64_t) * (R ? R : 1));
    int nb = bits_for(n);
    for (int64_t r = 0; r < R; r++) {
        int64_t a = u[r] < v[r] ? u[r] : v[r];
        int64_t b = u[r] < v[r] ? v[r] : u[r];
        key[r] = ((uint64_t)a << nb) | (uint64_t)b;   /* lexsort((b, a)) */
        idx[r] = r;
    }
    radix_sort_idx(key, idx, R, 2 * nb);
    /* merge runs of equal (a, b) with the reduceat rule (PL/graph.py:116-127) */
    int64_t *am = (int64_t *)malloc(sizeof(int64_t) * (R ? R : 1));
    int64_t *bm = (int64_t *)malloc(sizeof(int64_t) * (R ? R : 1));
    double *wm = (double *)malloc(sizeof(double) * (R ? R : 1));
    double *ws = (double *)malloc(sizeof(double) * (R ? R : 1));
    for (int64_t r = 0; r < R; r++) ws[r] = w[idx[r]];
    int64_t M = 0;
    int64_t s = 0;
    while (s < R) {
        int64_t e = s + 1;
        while (e < R && key[idx[e]] == key[idx[s]]) e++;
        int64_t a = u[idx[s]] < v[idx[s]] ? u[idx[s]] : v[idx[s]];
        int64_t b = u[idx[s]] < v[idx[s]] ? v[idx[s]] : u[idx[s]];
        am[M] = a; bm[M] = b; wm[M] = reduceat_seg(ws, s, e);
        M++;
        s = e;
    }
    int64_t merged = R - M;
    /* symmetrise + lexsort((dst, src)) (PL/graph.py:131-139): row i holds the
     * reversed records (a, i), a < i, ascending a, then the forward records
     * (i, b), b >= i, ascending b; merged records are unique, so this order is
     * the stable sort by (src, dst). */
    int64_t *nrev = (int64_t *)calloc(n + 1, sizeof(int64_t));
    int64_t *cnt = (int64_t *)calloc(n + 1, sizeof(int64_t));
    for (int64_t t = 0; t < M; t++) {
        cnt[am[t]]++;
        if (am[t] != bm[t]) { cnt[bm[t]]++; nrev[bm[t]]++; }
    }
    off[0] = 0;
    for (int64_t i = 0; i < n; i++) off[i + 1] = off[i] + cnt[i];
    int64_t *rcur = (int64_t *)calloc(n + 1, sizeof(int64_t));
    int64_t *fcur = (int64_t *)calloc(n + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) selfw[i] = 0.0;
    for (int64_t t = 0; t < M; t++) {
        int64_t a = am[t], b = bm[t];
        if (a != b) {
            int64_t p = off[b] + rcur[b]++;
            nbr[p] = a; wts[p] = wm[t];
        } else {
            selfw[a] = wm[t];
        }
        int64_t p = off[a] + nrev[a] + fcur[a]++;
        nbr[p] = b; wts[p] = wm[t];
    }
    int64_t nnz = off[n];
    /* Graph.__init__: k = bincount(row, weights) + selfw; m = k.sum() / 2 */
    int64_t num_self = 0, maxdeg = 0;
    for (int64_t i = 0; i < n; i++) {
        double acc = 0.0;
        for (int64_t e = off[i]; e < off[i + 1]; e++) acc += wts[e];
        k[i] = acc + selfw[i];
        if (selfw[i] != 0.0) num_self++;
        if (off[i + 1] - off[i] > maxdeg) maxdeg = off[i + 1] - off[i];
    }
    *m_out = orc_sum(k, n) / 2.0;
    info[0] = nnz;
    info[1] = merged;
    info[2] = (nnz + num_self) / 2;
    info[3] = maxdeg;
    free(idx); free(key); free(am); free(bm); free(wm); free(ws);
    free(nrev); free(cnt); free(rcur); free(fcur);
    return 0;
}

/* Graph.edge_records (PL/graph.py:169-174): a <= b half of the CSR, row-major.
 * Returns the record count. */
int64_t orc_edge_records(int64_t n, const int64_t *off, const int64_t *nbr, const double *wts,
                         int64_t *ra, int64_t *rb, double *rw)
{
    int64_t t = 0;
    for (int64_t i = 0; i < n; i++)
        for (int64_t e = off[i]; e < off[i + 1]; e++)
            if (nbr[e] >= i) { ra[t] = i; rb[t] = nbr[e]; rw[t] = wts[e]; t++; }
    return t;
}

/* --------------------------------------------------------- vertex following */

/*
 * vf_compact record emission (PL/heuristics.py:46-89).  Produces vertex_map[n]
 * and the compacted record list (kept records in edge_records order, then one
 * (t, t, w) self-loop record per folded vertex in ascending id); the caller
 * feeds the records to orc_from_edges.  rec_* must hold >= nnz + n entries.
 * info = {n_new, merged_count, num_records}.
 */
int orc_vf_records(int64_t n, const int64_t *off, const int64_t *nbr, const double *wts,
                   const double *selfw, int64_t *vertex_map, int64_t *rec_u, int64_t *rec_v,
                   double *rec_w, int64_t *info)
{
    uint8_t *cand = (uint8_t *)calloc(n + 1, 1);
    uint8_t *merged = (uint8_t *)calloc(n + 1, 1);
    int64_t *only = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
    int64_t *new_id = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
    for (int64_t i = 0; i < n; i++) {
        cand[i] = (off[i + 1] - off[i] == 1) && (selfw[i] == 0.0);
        only[i] = cand[i] ? nbr[off[i]] : -1;
    }
    for (int64_t i = 0; i < n; i++) {
        merged[i] = cand[i];
        /* isolated candidate pair: the lower id survives */
        if (cand[i] && cand[only[i]] && i < only[i]) merged[i] = 0;
    }
    int64_t run = 0, mcount = 0;
    for (int64_t i = 0; i < n; i++) {
        run += !merged[i];
        new_id[i] = run - 1;          /* np.cumsum(~merged) - 1 */
        mcount += merged[i];
    }
    for (int64_t i = 0; i < n; i++)
        vertex_map[i] = merged[i] ? new_id[only[i]] : new_id[i];
    int64_t t = 0;
    for (int64_t i = 0; i < n; i++)
        for (int64_t e = off[i]; e < off[i + 1]; e++) {
            int64_t j = nbr[e];
            if (j < i) continue;
            if (merged[i] || merged[j]) continue;
            rec_u[t] = new_id[i]; rec_v[t] = new_id[j]; rec_w[t] = wts[e]; t++;
        }
    for (int64_t i = 0; i < n; i++)
        if (merged[i]) {
            int64_t tg = new_id[only[i]];
            rec_u[t] = tg; rec_v[t] = tg; rec_w[t] = wts[off[i]]; t++;
        }
    info[0] = n - mcount;
    info[1] = mcount;
    info[2] = t;
    free(cand); free(merged); free(only); free(new_id);
    return 0;
}

/* ------------------------------------------------------------------ coloring */

/*
 * color_graph (PL/heuristics.py:92-118) with color_assign / color_conflicts
 * (PL/_kernels.pyx:148-195).  Returns the number of speculative rounds.
 */
int64_t orc_color(int64_t n, const int64_t *off, const int64_t *nbr, int64_t max_degree,
                  int64_t *colors)
{
    int64_t *active = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
    int64_t *tent = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
    uint8_t *keep = (uint8_t *)malloc(n + 1);
    int64_t scratch = max_degree + 2;
    int64_t *used = (int64_t *)calloc(scratch, sizeof(int64_t));
    int64_t stamp = 0;
    for (int64_t i = 0; i < n; i++) { colors[i] = -1; active[i] = i; }
    int64_t na = n, rounds = 0;
    while (na > 0) {
        rounds++;
        for (int64_t x = 0; x < na; x++) {
            int64_t i = active[x];
            stamp++;
            for (int64_t e = off[i]; e < off[i + 1]; e++) {
                int64_t j = nbr[e];
                if (j == i) continue;
                int64_t cj = colors[j];
                if (cj >= 0 && cj < scratch) used[cj] = stamp;
            }
            int64_t c = 0;
            while (used[c] == stamp) c++;
            tent[x] = c;
        }
        for (int64_t x = 0; x < na; x++) colors[active[x]] = tent[x];
        for (int64_t x = 0; x < na; x++) {
            int64_t i = active[x], ci = colors[i];
            keep[x] = 1;
            for (int64_t e = off[i]; e < off[i + 1]; e++) {
                int64_t j = nbr[e];
                if (j != i && j < i && colors[j] == ci) { keep[x] = 0; break; }
            }
        }
        int64_t nr = 0;
        for (int64_t x = 0; x < na; x++)
            if (!keep[x]) active[nr++] = active[x];   /* order preserved */
        for (int64_t x = 0; x < nr; x++) colors[active[x]] = -1;
        na = nr;
    }
    free(active); free(tent); free(keep); free(used);
    return rounds;
}

/* --------------------------------------------------------------- local move */

/*
 * run_iteration (PL/engine.py:140-163): decide_moves (PL/_kernels.pyx:21-101)
 * against the state at entry, then apply_moves (PL/_kernels.pyx:104-145)
 * sequentially in subset order with the live assignment.  Decide only reads
 * the state and finishes before apply starts, so the entry state *is* the
 * snapshot and no copies are needed.  labels may be NULL (labels[c] == c).
 * out_targets/out_moved (optional, may be NULL) receive the decide outputs.
 * Returns the move count.
 */
/* decide_moves alone (PL/_kernels.pyx:21-101): targets / moved per subset index. */
void orc_decide(int64_t n, const int64_t *off, const int64_t *nbr, const double *wts,
                const double *kdeg, double m, const int64_t *labels, const int64_t *subset,
                int64_t ns, const int64_t *assign, const double *a_tot, const int64_t *sizes,
                int64_t *tg, uint8_t *mv)
{
    /* per-community scratch is kept across calls (colour stages call this
     * hundreds of times per iteration); stamps grow monotonically so the
     * table never needs clearing. */
    static double *val = NULL;
    static int64_t *stampv = NULL, *cands = NULL, cap = 0, stamp_base = 0;
    if (n + 1 > cap) {
        free(val); free(stampv); free(cands);
        cap = n + 1;
        val = (double *)malloc(sizeof(double) * cap);
        stampv = (int64_t *)calloc(cap, sizeof(int64_t));
        cands = (int64_t *)malloc(sizeof(int64_t) * cap);
        stamp_base = 0;
    }
    const double four_m_sq = (2.0 * m) * (2.0 * m);
#define LBL(c) (labels ? labels[c] : (c))
    for (int64_t x = 0; x < ns; x++) {
        int64_t i = subset[x];
        int64_t stamp = ++stamp_base;
        int64_t c_old = assign[i];
        int64_t ncand = 0;
        for (int64_t e = off[i]; e < off[i + 1]; e++) {
            int64_t j = nbr[e];
            if (j == i) continue;
            int64_t c = assign[j];
            if (stampv[c] == stamp) {
                val[c] += wts[e];
            } else {
                stampv[c] = stamp;
                val[c] = 0.0 + wts[e];   /* e_to.get(c, 0.0) + w */
                cands[ncand++] = c;
            }
        }
        double ki = kdeg[i];
        double e_old = stampv[c_old] == stamp ? val[c_old] : 0.0;
        double a_old_excl = a_tot[c_old] - ki;
        double best_gain = 0.0;
        int64_t best_c = c_old, best_label = LBL(c_old);
        for (int64_t t = 0; t < ncand; t++) {
            int64_t c = cands[t];
            if (c == c_old) continue;
            double gain = (val[c] - e_old) / m
                          + (2.0 * ki * a_old_excl - 2.0 * ki * a_tot[c]) / four_m_sq;
            if (gain > best_gain || (gain == best_gain && LBL(c) < best_label)) {
                best_gain = gain; best_c = c; best_label = LBL(c);
            }
        }
        int moved = best_gain > 0.0 && best_c != c_old;
        if (moved && sizes[c_old] == 1 && sizes[best_c] == 1 && LBL(best_c) > LBL(c_old))
            moved = 0;   /* singleton-pair guard */
        tg[x] = moved ? best_c : c_old;
        mv[x] = (uint8_t)moved;
    }
#undef LBL
}

/* apply_moves alone (PL/_kernels.pyx:104-145): sequential in subset order
 * against the live assignment; returns the move count. */
int64_t orc_apply(const int64_t *off, const int64_t *nbr, const double *wts, const double *kdeg,
                  const double *selfw, const int64_t *subset, int64_t ns, const int64_t *tg,
                  const uint8_t *mv, int64_t *assign, double *a_tot, double *w_int,
                  int64_t *sizes)
{
    int64_t count = 0;
    for (int64_t x = 0; x < ns; x++) {
        if (!mv[x]) continue;
        int64_t i = subset[x], b = tg[x], a = assign[i];
        if (b == a) continue;
        double e_a = 0.0, e_b = 0.0;
        for (int64_t e = off[i]; e < off[i + 1]; e++) {
            int64_t j = nbr[e];
            if (j == i) continue;
            int64_t c = assign[j];
            if (c == a) e_a += wts[e];
            else if (c == b) e_b += wts[e];
        }
        double sw = selfw[i], ki = kdeg[i];
        w_int[a] -= 2.0 * e_a + 2.0 * sw;
        w_int[b] += 2.0 * e_b + 2.0 * sw;
        a_tot[a] -= ki;
        a_tot[b] += ki;
        sizes[a] -= 1;
        sizes[b] += 1;
        assign[i] = b;
        count++;
    }
    return count;
}

int64_t orc_run_iteration(int64_t n, const int64_t *off, const int64_t *nbr, const double *wts,
                          const double *kdeg, const double *selfw, double m,
                          const int64_t *labels, const int64_t *subset, int64_t ns,
                          int64_t *assign, double *a_tot, double *w_int, int64_t *sizes,
                          int64_t *out_targets, uint8_t *out_moved)
{
    int64_t *tg = (int64_t *)malloc(sizeof(int64_t) * (ns + 1));
    uint8_t *mv = (uint8_t *)malloc(ns + 1);
    orc_decide(n, off, nbr, wts, kdeg, m, labels, subset, ns, assign, a_tot, sizes, tg, mv);
    if (out_targets) memcpy(out_targets, tg, sizeof(int64_t) * ns);
    if (out_moved) memcpy(out_moved, mv, ns);
    int64_t count = orc_apply(off, nbr, wts, kdeg, selfw, subset, ns, tg, mv, assign, a_tot,
                              w_int, sizes);
    free(tg); free(mv);
    return count;
}

/* modularity (PL/modularity.py:59-64). */
double orc_modularity(int64_t n, const double *w_int, const double *a_tot, double m)
{
    double two_m = 2.0 * m;
    double *sq = (double *)malloc(sizeof(double) * (n + 1));
    for (int64_t i = 0; i < n; i++) { double x = a_tot[i] / two_m; sq[i] = x * x; }
    double q = orc_sum(w_int, n) / two_m - orc_sum(sq, n);
    free(sq);
    return q;
}

/* ------------------------------------------------------------------- rebuild */

/*
 * rebuild record stage (PL/engine.py:229-253): renumber = rank of the
 * community among np.unique(assignment); records (lo, hi, w) from
 * edge_records, stable-sorted by (lo, hi), runs merged with the reduceat rule.
 * The caller feeds (lo, hi, w) to orc_from_edges.  Outputs renumber[n]
 * (-1 for empty ids), lo/hi/w sized >= nnz; info = {n_new, num_records}.
 */
int orc_rebuild_records(int64_t n, const int64_t *off, const int64_t *nbr, const double *wts,
                        const int64_t *assign, int64_t *renumber, int64_t *lo, int64_t *hi,
                        double *w, int64_t *info)
{
    uint8_t *present = (uint8_t *)calloc(n + 1, 1);
    for (int64_t i = 0; i < n; i++) present[assign[i]] = 1;
    int64_t nc = 0;
    for (int64_t c = 0; c < n; c++) renumber[c] = present[c] ? nc++ : -1;
    int64_t R;
    int64_t cap = off[n];
    int64_t *ra = (int64_t *)malloc(sizeof(int64_t) * (cap + 1));
    int64_t *rb = (int64_t *)malloc(sizeof(int64_t) * (cap + 1));
    double *rw = (double *)malloc(sizeof(double) * (cap + 1));
    R = orc_edge_records(n, off, nbr, wts, ra, rb, rw);
    uint64_t *key = (uint64_t *)malloc(sizeof(uint64_t) * (R + 1));
    int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * (R + 1));
    int nb = bits_for(nc);
    for (int64_t t = 0; t < R; t++) {
        int64_t ca = renumber[assign[ra[t]]], cb = renumber[assign[rb[t]]];
        int64_t l = ca < cb ? ca : cb, h = ca < cb ? cb : ca;
        ra[t] = l; rb[t] = h;
        key[t] = ((uint64_t)l << nb) | (uint64_t)h;
        idx[t] = t;
    }
    radix_sort_idx(key, idx, R, 2 * nb);
    double *ws = (double *)malloc(sizeof(double) * (R + 1));
    for (int64_t t = 0; t < R; t++) ws[t] = rw[idx[t]];
    int64_t M = 0, s = 0;
    while (s < R) {
        int64_t e = s + 1;
        while (e < R && key[idx[e]] == key[idx[s]]) e++;
        lo[M] = ra[idx[s]]; hi[M] = rb[idx[s]]; w[M] = reduceat_seg(ws, s, e);
        M++;
        s = e;
    }
    info[0] = nc;
    info[1] = M;
    free(present); free(ra); free(rb); free(rw); free(key); free(idx); free(ws);
    return 0;
}
