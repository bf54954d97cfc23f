/*
 * oracle/oracle.c -- plain, slow, obviously-correct CPU oracle for the aggregate
 * risk analysis of arXiv 1308.2572 ("Achieving Speedup in Aggregate Risk Analysis
 * using Multiple GPUs"), Algorithm 1 (Sec. II).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_1308_2572_b200/,
 * include/) may include, link or call this file.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs use it.  It shares no code,
 * header, table or constant with the CUDA path.
 *
 * Arithmetic: IEEE fp64, round-to-nearest-even, NO contraction (built with
 * -O2 -ffp-contract=off; every product and difference is rounded separately).
 * min(x, y) is written  (y < x ? y : x)  and max(x, 0) is written  (x < 0 ? 0 : x).
 *
 * Readings of the paper where it is silent / garbled (DESIGN.md "Readings" R1-R12):
 *   R1 ApplyFinancialTerms(I) = min(max(x*rate - retention, 0), limit)   (
 *      SPEC.md L216-L224).  PARITY UNPINNED against the paper itself: the paper never
 *      defines I beyond "currency exchange rates and terms"; pinned only by SPEC's
 *      hand-derived examples and by the XL-layer interval characterisation in tests.
 *   R2 line 6: x_d = loss of occurrence d's event in ELT c, 0 if absent.
 *   R3 lo/l are indexed by occurrence position d (repeated events charged per occurrence).
 *   R4 lo = 0 and lr = 0 per (layer, trial); YLT[a][t] = lr after line 29.
 *   R5 lines 19 and 25 have simultaneous ("forall") semantics: they read the OLD values;
 *      lo_{x_0} = 0 for line 25.
 *   R6 an absent limit is +infinity.
 *   R7 sums are left-to-right: over ELTs in the layer's listed order (lines 11-13), over
 *      events in trial order (line 19, line 28).
 *   F4 outputs: max_occ[l][t] = max over the trial's events of lo_d after line 16 (the
 *      per-trial maximum occurrence loss, whose distribution is the OEP curve; 0 for an empty
 *      trial); inc[l][pos] = the per-event incremental aggregate loss of lines 24-26 at the
 *      event's position in the YET (the back-allocation of lr to events).
 *   R11 PML(p) = nearest-rank v[ceil(p*n) - 1] of the ascending YLT row; TVaR(p) = mean of
 *      all v >= PML(p).  The paper only names the metrics.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* Elementary operations                                                      */
/* ------------------------------------------------------------------------- */

static double o_min(double x, double y) { return (y < x) ? y : x; }
static double o_max0(double x) { return (x < 0.0) ? 0.0 : x; }

/* Alg. 1 line 9, reading R1: l = min(max(x*rate - retention, 0), limit). */
double oracle_apply_financial_terms(double x, double rate, double retention, double limit)
{
    double scaled = x * rate;          /* rounded product */
    double net = scaled - retention;   /* rounded difference (no FMA) */
    return o_min(o_max0(net), limit);
}

/* Alg. 1 line 16: lo = min(max(lo - T_OccR, 0), T_OccL). */
double oracle_apply_occurrence_terms(double lo, double occ_retention, double occ_limit)
{
    double net = lo - occ_retention;
    return o_min(o_max0(net), occ_limit);
}

/* Alg. 1 lines 18-26 on one trial's occurrence-capped losses lo[0..k):
 *   line 19 (simultaneous): cum[d] = sum_{i<=d} lo[i]   (left-to-right running sum)
 *   line 22:                cum[d] = min(max(cum[d] - T_AggR, 0), T_AggL)
 *   line 25 (simultaneous): inc[d] = cum[d] - cum[d-1], cum[-1] = 0
 * Writes inc[0..k).  cum is caller-provided scratch of length k. */
void oracle_apply_aggregate_terms(const double *lo, uint64_t k, double agg_retention,
                                  double agg_limit, double *cum, double *inc)
{
    double s = 0.0;
    for (uint64_t d = 0; d < k; ++d) { /* line 18-20 */
        s = s + lo[d];
        cum[d] = s;
    }
    for (uint64_t d = 0; d < k; ++d) /* line 21-23 */
        cum[d] = o_min(o_max0(cum[d] - agg_retention), agg_limit);
    for (uint64_t d = 0; d < k; ++d) /* line 24-26, reading the un-overwritten cum[d-1] */
        inc[d] = cum[d] - (d == 0 ? 0.0 : cum[d - 1]);
}

/* ------------------------------------------------------------------------- */
/* Direct access tables (PAPER: one dense slot per catalogue event)       */
/* ------------------------------------------------------------------------- */

/* dat[0..C] := 0; dat[e] := loss of e.  Returns 0, or 1 + index of the first record whose
 * event id is 0 or exceeds the catalogue. */
int64_t oracle_build_dat(uint32_t catalogue_size, uint64_t n_records, const uint32_t *event_ids,
                         const double *losses, double *dat)
{
    for (uint64_t e = 0; e <= catalogue_size; ++e) dat[e] = 0.0;
    for (uint64_t r = 0; r < n_records; ++r) {
        uint32_t e = event_ids[r];
        if (e == 0 || e > catalogue_size) return (int64_t)r + 1;
        dat[e] = losses[r];
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* One (layer, trial): Algorithm 1 lines 4-29 in the paper's order             */
/* ------------------------------------------------------------------------- */

typedef struct {
    uint32_t n_elts;          /* |E| of the layer */
    const double *const *dat; /* [n_elts] direct access tables, layer order */
    const double *rate, *retention, *limit; /* [n_elts] financial terms I, layer order */
    double occ_retention, occ_limit, agg_retention, agg_limit; /* layer terms T */
} o_layer;

typedef struct {
    double *x, *l, *lo, *cum, *inc; /* workspaces of length >= k (Alg. 1 symbols) */
    uint64_t cap;
} o_work;

static int o_work_reserve(o_work *w, uint64_t k)
{
    if (k <= w->cap) return 0;
    double **bufs[5] = {&w->x, &w->l, &w->lo, &w->cum, &w->inc};
    for (int i = 0; i < 5; ++i) {
        free(*bufs[i]);
        *bufs[i] = (double *)malloc((k ? k : 1) * sizeof(double));
        if (!*bufs[i]) return -1;
    }
    w->cap = k;
    return 0;
}

static void o_work_free(o_work *w)
{
    free(w->x); free(w->l); free(w->lo); free(w->cum); free(w->inc);
    memset(w, 0, sizeof(*w));
}

/* Returns lr; *max_occ = max_d lo_d after line 16 (0 for an empty trial); the per-event
 * increments of lines 24-26 are left in w->inc[0..k). */
static double o_run_trial(const o_layer *a, const uint32_t *events, uint64_t k, o_work *w,
                          double *max_occ)
{
    for (uint64_t d = 0; d < k; ++d) w->lo[d] = 0.0;               /* R4 */
    for (uint32_t c = 0; c < a->n_elts; ++c) {                      /* line 4 */
        const double *dat = a->dat[c];
        for (uint64_t d = 0; d < k; ++d) w->x[d] = dat[events[d]];  /* lines 5-7 */
        for (uint64_t d = 0; d < k; ++d)                            /* lines 8-10 */
            w->l[d] = oracle_apply_financial_terms(w->x[d], a->rate[c], a->retention[c],
                                                   a->limit[c]);
        for (uint64_t d = 0; d < k; ++d) w->lo[d] = w->lo[d] + w->l[d]; /* lines 11-13 */
    }
    for (uint64_t d = 0; d < k; ++d)                                /* lines 15-17 */
        w->lo[d] = oracle_apply_occurrence_terms(w->lo[d], a->occ_retention, a->occ_limit);
    double m = 0.0;                                                 /* F4: OEP basis */
    for (uint64_t d = 0; d < k; ++d) m = (m < w->lo[d]) ? w->lo[d] : m;
    *max_occ = m;
    oracle_apply_aggregate_terms(w->lo, k, a->agg_retention, a->agg_limit, w->cum,
                                 w->inc);                           /* lines 18-26 */
    double lr = 0.0;                                                /* R4 */
    for (uint64_t d = 0; d < k; ++d) lr = lr + w->inc[d];           /* lines 27-29 */
    return lr;
}

/* ------------------------------------------------------------------------- */
/* Whole analysis: lines 2-3 over layers x trials, trial-parallel threads      */
/* ------------------------------------------------------------------------- */

typedef struct {
    const o_layer *layers;
    uint32_t n_layers;
    const uint64_t *trial_offsets;
    const uint32_t *events;
    uint64_t n_trials;          /* YLT row length */
    const uint64_t *selection;  /* NULL: trials [t0, t1); else selected trial indices */
    uint64_t t0, t1;            /* range of trials (or of selection entries) */
    double *ylt;                /* [n_layers][n_out] */
    double *max_occ;            /* NULL or [n_layers][n_out] */
    double *inc;                /* NULL or [n_layers][n_events] (positions of the whole YET) */
    uint64_t n_events;
    uint64_t n_out;
    int status;
} o_job;

static void *o_job_run(void *arg)
{
    o_job *j = (o_job *)arg;
    o_work w;
    memset(&w, 0, sizeof(w));
    for (uint64_t i = j->t0; i < j->t1; ++i) {
        uint64_t t = j->selection ? j->selection[i] : i;
        const uint32_t *ev = j->events + (j->trial_offsets[t] - j->trial_offsets[0]);
        uint64_t k = j->trial_offsets[t + 1] - j->trial_offsets[t];
        if (o_work_reserve(&w, k)) { j->status = -1; break; }
        for (uint32_t a = 0; a < j->n_layers; ++a) {
            double m;
            j->ylt[(uint64_t)a * j->n_out + i] = o_run_trial(&j->layers[a], ev, k, &w, &m);
            if (j->max_occ) j->max_occ[(uint64_t)a * j->n_out + i] = m;
            if (j->inc) {
                double *dst = j->inc + (uint64_t)a * j->n_events +
                              (j->trial_offsets[t] - j->trial_offsets[0]);
                for (uint64_t d = 0; d < k; ++d) dst[d] = w.inc[d];
            }
        }
    }
    o_work_free(&w);
    return NULL;
}

/*
 * Full oracle analysis.
 *   ELTs as CSR: rec_offsets[n_elts+1], rec_event_ids[], rec_losses[];
 *   financial terms fin[n_elts*3] = (rate, retention, limit) per ELT (limit may be +inf);
 *   layers: layer_terms[n_layers*4] = (OccR, OccL, AggR, AggL); CSR elt_offsets[n_layers+1],
 *   elt_index[] (order = the layer's ELT order = the summation order of lines 11-13);
 *   YET as CSR: trial_offsets[n_trials+1] (may start at a non-zero base), events[];
 *   selection: NULL for all trials, or n_sel trial indices (YLT columns follow selection);
 *   ylt[n_layers * n_out] with n_out = selection ? n_sel : n_trials.
 * Returns 0; -1 out of memory; -(2+r) if record r has an invalid event id; -3 for a
 * trial event outside [1, C].
 */
int oracle_run_analysis_ex(uint32_t catalogue_size, uint32_t n_elts,
                           const uint64_t *rec_offsets, const uint32_t *rec_event_ids,
                           const double *rec_losses, const double *fin, uint32_t n_layers,
                           const double *layer_terms, const uint32_t *elt_offsets,
                           const uint32_t *elt_index, uint64_t n_trials,
                           const uint64_t *trial_offsets, const uint32_t *events, uint64_t n_sel,
                           const uint64_t *selection, double *ylt, double *max_occ,
                           double *inc, int n_threads)
{
    int status = 0;
    uint64_t n_ev = trial_offsets[n_trials] - trial_offsets[0];
    for (uint64_t i = 0; i < n_ev; ++i)
        if (events[i] == 0 || events[i] > catalogue_size) return -3;

    double **dats = (double **)calloc(n_elts ? n_elts : 1, sizeof(double *));
    o_layer *layers = (o_layer *)calloc(n_layers ? n_layers : 1, sizeof(o_layer));
    const double **dat_refs = (const double **)calloc(elt_offsets[n_layers] + 1,
                                                      sizeof(double *));
    double *terms3 = (double *)calloc(3 * (size_t)elt_offsets[n_layers] + 1, sizeof(double));
    if (!dats || !layers || !dat_refs || !terms3) { status = -1; goto done; }

    for (uint32_t j = 0; j < n_elts; ++j) { /* preprocessing stage */
        dats[j] = (double *)malloc(((size_t)catalogue_size + 1) * sizeof(double));
        if (!dats[j]) { status = -1; goto done; }
        int64_t bad = oracle_build_dat(catalogue_size, rec_offsets[j + 1] - rec_offsets[j],
                                       rec_event_ids + rec_offsets[j],
                                       rec_losses + rec_offsets[j], dats[j]);
        if (bad) { status = -(int)(2 + rec_offsets[j] + (uint64_t)bad - 1); goto done; }
    }
    uint32_t m = elt_offsets[n_layers];
    double *rate = terms3, *ret = terms3 + m, *lim = terms3 + 2 * (size_t)m;
    for (uint32_t a = 0; a < n_layers; ++a) {
        o_layer *L = &layers[a];
        L->n_elts = elt_offsets[a + 1] - elt_offsets[a];
        for (uint32_t c = elt_offsets[a]; c < elt_offsets[a + 1]; ++c) {
            uint32_t j = elt_index[c];
            dat_refs[c] = dats[j];
            rate[c] = fin[3 * (size_t)j + 0];
            ret[c] = fin[3 * (size_t)j + 1];
            lim[c] = fin[3 * (size_t)j + 2];
        }
        L->dat = dat_refs + elt_offsets[a];
        L->rate = rate + elt_offsets[a];
        L->retention = ret + elt_offsets[a];
        L->limit = lim + elt_offsets[a];
        L->occ_retention = layer_terms[4 * (size_t)a + 0];
        L->occ_limit = layer_terms[4 * (size_t)a + 1];
        L->agg_retention = layer_terms[4 * (size_t)a + 2];
        L->agg_limit = layer_terms[4 * (size_t)a + 3];
    }

    uint64_t n_out = selection ? n_sel : n_trials;
    if (n_threads < 1) n_threads = 1;
    if ((uint64_t)n_threads > n_out) n_threads = n_out ? (int)n_out : 1;
    o_job *jobs = (o_job *)calloc((size_t)n_threads, sizeof(o_job));
    pthread_t *th = (pthread_t *)calloc((size_t)n_threads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); status = -1; goto done; }
    for (int i = 0; i < n_threads; ++i) { /* contiguous ranges: per-trial order unchanged */
        o_job *j = &jobs[i];
        j->layers = layers; j->n_layers = n_layers;
        j->trial_offsets = trial_offsets; j->events = events; j->n_trials = n_trials;
        j->selection = selection; j->ylt = ylt; j->n_out = n_out;
        j->max_occ = max_occ; j->inc = inc; j->n_events = n_ev;
        j->t0 = n_out * (uint64_t)i / (uint64_t)n_threads;
        j->t1 = n_out * (uint64_t)(i + 1) / (uint64_t)n_threads;
    }
    for (int i = 1; i < n_threads; ++i) pthread_create(&th[i], NULL, o_job_run, &jobs[i]);
    o_job_run(&jobs[0]);
    for (int i = 1; i < n_threads; ++i) pthread_join(th[i], NULL);
    for (int i = 0; i < n_threads; ++i) if (jobs[i].status) status = jobs[i].status;
    free(jobs); free(th);

done:
    if (dats) for (uint32_t j = 0; j < n_elts; ++j) free(dats[j]);
    free(dats); free(layers); free(dat_refs); free(terms3);
    return status;
}

int oracle_run_analysis(uint32_t catalogue_size, uint32_t n_elts, const uint64_t *rec_offsets,
                        const uint32_t *rec_event_ids, const double *rec_losses,
                        const double *fin, uint32_t n_layers, const double *layer_terms,
                        const uint32_t *elt_offsets, const uint32_t *elt_index,
                        uint64_t n_trials, const uint64_t *trial_offsets,
                        const uint32_t *events, uint64_t n_sel, const uint64_t *selection,
                        double *ylt, int n_threads)
{
    return oracle_run_analysis_ex(catalogue_size, n_elts, rec_offsets, rec_event_ids, rec_losses,
                                  fin, n_layers, layer_terms, elt_offsets, elt_index, n_trials,
                                  trial_offsets, events, n_sel, selection, ylt, NULL, NULL,
                                  n_threads);
}

/* ------------------------------------------------------------------------- */
/* Metrics (reading R11)                                   */
/* ------------------------------------------------------------------------- */

static int o_cmp(const void *a, const void *b)
{
    double x = *(const double *)a, y = *(const double *)b;
    return (x < y) ? -1 : (y < x) ? 1 : 0;
}

/* PML and TVaR of one YLT row at probabilities p[0..n_p).  Returns 0, -1 if n == 0,
 * -2 if some p is outside (0, 1), -3 out of memory. */
int oracle_metrics(const double *ylt_row, uint64_t n, uint32_t n_p, const double *p,
                   double *pml_out, double *tvar_out)
{
    if (n == 0) return -1;
    for (uint32_t i = 0; i < n_p; ++i) if (!(p[i] > 0.0 && p[i] < 1.0)) return -2;
    double *v = (double *)malloc(n * sizeof(double));
    if (!v) return -3;
    memcpy(v, ylt_row, n * sizeof(double));
    qsort(v, n, sizeof(double), o_cmp);                     /* ascending */
    for (uint32_t i = 0; i < n_p; ++i) {
        uint64_t r = (uint64_t)ceil(p[i] * (double)n);      /* nearest rank, 1-based */
        if (r < 1) r = 1;
        if (r > n) r = n;
        double q = v[r - 1];
        uint64_t i0 = r - 1;                                /* lower_bound(v, q) */
        while (i0 > 0 && !(v[i0 - 1] < q)) --i0;
        double s = 0.0;
        for (uint64_t t = i0; t < n; ++t) s = s + v[t];     /* left-to-right tail sum */
        pml_out[i] = q;
        tvar_out[i] = s / (double)(n - i0);
    }
    free(v);
    return 0;
}
