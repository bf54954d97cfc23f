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
 *      SPEC.md L216-L224).  The paper never defines I beyond "currency exchange rates and
 *      terms", so WHICH terms I holds is a reading (SPEC's); the oracle's implementation of
 *      that reading is pinned by tests independent of this file: SPEC's hand-derived
 *      examples, the exhaustive excess-of-loss interval characterisation |[0,x] n [R,R+L]|
 *      in exact rationals, the stop-loss / per-occurrence-XL special cases and the
 *      separate-rounding (no FMA) check.
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

#define REAL double
#define SFX(name) name
#include "alg1.inc"
#undef REAL
#undef SFX

#define REAL float
#define SFX(name) name##_f32
#include "alg1.inc"
#undef REAL
#undef SFX

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

int oracle_run_analysis_f32(uint32_t catalogue_size, uint32_t n_elts, const uint64_t *rec_offsets,
                            const uint32_t *rec_event_ids, const double *rec_losses,
                            const double *fin, uint32_t n_layers, const double *layer_terms,
                            const uint32_t *elt_offsets, const uint32_t *elt_index,
                            uint64_t n_trials, const uint64_t *trial_offsets,
                            const uint32_t *events, uint64_t n_sel, const uint64_t *selection,
                            double *ylt, double *max_occ, double *inc, int n_threads)
{
    return oracle_run_analysis_ex_f32(catalogue_size, n_elts, rec_offsets, rec_event_ids,
                                      rec_losses, fin, n_layers, layer_terms, elt_offsets,
                                      elt_index, n_trials, trial_offsets, events, n_sel,
                                      selection, ylt, max_occ, inc, n_threads);
}

/* ------------------------------------------------------------------------- */
/* Metrics (reading R11)                                   */
/* Portfolio-scope trial losses ("portfolio = per-trial sum over layers";
 * SURVEY 8(f) F1, reading G10): out[t] = ((0 + ylt[0][t]) + ylt[1][t]) + ... + ylt[L-1][t],
 * left to right in layer order.  ylt is layer-major with row stride ld. */
void oracle_portfolio_row(const double *ylt, uint32_t n_layers, uint64_t n, uint64_t ld,
                          double *out)
{
    for (uint64_t t = 0; t < n; ++t) {
        double s = 0.0;
        for (uint32_t l = 0; l < n_layers; ++l) s = s + ylt[(size_t)l * ld + t];
        out[t] = s;
    }
}

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

/* Exceedance-probability curve of a YLT-like row ("financial
 * functions or filters are then applied on the aggregate loss values"; reading R15 of DESIGN.md):
 * the row sorted from the largest value down, out[i] = the (i+1)-th largest, whose empirical
 * exceedance probability is (i+1)/n (return period n/(i+1) years).  From a YLT row it is the AEP
 * curve, from the per-trial maximum occurrence losses (R13) the OEP curve.  The nearest-rank PML
 * of R11 is a point on it: PML(p) = out[n - ceil(p n)].  Returns 0, -1 if n == 0, -3 out of
 * memory. */
static int o_cmp_desc(const void *a, const void *b) { return o_cmp(b, a); }

int oracle_ep_curve(const double *row, uint64_t n, double *out)
{
    if (n == 0) return -1;
    memcpy(out, row, n * sizeof(double));
    qsort(out, n, sizeof(double), o_cmp_desc);
    return 0;
}
