/*
 * ara.h -- C ABI of the B200-native aggregate risk analysis library (libara.so).
 *
 * The calls follow the paper's statement of the problem (arXiv 1308.2572, Sec. II):
 *   inputs  : a Year Event Table (YET) of trials, Event Loss Tables (ELTs)
 *             with per-ELT financial terms I (L49-L53), Layers = a set of ELTs plus layer terms
 *             T = (OccR, OccL, AggR, AggL) (L55-L59);
 *   method  : Algorithm 1 (L63-L112) -- per layer, per trial, per event: look up the event's
 *             loss in every ELT of the layer (lines 4-7), apply financial terms (lines 8-10),
 *             sum over ELTs (lines 11-13), apply occurrence terms (lines 15-17), take the running
 *             sum over the trial's events (lines 18-20), apply aggregate terms (lines 21-23),
 *             difference (lines 24-26) and sum (lines 27-29) into the trial loss lr;
 *   outputs : the Year Loss Table (YLT) and, from a YLT, PML and TVaR (L32).
 *
 * Exact semantics (DESIGN.md "Readings" R1-R12; SPEC.md engine/metrics):
 *   F_j(x)  = min(max(x * rate_j - retention_j, 0), limit_j)      (R1; * and - rounded apart)
 *   lo_d    = ((0 + F_0(x_d0)) + F_1(x_d1)) + ... in the layer's ELT order (R7)
 *   oc_d    = min(max(lo_d - OccR, 0), OccL)
 *   S_d     = S_{d-1} + oc_d, S_0 = +0, in trial order (R5, R7)
 *   C_d     = min(max(S_d - AggR, 0), AggL), C_0 = 0
 *   lr      = (((0 + (C_1 - C_0)) + (C_2 - C_1)) + ...)            (R4, R5)
 *   min(x,y) = (y < x ? y : x), max(x,0) = (x < 0 ? 0 : x); fp64, round-to-nearest-even, no FMA.
 * The library reproduces these operations in this order, so its YLT is bit-identical to a
 * sequential fp64 evaluation of Algorithm 1 (up to the sign of zero).
 *
 * Conventions
 *   - Every call returns ara_status; no C++ exception crosses the ABI.  On failure nothing is
 *     written to caller outputs and ara_last_error(ctx) names the offending item.
 *   - Host arrays (h_ / unprefixed pointers in load/set calls) are caller-owned and read only
 *     during the call.  Device arrays (d_) are caller-owned device memory of the context's
 *     device; the library never frees or retains them beyond the call (or, for asynchronous
 *     calls, beyond the stream-ordered completion of the enqueued work).
 *   - The context owns every buffer it allocates (the device ELT store, staging buffers).
 *   - Order: ara_create -> ara_load_elts -> ara_set_layers -> ara_run / ara_metrics.
 *     ara_load_elts invalidates the layers (ARA_ERR_STATE until ara_set_layers is called).
 *   - A context is not thread-safe; callers serialise calls on one context.
 *     Distinct contexts may be used from distinct threads.
 *   - Absent limits are +INFINITY.  Retentions and limits may not be NaN or negative.
 */
#ifndef ARA_H
#define ARA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ara_ctx ara_ctx; /* opaque */

typedef enum {
    ARA_OK = 0,
    ARA_ERR_ARG = 1,        /* NULL pointer, zero size where one is required, unknown flag   */
    ARA_ERR_RANGE = 2,      /* event id 0 or > catalogue_size            */
    ARA_ERR_VALIDATION = 3, /* bad terms, duplicate ids, non-monotone offsets, empty layer   */
    ARA_ERR_STATE = 4,      /* call out of order (e.g. ara_run before ara_set_layers)        */
    ARA_ERR_EMPTY = 5,      /* metrics over zero trials                       */
    ARA_ERR_OOM = 6,        /* host or device allocation failed                              */
    ARA_ERR_CUDA = 7,       /* CUDA runtime error (message in ara_last_error)                */
    ARA_ERR_UNSUPPORTED = 8 /* a limit of this build (e.g. more than ARA_MAX_ELTS_PER_LAYER) */
} ara_status;

/* Financial terms I of one ELT (reading R1):
 * rate > 0 finite (currency exchange rate), retention >= 0 finite, limit >= 0 or +INFINITY. */
typedef struct {
    double rate, retention, limit;
} ara_fin_terms;

/* Layer terms T: retentions >= 0 finite, limits >= 0 or +INF. */
typedef struct {
    double occ_retention, occ_limit, agg_retention, agg_limit;
} ara_layer_terms;

/* Limits of this build. */
#define ARA_MAX_ELTS_PER_LAYER 64 /* "approximately 3 to 30" ELTs per layer  */
#define ARA_MAX_P 32              /* probabilities per ara_metrics call                     */

/* ara_run flags */
#define ARA_RUN_SYNC 1u     /* wait for completion and report device-side errors           */
#define ARA_RUN_VALIDATE 2u /* check offsets and event ids on the device BEFORE the scan
                               (one extra YET read); implies ARA_RUN_SYNC; on error nothing
                               is written to the YLT                                        */
#define ARA_RUN_BALANCE 4u  /* length-bucketed scheduling for variable-length trials
                               (800-1500 events): the trials are sorted by
                               length on the device and handed out in warp-sized batches, so
                               the thread groups of a warp run trials of nearly equal length.
                               This is the default schedule; the flag is accepted for clarity.
                               When the previous run on this context found all trials equally
                               long, the sort is replaced by the identity order.  Results are
                               identical under any schedule.                                 */
#define ARA_RUN_HOIST 8u    /* hoisted scan (deferred exact lever): Alg. 1
                               lines 4-17 depend only on (event, layer), so each run first
                               evaluates them once per distinct event of the layers' union
                               (same fp ops, same order) into a per-event table, then scans
                               the trials reading one value per (occurrence, layer) for lines
                               18-29.  The YLT is bit-identical to the full scan.  Up to 8
                               layers (else ARA_ERR_UNSUPPORTED); ignored by ara_run_outputs
                               when per-event outputs are requested.  Reported separately
                               from the full per-occurrence scan (bench.py --hoist).          */

/* Human-readable name of a status code (static storage). */
const char *ara_status_string(ara_status s);

/* Create a context on CUDA device `cuda_device`.  `cuda_stream` is a cudaStream_t (or NULL for
 * the legacy default stream) on which every asynchronous operation of the context is ordered;
 * the caller keeps ownership of the stream.  *out receives the context. */
ara_status ara_create(int cuda_device, void *cuda_stream, ara_ctx **out);

/*
 * Arithmetic precision of the store and the scan: 64 (default: fp64, the graded path, bit-
 * identical to the fp64 oracle) or 32 (the paper's optimisation "changing the double variables to
 * float variables"): losses and terms are rounded to float once
 * when the store is built, every step of Algorithm 1 runs in float in the same order, and the
 * YLT is widened to double.  Invalidates the layers: call before ara_set_layers.
 * Errors: ARA_ERR_ARG (bits not 32 or 64).
 */
ara_status ara_set_precision(ara_ctx *ctx, uint32_t bits);

/* Change the stream of an existing context (caller-owned cudaStream_t or NULL). */
ara_status ara_set_stream(ara_ctx *ctx, void *cuda_stream);

/* Release the context and every buffer it owns.  NULL is a no-op. */
void ara_destroy(ara_ctx *ctx);

/* Message describing the last failed call on ctx ("" if none).  Valid until the next call. */
const char *ara_last_error(const ara_ctx *ctx);

/*
 * ara_load_elts -- the second input of PAPER.md Sec. II: ELTs as CSR over records.
 *   catalogue_size        number of events in the global catalogue C (ids are 1..C)
 *   n_elts                number of ELTs (>= 1)
 *   rec_offsets[n_elts+1] non-decreasing; ELT j's records are [rec_offsets[j], rec_offsets[j+1])
 *   rec_event_ids[]       event id of each record, in [1, C], unique within an ELT
 *   rec_losses[]          loss l_i of each record, finite and >= 0 (0 is the same as absent)
 *   fin[n_elts]           financial terms of each ELT
 * Copies what it needs; the arrays may be freed afterwards.  Invalidates any layers.
 * Errors: ARA_ERR_ARG, ARA_ERR_RANGE (id 0 or > C), ARA_ERR_VALIDATION (duplicate id in an
 * ELT, bad loss or terms, decreasing offsets), ARA_ERR_OOM.
 */
ara_status ara_load_elts(ara_ctx *ctx, uint32_t catalogue_size, uint32_t n_elts,
                         const uint64_t *rec_offsets, const uint32_t *rec_event_ids,
                         const double *rec_losses, const ara_fin_terms *fin);

/*
 * ara_set_layers -- the third input of PAPER.md Sec. II (L55-L59) and the preprocessing stage
 * of Algorithm 1 (L61): builds, per layer, the device ELT store:
 *   map[0..C]  (u32)  catalogue id -> dense row, 0 = event in none of the layer's ELTs
 *   rows[0..U][W]     fp64, row r = the losses of the r-th event of the union U of the layer's
 *                     ELT events, column j = the layer's j-th ELT (0 where absent); row 0 zero;
 *                     W = |E_l| rounded up to whole 32-byte chunks: 4, 8, 16, 24 (17-24
 *                     ELTs on the 3-lane pair scan), 32, 48 or 64 doubles (row_width_for in
 *                     csrc/ara_internal.h); on the device the columns of W >= 24 rows are
 *                     lane-interleaved for the kernel that reads them (row_phys_col), exported
 *                     in this logical order by ara_export_store
 * i.e. the paper's direct access tables (L124) re-laid-out event-major and compacted.
 *   n_layers               >= 1
 *   terms[n_layers]        layer terms T
 *   elt_offsets[n_layers+1] non-decreasing; layer l covers elt_index[elt_offsets[l] ..
 *                          elt_offsets[l+1]), non-empty, at most ARA_MAX_ELTS_PER_LAYER
 *   elt_index[]            ELT numbers < n_elts, distinct within a layer; the listed order is
 *                          the summation order of Alg. 1 lines 11-13
 * Errors: ARA_ERR_STATE (no ELTs), ARA_ERR_ARG, ARA_ERR_VALIDATION, ARA_ERR_UNSUPPORTED,
 * ARA_ERR_OOM, ARA_ERR_CUDA.  Synchronous.
 */
ara_status ara_set_layers(ara_ctx *ctx, uint32_t n_layers, const ara_layer_terms *terms,
                          const uint32_t *elt_offsets, const uint32_t *elt_index);

/*
 * ara_run -- Algorithm 1 lines 2-29 over a device-resident YET: YET -> YLT.
 *   n_trials                  number of trials (0 is a no-op)
 *   d_trial_offsets[n+1]      device, u64, non-decreasing; trial t's events are
 *                             d_event_ids[d_trial_offsets[t] - d_trial_offsets[0] ...
 *                             d_trial_offsets[t+1] - d_trial_offsets[0]) in ascending time order
 *                             (only the order is used: PAPER.md L42; timestamps are not taken)
 *   d_event_ids[]             device, u32 catalogue ids in [1, C]
 *   d_ylt                     device, fp64, YLT[l][t] at d_ylt[l * ylt_ld + t]
 *   ylt_ld                    row stride of the YLT in elements (0 means n_trials)
 *   flags                     ARA_RUN_SYNC | ARA_RUN_VALIDATE | ARA_RUN_BALANCE | ARA_RUN_HOIST
 * Without ARA_RUN_SYNC the call only enqueues work on the context stream and returns ARA_OK;
 * an event id outside [1, C] then reads the zero row (never out of bounds) and sets a device
 * error flag that the next ara_synchronize() (or synchronous call) reports as ARA_ERR_RANGE.
 * Performance heuristics (never results): in row addressing mode 2 each run samples 65,536 of
 * the YET's ids (hit probe) and skips the presence-bitmap test when >= 99% are in the store;
 * the length check / probe counts of a run are copied back asynchronously and steer the next
 * run's schedule and kernel choice (see ARA_RUN_BALANCE).
 * Errors: ARA_ERR_STATE, ARA_ERR_ARG, ARA_ERR_RANGE, ARA_ERR_VALIDATION, ARA_ERR_CUDA.
 */
ara_status ara_run(ara_ctx *ctx, uint64_t n_trials, const uint64_t *d_trial_offsets,
                   const uint32_t *d_event_ids, double *d_ylt, uint64_t ylt_ld, uint32_t flags);

/*
 * ara_run_outputs -- ara_run with the optional per-trial and per-event outputs of the same pass
 * (YLT consumers; "financial functions or filters are then
 * applied on the aggregate loss values"):
 *   ylt, ylt_ld               as ara_run (required)
 *   max_occ, max_occ_ld       optional [n_layers][ld] device fp64: per (layer, trial) the largest
 *                             occurrence loss lo_d after line 16 (0 for an empty trial); its
 *                             distribution is the occurrence exceedance (OEP) curve, e.g.
 *                             ara_metrics on a max_occ row gives OEP PML / TVaR
 *   event_inc, event_inc_ld   optional [n_layers][ld] device fp64: the incremental aggregate
 *                             loss of lines 24-26 of every event, stored at the event's YET
 *                             position offsets[t] - offsets[0] + d (ld >= the YET's event count;
 *                             0 means exactly that count); a trial's entries sum to lr (line 28)
 *                             and allocate the trial loss to its events
 * A leading dimension of 0 means the minimum.  Requesting event_inc costs one synchronous read of
 * offsets[0] and offsets[n] (to check ld).  Errors: as ara_run.
 */
typedef struct {
    double *ylt;
    uint64_t ylt_ld;
    double *max_occ;
    uint64_t max_occ_ld;
    double *event_inc;
    uint64_t event_inc_ld;
} ara_outputs;

ara_status ara_run_outputs(ara_ctx *ctx, uint64_t n_trials, const uint64_t *d_trial_offsets,
                           const uint32_t *d_event_ids, const ara_outputs *out, uint32_t flags);

/*
 * ara_run_host -- ara_run with HOST buffers (end-to-end path): h_trial_offsets[n+1] and
 * h_event_ids as in ara_run but in host memory (page-locked memory gives full PCIe bandwidth),
 * h_ylt[l * ylt_ld + t] in host memory.  The YET is streamed to the device in chunks on the
 * context stream and a copy stream, overlapping copies with the scan.  Synchronous.
 * Errors: as ara_run (validation of ids is always performed on the device).
 */
ara_status ara_run_host(ara_ctx *ctx, uint64_t n_trials, const uint64_t *h_trial_offsets,
                        const uint32_t *h_event_ids, double *h_ylt, uint64_t ylt_ld,
                        uint32_t flags);

/* Wait for all work enqueued on the context stream; report deferred device errors. */
ara_status ara_synchronize(ara_ctx *ctx);

/*
 * ara_metrics -- PML and TVaR of one YLT row (reading R11):
 *   PML(p)  = v[ceil(p * n) - 1] of the row sorted ascending (nearest rank)
 *   TVaR(p) = mean of all v >= PML(p)
 *   d_ylt_row[n]   device, fp64, finite
 *   p[n_p]         host, each in (0, 1), n_p <= ARA_MAX_P
 *   pml_out, tvar_out  host, [n_p]
 * Computed on the device (radix select + tail mean); synchronous.
 * Errors: ARA_ERR_EMPTY (n == 0), ARA_ERR_ARG (p outside (0,1), n_p == 0 or > ARA_MAX_P),
 * ARA_ERR_CUDA.
 */
ara_status ara_metrics(ara_ctx *ctx, const double *d_ylt_row, uint64_t n, uint32_t n_p,
                       const double *p, double *pml_out, double *tvar_out);

/*
 * ara_metrics_rows -- ara_metrics for n_rows rows of one matrix in the same radix-select passes
 * (e.g. every layer of a YLT plus the portfolio row): one cooperative launch per
 * floor(64 / n_p) rows instead of one per row.  Row r is d_rows[r * ld .. r * ld + n) (ld = 0
 * means n).  pml_out / tvar_out are host arrays [n_rows][n_p].  Results equal ara_metrics on
 * each row.  Synchronous.  Errors: as ara_metrics.
 */
ara_status ara_metrics_rows(ara_ctx *ctx, const double *d_rows, uint32_t n_rows, uint64_t ld,
                            uint64_t n, uint32_t n_p, const double *p, double *pml_out,
                            double *tvar_out);

/*
 * ara_portfolio_ylt -- portfolio-scope trial losses (a loss distribution's
 * scope is a single layer or the portfolio = per-trial sum over layers):
 *   d_out[t] = ((0 + YLT[0][t]) + YLT[1][t]) + ... + YLT[L-1][t], left to right in layer order,
 * for the context's L layers.  Feed d_out to ara_metrics for portfolio PML / TVaR.
 *   d_ylt    device fp64, YLT[l][t] at d_ylt[l * ylt_ld + t] (as written by ara_run)
 *   ylt_ld   row stride in elements (0 means n_trials);  d_out  device fp64[n_trials]
 *   flags    ARA_RUN_SYNC or 0 (stream-ordered)
 * Errors: ARA_ERR_STATE, ARA_ERR_ARG, ARA_ERR_CUDA.
 */
ara_status ara_portfolio_ylt(ara_ctx *ctx, const double *d_ylt, uint64_t n_trials,
                             uint64_t ylt_ld, double *d_out, uint32_t flags);

/*
 * ara_metrics_sharded -- PML / TVaR of a YLT row that is split over several processes (one
 * contiguous slice per rank, e.g. the trial shards of SURVEY.md 8(e)), without gathering the
 * row: the same MSB radix select as ara_metrics runs pass by pass on every rank's slice, and
 * between passes the caller's reduction sums the per-rank 256-bin histograms; the tail sums
 * and counts are reduced the same way.  Every rank must call it with the same n_global, n_p and
 * p; every rank receives the same PML (exact) and TVaR (the tail sum's order differs from
 * ara_metrics': equal within rounding).
 *   d_ylt_slice[n_local]  device fp64, this rank's part of the row (n_local may be 0)
 *   n_global              the whole row's length (sum of n_local over ranks), > 0
 *   d_xbuf, xbuf_bytes    caller-owned device exchange buffer of >= ARA_MAX_P * 256 * 8 bytes
 *   reduce(offset, count, is_f64, user): the caller's element-wise SUM across all ranks, in
 *                         place, of `count` int64 (is_f64 = 0) or fp64 (is_f64 = 1) values at
 *                         byte `offset` of d_xbuf, ordered after the work already enqueued on
 *                         the context's stream and before what follows (e.g. an NCCL
 *                         all-reduce on that stream); returns 0 on success.  Called 10 times.
 * Synchronous.  Errors: ARA_ERR_EMPTY (n_global == 0), ARA_ERR_ARG (p outside (0,1), NULL,
 * small buffer, n_local > n_global, the callback failed), ARA_ERR_CUDA.
 */
typedef int (*ara_shard_reduce)(uint64_t offset, uint64_t count, int is_f64, void *user);
ara_status ara_metrics_sharded(ara_ctx *ctx, const double *d_ylt_slice, uint64_t n_local,
                               uint64_t n_global, uint32_t n_p, const double *p, double *pml_out,
                               double *tvar_out, void *d_xbuf, uint64_t xbuf_bytes,
                               ara_shard_reduce reduce, void *user);

/* ara_metrics on a HOST YLT row (copied to the device first).  Synchronous. */
ara_status ara_metrics_host(ara_ctx *ctx, const double *h_ylt_row, uint64_t n, uint32_t n_p,
                            const double *p, double *pml_out, double *tvar_out);

/* F4 ("financial functions or filters are then applied on the
 * aggregate loss values"; L32): the exceedance-probability curve of one row -- the AEP curve of a
 * YLT row (annual aggregate loss per trial) or the OEP curve of a max_occ row of ara_run_outputs
 * (annual maximum occurrence loss).  d_curve[i] = the (i+1)-th largest of d_row[0..n), i.e. the
 * loss whose empirical exceedance probability is (i+1)/n (return period n/(i+1) years); -0 is
 * returned as +0.  Every PML of ara_metrics is a point on it: PML(p) = d_curve[n - ceil(p n)]
 * (readings R11, R15).
 *   d_row    device, n doubles, caller-owned, read only;
 *   d_curve  device, n doubles, caller-owned, must not overlap d_row.
 * Stream-ordered on the context stream (no host synchronisation); the context keeps an internal
 * scratch buffer (2n keys + the sort's temporary storage), grown on demand.
 * Errors: ARA_ERR_EMPTY (n = 0), ARA_ERR_ARG (NULL or overlapping pointers), ARA_ERR_CUDA. */
ara_status ara_ep_curve(ara_ctx *ctx, const double *d_row, uint64_t n, double *d_curve);

/* Introspection (tests, benchmarks). */
typedef struct {
    uint32_t catalogue_size;
    uint32_t n_elts;
    uint32_t n_layers;
    uint32_t max_row_width;      /* max W over layers (doubles per row)                  */
    uint64_t store_bytes;        /* device bytes of maps + rows of all layers            */
    uint64_t kernel_launches;    /* kernels launched by this context so far               */
    int device;
    int sm_count;
    int row_addressing;          /* how the scan finds an event's row:
                                    0 = catalogue map -> dense row; 1 = rows indexed by
                                    catalogue id; 2 = as 1 behind a shared-memory presence
                                    bitmap.  Results are identical in every mode.          */
    int layer_kernel;            /* how several layers are scanned: 0 = rows
                                    per layer (one fused launch); 1 = union rows, layer sums
                                    through a shared-memory F row; 2 = union rows, layer sums
                                    through register shuffles; 3 = union rows, half of each
                                    layer's ELTs in its own lane (blocks of 8), the other half
                                    by shuffles.  Identical results.                        */
    uint32_t gather_row_bytes;   /* row bytes the scan gathers per event (all layers; the
                                    union row when layer_kernel > 0)                        */
    char last_kernel[64];        /* the scan-kernel instantiation the last ara_run* launched,
                                    as ncu names it (e.g. "pair_scan_kernel<2, 2, 3, 1, 0>");
                                    "" before the first run                                 */
} ara_info;

ara_status ara_get_info(const ara_ctx *ctx, ara_info *out);

/* Per-layer store shape: number of union events U (rows = U + 1) and row width W. */
ara_status ara_layer_store_shape(const ara_ctx *ctx, uint32_t layer, uint32_t *n_union,
                                 uint32_t *row_width);

/* Copy a layer's device store back to the host (store round-trip tests):
 * h_map[C+1] (u32) and h_rows[(U+1) * W] (fp64, logical column order: column j = the layer's
 * j-th ELT).  Either pointer may be NULL.  Synchronous. */
ara_status ara_export_store(ara_ctx *ctx, uint32_t layer, uint32_t *h_map, double *h_rows);

#ifdef __cplusplus
}
#endif
#endif /* ARA_H */
