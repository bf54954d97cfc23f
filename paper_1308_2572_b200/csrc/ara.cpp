// ara.cpp -- host side of libara: the C ABI of include/ara.h.
//
// Context state machine, input validation (SPEC.md core-model rules), the device ELT store
// build of ara_set_layers (A1: event-major rows + catalogue map),
// and orchestration of the scan (A2-A8) and metrics (A9) kernels on the context stream.
#include <cuda_runtime.h>
#include <math.h>

#include <cmath>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <new>
#include <string>
#include <vector>

#include "ara.h"
#include <nvtx3/nvToolsExt.h>

#include "ara_internal.h"

struct ara_ctx {
    int device = 0;
    int sm_count = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;
    std::string err;
    std::string last_kernel;  // ara_info.last_kernel

    bool have_elts = false;
    bool have_layers = false;
    uint32_t C = 0;
    uint32_t n_elts = 0;
    std::vector<uint64_t> rec_off;
    std::vector<uint32_t> rec_ids;
    std::vector<double> rec_losses;
    std::vector<ara_fin_terms> fin;

    ara::DeviceStore store;  // all layers (valid when have_layers)
    uint64_t store_bytes = 0;

    uint32_t *d_err = nullptr;  // device error word (ara::kErr*)
    unsigned long long *d_ticket = nullptr;  // dynamic scheduling: ticket + done counters
    // Per-run statistics on the device: [0] hit-probe ids present, [1] ids sampled (map mode
    // 2), [2] trial lengths not all equal, [3] set when [2] was measured.  Copied back
    // asynchronously and read by the host one run later (never waited for): performance
    // heuristics only -- every choice they drive gives the same YLT.
    unsigned long long *d_probe = nullptr;
    unsigned long long *h_probe = nullptr;  // pinned copy of the last completed run's stats
    cudaEvent_t ev_probe = nullptr;
    bool probe_pending = false;             // a copy into h_probe is in flight
    bool probe_mode1 = false;               // the last probe said ">= 99% present"
    bool lengths_equal = false;             // the last check said "all trials equally long"
    int sched = 0;              // 0 auto, 1 static, 2 dynamic (env ARA_SCAN_SCHED)
    bool probe = true;          // map mode 2 hit probe (env ARA_MAP_PROBE=0 disables)
    int bits = 64;              // store / arithmetic precision (ara_set_precision)
    uint32_t *h_err = nullptr;  // pinned mirror
    uint64_t launches = 0;
    ara::MetricsScratch metrics;
    ara::EpScratch ep;
    ara::SortScratch sort;

    // ara_run_host staging (double-buffered)
    uint32_t *d_ids_stage[2] = {nullptr, nullptr};
    uint64_t *d_off_stage[2] = {nullptr, nullptr};
    size_t ids_stage_cap = 0;   // u32 elements per buffer
    size_t off_stage_cap = 0;   // u64 elements per buffer
    double *d_ylt_stage = nullptr;
    size_t ylt_stage_cap = 0;
    cudaEvent_t ev_copy[2] = {nullptr, nullptr};
    cudaEvent_t ev_done[2] = {nullptr, nullptr};
    double *d_row_stage = nullptr;  // ara_metrics_host
    size_t row_stage_cap = 0;
};

namespace {

ara_status fail(ara_ctx *ctx, ara_status s, const char *fmt, ...)
{
    if (ctx) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof(buf), fmt, ap);
        va_end(ap);
        ctx->err = buf;
    }
    return s;
}

ara_status cuda_fail(ara_ctx *ctx, cudaError_t e, const char *what)
{
    return fail(ctx, e == cudaErrorMemoryAllocation ? ARA_ERR_OOM : ARA_ERR_CUDA, "%s: %s (%s)",
                what, cudaGetErrorString(e), cudaGetErrorName(e));
}

#define ARA_CUDA(ctx, call)                                   \
    do {                                                      \
        cudaError_t e_ = (call);                              \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev)
    {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard()
    {
        int cur;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

bool finite_nonneg(double x) { return isfinite(x) && x >= 0.0; }
bool limit_ok(double x) { return !isnan(x) && x >= 0.0; }  // +inf allowed

void free_layers(ara_ctx *ctx)
{
    cudaFree(ctx->store.d_map);
    cudaFree(ctx->store.d_rows);
    cudaFree(ctx->store.d_terms);
    cudaFree(ctx->store.uni.d_rows);
    cudaFree(ctx->store.uni.d_terms);
    cudaFree(ctx->store.uni.d_rows_direct);
    cudaFree(ctx->store.d_rows_direct);
    cudaFree(ctx->store.d_bitmap);
    cudaFree(ctx->store.d_union_ids);
    cudaFree(ctx->store.d_oc);
    cudaFree(ctx->store.d_oc_bitmap);
    ctx->store = ara::DeviceStore();
    ctx->store_bytes = 0;
    ctx->probe_mode1 = false;  // a new store: no probe verdict yet
    ctx->have_layers = false;
}

// NVTX range around every C-ABI call (header-only NVTX3; visible in nsys / ncu timelines).
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

template <typename F>
ara_status guarded(ara_ctx *ctx, const char *name, F &&f)
{
    if (!ctx) return ARA_ERR_ARG;
    NvtxRange range(name);
    try {
        ctx->err.clear();
        DeviceGuard g(ctx->device);
        return f();
    } catch (const std::bad_alloc &) {
        return fail(ctx, ARA_ERR_OOM, "host allocation failed");
    } catch (...) {
        return fail(ctx, ARA_ERR_ARG, "unexpected exception");
    }
}

ara_status validate_p(ara_ctx *ctx, uint32_t n_p, const double *p)
{
    if (n_p == 0 || n_p > ARA_MAX_P)
        return fail(ctx, ARA_ERR_ARG, "n_p = %u outside [1, %d]", n_p, ARA_MAX_P);
    if (!p) return fail(ctx, ARA_ERR_ARG, "p is NULL");
    for (uint32_t i = 0; i < n_p; ++i)
        if (!(p[i] > 0.0 && p[i] < 1.0))
            return fail(ctx, ARA_ERR_ARG, "p[%u] = %g outside (0, 1)", i, p[i]);
    return ARA_OK;
}

ara_status check_device_error(ara_ctx *ctx)
{
    ARA_CUDA(ctx, cudaMemcpyAsync(ctx->h_err, ctx->d_err, 4, cudaMemcpyDeviceToHost, ctx->stream));
    ARA_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    const uint32_t e = *ctx->h_err;
    if (e) {
        ARA_CUDA(ctx, cudaMemsetAsync(ctx->d_err, 0, 4, ctx->stream));
        ARA_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        if (e & ara::kErrOffsets)
            return fail(ctx, ARA_ERR_VALIDATION, "trial offsets are decreasing");
        return fail(ctx, ARA_ERR_RANGE, "a trial event id is 0 or exceeds the catalogue (%u)",
                    ctx->C);
    }
    return ARA_OK;
}

// One scan launch covers every layer (layer-fused pass: one id read and one map lookup per
// event serve all layers).
// ARA_RUN_HOIST (hoist.cu): the per-event layer-loss table, allocated (zeroed) on first use.
ara_status prepare_hoist(ara_ctx *ctx)
{
    ara::DeviceStore &st = ctx->store;
    if (st.n_layers > 8)
        return fail(ctx, ARA_ERR_UNSUPPORTED, "ARA_RUN_HOIST supports up to 8 layers (%u)",
                    st.n_layers);
    if (!st.d_oc) {
        uint32_t lp = 1;
        while (lp < st.n_layers) lp *= 2;
        const size_t rb = (size_t)lp * (st.bits / 8);
        int direct = st.map_mode >= 1;
        size_t bytes = ((size_t)(direct ? ctx->C : st.n_union) + 1) * rb;
        size_t free_b = 0, total_b = 0;
        if (direct && (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess || bytes > free_b / 4)) {
            direct = 0;
            bytes = ((size_t)st.n_union + 1) * rb;
        }
        ARA_CUDA(ctx, cudaMalloc(&st.d_oc, bytes));
        ARA_CUDA(ctx, cudaMemsetAsync(st.d_oc, 0, bytes, ctx->stream));
        st.oc_lp = lp;
        st.oc_direct = direct;
        ctx->store_bytes += bytes;
        if (direct && st.map_mode == 2) {
            const size_t bb = ara::bitmap_bytes(ara::kBitmapLog2Hoist);
            ARA_CUDA(ctx, cudaMalloc(&st.d_oc_bitmap, bb));
            ARA_CUDA(ctx, ara::launch_build_bitmap(st.d_map, ctx->C, st.d_oc_bitmap,
                                                   ara::kBitmapLog2Hoist, ctx->stream));
            ctx->store_bytes += bb;
        }
    }
    cudaError_t e = ara::launch_hoist_oc(st, ctx->stream, &ctx->launches);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "hoist kernel launch");
    return ARA_OK;
}

ara_status launch_layers(ara_ctx *ctx, uint64_t n, const uint64_t *d_off, const uint32_t *d_ids,
                         double *d_ylt, uint64_t ld, uint32_t flags,
                         const ara_outputs *extra = nullptr)
{
    // Scheduling (results are identical either way).  Default: trials sorted by length on the
    // device and handed out in warp-sized batches, so the thread groups of a warp run trials of
    // nearly equal length (variable-length YETs keep full SIMT width; measured neutral for
    // equal lengths, profiles/README.md).  ARA_SCAN_SCHED=static|dynamic selects the plain
    // round-robin / per-group ticket schedules (tuning); the F4 outputs use per-group tickets.
    const bool hoist = (flags & ARA_RUN_HOIST) && !extra;
    const bool hoist_bm = hoist && ctx->store.d_oc_bitmap;
    const bool probing = !extra && ctx->probe && (ctx->store.map_mode == 2 || hoist_bm);
    // the previous run's statistics, if their copy has landed
    if (ctx->probe_pending) {
        const cudaError_t q = cudaEventQuery(ctx->ev_probe);
        if (q == cudaSuccess) {
            const unsigned long long *h = ctx->h_probe;
            if (h[1] > 0) ctx->probe_mode1 = 100ull * h[0] >= 99ull * h[1];
            if (h[3]) ctx->lengths_equal = h[2] == 0;
            ctx->probe_pending = false;
        } else if (q == cudaErrorNotReady) {
            cudaGetLastError();  // "not ready" is not an error; keep it out of the launch checks
        } else {
            return cuda_fail(ctx, q, "run statistics event");
        }
    }
    ARA_CUDA(ctx, cudaMemsetAsync(ctx->d_probe, 0, 32, ctx->stream));
    // Scheduling (results are identical either way).  Default: trials sorted by length on the
    // device and handed out in warp-sized batches, so the thread groups of a warp run trials of
    // nearly equal length (variable-length YETs keep full SIMT width; measured neutral for
    // equal lengths, profiles/README.md).  When the previous run's trials were all equally long
    // the sort is skipped (identity order; a cheap check keeps the verdict current).
    // ARA_SCAN_SCHED=static|dynamic selects the plain round-robin / per-group ticket schedules
    // (tuning); the F4 outputs of an fp32 store use per-group tickets.
    const bool balance = ctx->sched == 0 && (!extra || ctx->store.bits == 64) &&
                         n <= 0x7fffffffull;  // u32 permutation, CUB's int item count
    const bool sorted = balance && !ctx->lengths_equal;
    // (rows laid out for the 3-lane pair scan -- 17-24 ELTs -- are read by no other kernel: its
    // warp-batched tickets whatever the trial count)
    const bool dyn = balance || ctx->sched == 2 || (ctx->sched == 0 && ctx->store.n_layers == 1) ||
                     (ctx->sched != 1 && (ctx->store.ilv == 2 || ctx->store.ilv == 3));
    const uint32_t *perm = nullptr;
    if (sorted) {
        cudaError_t e = ara::launch_length_sort(d_off, n, ctx->sort, ctx->sm_count, ctx->stream,
                                                &ctx->launches, ctx->d_probe + 2);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "length sort");
        perm = ctx->sort.perm;
    } else if (balance) {  // equally long trials: identity order, same warp-batched kernel
        cudaError_t e = ara::launch_length_check(d_off, n, ctx->sort, ctx->d_probe + 2,
                                                 ctx->sm_count, ctx->stream, &ctx->launches);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "length check");
        perm = ctx->sort.perm;
    }
    ara::ScanLaunch s{d_off, d_ids, d_ylt, ld, n, ctx->C, ctx->d_err,
                      0u, 0u,  // zero_base, bitmap_log2: set per launch by the kernel's store
                      dyn ? ctx->d_ticket : nullptr,
                      dyn ? (unsigned int *)(ctx->d_ticket + 1) : nullptr,
                      extra ? extra->max_occ : nullptr, extra ? extra->max_occ_ld : 0,
                      extra ? extra->event_inc : nullptr, extra ? extra->event_inc_ld : 0, perm,
                      nullptr};
    // Map mode 2 (direct rows behind the presence bitmap): a probe of the YET's hit rate lets
    // the scan skip the bitmap test when (nearly) every id is in the store; results do not
    // depend on it.  ARA_MAP_PROBE=0 disables the probe (tuning).  The kernels read the probe
    // on the device and run their mode-1 body when >= 99% of the sampled ids are present; when
    // the previous run's probe said the same, the host launches the plain mode-1 kernel (~3%
    // faster than the combined one).
    const bool mode1 = probing && ctx->probe_mode1;
    if (probing) {
        cudaError_t pe = ara::launch_hit_probe(d_off, d_ids, n, ctx->store.d_map, ctx->C,
                                               ctx->d_probe, ctx->stream, &ctx->launches);
        if (pe != cudaSuccess) return cuda_fail(ctx, pe, "hit probe");
        s.probe = ctx->d_probe;
    }
    if (balance) {  // mark the length verdict as measured ([3] = 1) via a 1-value memset
        ARA_CUDA(ctx, cudaMemsetAsync((char *)(ctx->d_probe + 3), 1, 1, ctx->stream));
    }
    if (!ctx->probe_pending && (probing || balance)) {
        ARA_CUDA(ctx, cudaMemcpyAsync(ctx->h_probe, ctx->d_probe, 32, cudaMemcpyDeviceToHost,
                                      ctx->stream));
        ARA_CUDA(ctx, cudaEventRecord(ctx->ev_probe, ctx->stream));
        ctx->probe_pending = true;
    }
    cudaError_t e;
    if (mode1) {  // a store view addressed like map mode 1 (same buffers)
        ara::DeviceStore st1 = ctx->store;
        st1.map_mode = 1;
        st1.d_oc_bitmap = nullptr;
        e = hoist ? ara::launch_hoisted_scan(st1, s, ctx->sm_count, ctx->stream, &ctx->launches)
            : st1.uni.enabled
                ? ara::launch_portfolio(st1.uni, st1.d_map, 1, st1.d_bitmap, s, ctx->sm_count,
                                        ctx->stream, &ctx->launches)
                : ara::pair_scan_eligible(st1, s)
                    ? ara::launch_pair_scan(st1, s, ctx->sm_count, ctx->stream, &ctx->launches)
                    : ara::launch_scan(st1, s, ctx->sm_count, ctx->stream, &ctx->launches);
    } else {
        e = hoist ? ara::launch_hoisted_scan(ctx->store, s, ctx->sm_count, ctx->stream,
                                             &ctx->launches)
            : (ctx->store.uni.enabled && !extra)
                ? ara::launch_portfolio(ctx->store.uni, ctx->store.d_map, ctx->store.map_mode,
                                        ctx->store.d_bitmap, s, ctx->sm_count, ctx->stream,
                                        &ctx->launches)
                : ara::pair_scan_eligible(ctx->store, s)
                    ? ara::launch_pair_scan(ctx->store, s, ctx->sm_count, ctx->stream,
                                            &ctx->launches)
                    : ara::launch_scan(ctx->store, s, ctx->sm_count, ctx->stream, &ctx->launches);
    }
    if (e == cudaErrorInvalidValue && (ctx->store.ilv == 2 || ctx->store.ilv == 3))
        return fail(ctx, ARA_ERR_UNSUPPORTED,  // only the pair scan reads these row layouts
                    "rows laid out for the pair scan need the warp-batched schedule "
                    "(ARA_SCAN_SCHED unset, <= 2^31 trials)");
    if (e != cudaSuccess) return cuda_fail(ctx, e, "scan kernel launch");
    if (ara::t_last_kernel) ctx->last_kernel = ara::t_last_kernel;
    return ARA_OK;
}

// Event-major rows and per-layer terms of the store in precision R (double: bit copies of the
// losses; float: each value rounded to nearest once, F3).  Layer l's columns sit at l * W.
template <typename R>
void build_rows(const ara_ctx *ctx, const ara::DeviceStore &st, const std::vector<uint32_t> &map,
                const ara_layer_terms *terms, const uint32_t *elt_offsets,
                const uint32_t *elt_index, std::vector<char> &rows_buf,
                std::vector<char> &terms_buf)
{
    const uint32_t n_layers = st.n_layers, W = st.width;
    const size_t stride = (size_t)n_layers * W;
    rows_buf.assign((size_t)(st.n_union + 1 + ara::kZeroRows) * stride * sizeof(R), 0);
    terms_buf.assign((size_t)n_layers * sizeof(ara::LayerTermsT<R>), 0);
    R *rows = (R *)rows_buf.data();
    ara::LayerTermsT<R> *lt = (ara::LayerTermsT<R> *)terms_buf.data();
    for (uint32_t l = 0; l < n_layers; ++l) {
        const uint32_t E = st.n_cols[l];
        for (uint32_t c = 0; c < E; ++c) {
            const uint32_t j = elt_index[elt_offsets[l] + c];
            for (uint64_t r = ctx->rec_off[j]; r < ctx->rec_off[j + 1]; ++r)
                rows[(size_t)map[ctx->rec_ids[r]] * stride + (size_t)l * W +
                     ara::row_phys_col(c, W, st.ilv)] = (R)ctx->rec_losses[r];
            lt[l].rate[c] = (R)ctx->fin[j].rate;
            lt[l].ret[c] = (R)ctx->fin[j].retention;
            lt[l].lim[c] = (R)ctx->fin[j].limit;
        }
        for (uint32_t c = E; c < ara::kMaxCols; ++c) {  // neutral padding columns
            lt[l].rate[c] = (R)1;
            lt[l].ret[c] = (R)0;
            lt[l].lim[c] = (R)INFINITY;
        }
        lt[l].occ_ret = (R)terms[l].occ_retention;
        lt[l].occ_lim = (R)terms[l].occ_limit;
        lt[l].agg_ret = (R)terms[l].agg_retention;
        lt[l].agg_lim = (R)terms[l].agg_limit;
    }
}

// scan_pair.cu carries 2^m multiples of the oracle's values (exact scaled clamps); this bounds
// every input magnitude it scales: each record's loss * rate (rounded up), each retention and
// finite limit, each layer term.  With all of them below 2^960 no scaled intermediate of a trial
// of k < 2^36 events over E <= 64 ELTs can overflow (8 (k (E + 1) + 1) 2^960 < 2^1023).
bool scaled_terms_ok(const ara_ctx *ctx, uint32_t n_layers, const ara_layer_terms *terms,
                     const uint32_t *elt_offsets, const uint32_t *elt_index)
{
    const double bound = std::ldexp(1.0, 960);
    auto ok = [&](double v) { return std::isinf(v) || v < bound; };  // +inf limits scale to +inf
    for (uint32_t l = 0; l < n_layers; ++l) {
        const ara_layer_terms &t = terms[l];
        if (!ok(t.occ_limit) || !ok(t.agg_limit) || !(t.occ_retention < bound) ||
            !(t.agg_retention < bound))
            return false;
        for (uint32_t c = elt_offsets[l]; c < elt_offsets[l + 1]; ++c) {
            const uint32_t j = elt_index[c];
            const ara_fin_terms &f = ctx->fin[j];
            if (!(f.retention < bound) || !(f.rate < bound) || !ok(f.limit)) return false;
            for (uint64_t r = ctx->rec_off[j]; r < ctx->rec_off[j + 1]; ++r)
                if (!(ctx->rec_losses[r] * f.rate * 1.0000001 < bound)) return false;
        }
    }
    return true;
}

// F1 union-row store (portfolio.cu) when the portfolio qualifies; returns ARA_OK either way
// unless a CUDA call fails.
ara_status build_union(ara_ctx *ctx, const std::vector<uint32_t> &map,
                       const ara_layer_terms *terms, const uint32_t *elt_offsets,
                       const uint32_t *elt_index)
{
    ara::DeviceStore &st = ctx->store;
    const uint32_t L = st.n_layers;
    if (ctx->bits != 64 || L < 2 || L > (uint32_t)ara::kUnionMaxLayers) return ARA_OK;
    if (const char *e = getenv("ARA_PORTFOLIO"))
        if (atoi(e) == 0) return ARA_OK;
    std::vector<uint32_t> J;  // distinct ELTs in order of first appearance
    std::vector<int> col_of(ctx->n_elts, -1);
    for (uint32_t l = 0; l < L; ++l) {
        if (st.n_cols[l] > (uint32_t)ara::kUnionMaxE) return ARA_OK;
        for (uint32_t c = elt_offsets[l]; c < elt_offsets[l + 1]; ++c)
            if (col_of[elt_index[c]] < 0) {
                col_of[elt_index[c]] = (int)J.size();
                J.push_back(elt_index[c]);
            }
    }
    if (J.size() > (size_t)ara::kMaxCols) return ARA_OK;
    uint32_t GU = 2;
    while (8 * GU < J.size() || GU < L) GU *= 2;
    if (GU > 8) return ARA_OK;
    const uint32_t WU = 8 * GU;
    auto u_slot = [](uint32_t col) { return col + 2 * (col >> 3); };
    // Register-shuffle layout (portfolio.cu): every ELT must sit in register (i mod 8) of some
    // lane for each position i it takes in a layer, so that one shuffle per position serves
    // every layer of the group; at most GU ELTs per register.  When the layer lists allow it
    // (configuration P does: ELT e is at positions e mod 8 and 8 + e mod 8), union column
    // `col` moves to lane lane_of[col], register reg_of[col]; otherwise the shared-memory F row
    // serves the layer sums.
    std::vector<int> reg_of(J.size(), -1), lane_of(J.size(), -1);
    bool shfl = true;
    for (uint32_t l = 0; l < L && shfl; ++l)
        for (uint32_t c = elt_offsets[l]; c < elt_offsets[l + 1]; ++c) {
            const int col = col_of[elt_index[c]], r = (int)((c - elt_offsets[l]) % 8);
            if (reg_of[col] >= 0 && reg_of[col] != r) shfl = false;
            reg_of[col] = r;
        }
    if (shfl) {
        std::vector<int> used(8, 0);
        for (size_t col = 0; col < J.size() && shfl; ++col) {
            lane_of[col] = used[reg_of[col]]++;
            if (lane_of[col] >= (int)GU) shfl = false;
        }
    }
    if (GU != 8) shfl = false;  // shuffle variants are built for GU = 8 only (portfolio.cu)
    // Block layout (portfolio.cu SH = 3): every layer has 16 ELTs, its first 8 (in layer order)
    // form a block no other layer starts with, its last 8 another layer's first block or a block
    // of its own, and the blocks partition J.  Lane l then holds layer l's first block in
    // registers 0-7 (no shuffle for half the positions) and the second half comes from one
    // source lane (configuration P: lane l + 1).  blk_lane[col] / blk_reg[col] place the columns.
    std::vector<int> blk_lane(J.size(), -1), blk_reg(J.size(), -1);
    std::vector<uint32_t> src2(L, 0);
    bool blocks = GU == 8;
    {
        int n_blocks = 0;
        auto place = [&](uint32_t l, uint32_t from, int lane) -> bool {  // 8 ELTs -> lane
            for (uint32_t i = 0; i < 8; ++i) {
                const int col = col_of[elt_index[elt_offsets[l] + from + i]];
                if (blk_lane[col] >= 0) return false;
                blk_lane[col] = lane;
                blk_reg[col] = (int)i;
            }
            return true;
        };
        for (uint32_t l = 0; l < L && blocks; ++l)
            blocks = st.n_cols[l] == (uint32_t)ara::kUnionMaxE && place(l, 0, (int)l);
        n_blocks = (int)L;
        for (uint32_t l = 0; l < L && blocks; ++l) {
            const int c0 = col_of[elt_index[elt_offsets[l] + 8]];
            int lane = blk_lane[c0];
            if (lane >= 0) {  // an existing block: the same 8 ELTs in the same order
                for (uint32_t i = 0; i < 8 && blocks; ++i) {
                    const int col = col_of[elt_index[elt_offsets[l] + 8 + i]];
                    blocks = blk_lane[col] == lane && blk_reg[col] == (int)i;
                }
            } else {
                lane = n_blocks++;
                blocks = lane < (int)GU && place(l, 8, lane);
            }
            src2[l] = (uint32_t)lane;
        }
        for (size_t col = 0; col < J.size() && blocks; ++col) blocks = blk_lane[col] >= 0;
    }
    if (const char *e = getenv("ARA_PORTFOLIO_SHFL")) {
        if (atoi(e) == 0) shfl = false;
        if (atoi(e) == 0 || atoi(e) == 2) blocks = false;  // 2: the per-position shuffles (tuning)
    }
    // the union column that holds J[col]: lane c's registers 0-3 are columns 4c..4c+3 and
    // registers 4-7 are columns 4(c+GU)..4(c+GU)+3 (portfolio.cu, the two gathers of a group)
    auto ucol = [&](uint32_t col) -> uint32_t {
        if (!shfl && !blocks) return col;
        const uint32_t r = (uint32_t)(blocks ? blk_reg[col] : reg_of[col]);
        const uint32_t c = (uint32_t)(blocks ? blk_lane[col] : lane_of[col]);
        return r < 4 ? 4 * c + r : 4 * (c + GU) + (r - 4);
    };
    std::vector<double> rows((size_t)(st.n_union + 1 + ara::kZeroRows) * WU, 0.0);
    ara::UnionTermsDev ut{};
    for (uint32_t col = 0; col < WU; ++col) {  // padding columns: neutral terms, zero losses
        ut.rate[col] = 1.0;
        ut.ret[col] = 0.0;
        ut.lim[col] = INFINITY;
    }
    for (uint32_t col = 0; col < J.size(); ++col) {
        const uint32_t j = J[col], u = ucol(col);
        for (uint64_t r = ctx->rec_off[j]; r < ctx->rec_off[j + 1]; ++r)  // bit copies
            rows[(size_t)map[ctx->rec_ids[r]] * WU + u] = ctx->rec_losses[r];
        ut.rate[u] = ctx->fin[j].rate;
        ut.ret[u] = ctx->fin[j].retention;
        ut.lim[u] = ctx->fin[j].limit;
    }
    ut.n_layers = L;
    bool full16 = true;
    for (uint32_t l = 0; l < L; ++l) {
        ut.n_cols[l] = st.n_cols[l];
        full16 = full16 && st.n_cols[l] == (uint32_t)ara::kUnionMaxE;
        for (uint32_t i = 0; shfl && !blocks && i < st.n_cols[l]; ++i) {
            const uint32_t lane = (uint32_t)lane_of[col_of[elt_index[elt_offsets[l] + i]]];
            ut.src5[l][i / 6] |= lane << (5 * (i % 6));
        }
    }
    for (uint32_t l = 0; l < (uint32_t)ara::kUnionMaxLayers; ++l) {
        const bool real = l < L;
        ut.occ_ret[l] = real ? terms[l].occ_retention : 0.0;
        ut.occ_lim[l] = real ? terms[l].occ_limit : 0.0;
        ut.agg_ret[l] = real ? terms[l].agg_retention : 0.0;
        ut.agg_lim[l] = real ? terms[l].agg_limit : 0.0;
        for (uint32_t i = 0; i < (uint32_t)ara::kUnionMaxE; ++i) {
            // layer order = summation order; past the layer's ELTs: the zero slot (+0 neutral)
            uint32_t slot = u_slot(WU);
            if (real && i < st.n_cols[l]) slot = u_slot(ucol(col_of[elt_index[elt_offsets[l] + i]]));
            ut.slot2[l][i / 2] |= slot << (16 * (i % 2));
        }
    }
    ara::UnionStore &us = st.uni;
    us.GU = GU;
    for (uint32_t l = 0; l < L; ++l) ut.src2[l] = src2[l];
    us.shfl = blocks ? 3 : shfl ? (full16 ? 2 : 1) : 0;
    us.scaled = st.scaled && st.pair_scan;  // ARA_PAIR_SCAN=0 also keeps the compare-selects
    us.n_cols = (uint32_t)J.size();
    us.zero_base = st.n_union + 1;
    const size_t row_bytes = rows.size() * 8;
    cudaError_t e = cudaMalloc(&us.d_rows, row_bytes);
    if (e == cudaSuccess) e = cudaMalloc(&us.d_terms, sizeof(ut));
    if (e == cudaSuccess) e = cudaMemcpy(us.d_rows, rows.data(), row_bytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(us.d_terms, &ut, sizeof(ut), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "union store");
    us.enabled = true;
    ctx->store_bytes += row_bytes + sizeof(ut);
    return ARA_OK;
}

// Map modes 1 and 2 (ara_internal.h): the rows the scan will read (union rows when the portfolio
// kernel serves the layers, else the per-layer rows) expanded on the device to one row per
// catalogue id, plus the presence bitmap for mode 2.  The direct rows are bit copies of the dense
// ones (direct[id] = dense[map[id]]; absent ids get the zero row), so the YLT does not depend
// on the mode.  Default mode 2; ARA_MAP_MODE=0|1|2 overrides (tuning).  The direct store costs
// (C+1) row strides of HBM; when that exceeds a quarter of the free device memory the scan
// stays on the map (mode 0).
ara_status build_direct(ara_ctx *ctx)
{
    ara::DeviceStore &st = ctx->store;
    int mode = 2;
    if (const char *m = getenv("ARA_MAP_MODE")) mode = atoi(m);
    // row indices (ids and the zero-row block after them) stay below 2^32 - 1 (pin)
    if ((mode != 1 && mode != 2) || ctx->C > 0xfffffffeu - ara::kZeroRows - 1) return ARA_OK;
    const bool uni = st.uni.enabled;
    const size_t row_bytes = uni ? (size_t)8 * 8 * st.uni.GU
                                 : (size_t)st.n_layers * st.width * (st.bits / 8);
    const size_t bytes = ((size_t)ctx->C + 1 + ara::kZeroRows) * row_bytes;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess || bytes > free_b / 4) return ARA_OK;
    void *direct = nullptr;
    cudaError_t e = cudaMalloc(&direct, bytes);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        return ARA_OK;  // stay on the map
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "direct store");
    if (uni)
        st.uni.d_rows_direct = (double *)direct;
    else
        st.d_rows_direct = direct;
    e = ara::launch_expand_rows(st.d_map, ctx->C, uni ? (const void *)st.uni.d_rows : st.d_rows,
                                direct, row_bytes, ctx->stream);
    if (e == cudaSuccess && mode == 2) {
        st.bitmap_log2 = uni ? ara::kBitmapLog2Union : ara::kBitmapLog2Scan;
        e = cudaMalloc(&st.d_bitmap, ara::bitmap_bytes(st.bitmap_log2));
        if (e == cudaSuccess)
            e = ara::launch_build_bitmap(st.d_map, ctx->C, st.d_bitmap, st.bitmap_log2,
                                         ctx->stream);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "direct store");
    st.map_mode = mode;
    st.zero_base_direct = ctx->C + 1;
    st.uni.zero_base_direct = ctx->C + 1;
    ctx->store_bytes += bytes + (mode == 2 ? ara::bitmap_bytes(st.bitmap_log2) : 0);
    return ARA_OK;
}

}  // namespace

extern "C" {

const char *ara_status_string(ara_status s)
{
    switch (s) {
        case ARA_OK: return "ARA_OK";
        case ARA_ERR_ARG: return "ARA_ERR_ARG";
        case ARA_ERR_RANGE: return "ARA_ERR_RANGE";
        case ARA_ERR_VALIDATION: return "ARA_ERR_VALIDATION";
        case ARA_ERR_STATE: return "ARA_ERR_STATE";
        case ARA_ERR_EMPTY: return "ARA_ERR_EMPTY";
        case ARA_ERR_OOM: return "ARA_ERR_OOM";
        case ARA_ERR_CUDA: return "ARA_ERR_CUDA";
        case ARA_ERR_UNSUPPORTED: return "ARA_ERR_UNSUPPORTED";
    }
    return "ARA_ERR_UNKNOWN";
}

ara_status ara_create(int cuda_device, void *cuda_stream, ara_ctx **out)
{
    if (!out) return ARA_ERR_ARG;
    *out = nullptr;
    int n_dev = 0;
    if (cudaGetDeviceCount(&n_dev) != cudaSuccess || cuda_device < 0 || cuda_device >= n_dev)
        return ARA_ERR_CUDA;
    ara_ctx *ctx = new (std::nothrow) ara_ctx();
    if (!ctx) return ARA_ERR_OOM;
    ctx->device = cuda_device;
    ctx->stream = (cudaStream_t)cuda_stream;
    DeviceGuard g(cuda_device);
    cudaError_t e = cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount,
                                           cuda_device);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->d_err, 4);
    if (e == cudaSuccess) e = cudaMemset(ctx->d_err, 0, 4);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->d_ticket, 16);
    if (e == cudaSuccess) e = cudaMemset(ctx->d_ticket, 0, 16);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->d_probe, 32);
    if (e == cudaSuccess) e = cudaMemset(ctx->d_probe, 0, 32);
    if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_probe, 32);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_probe, cudaEventDisableTiming);
    if (const char *sc = getenv("ARA_SCAN_SCHED"))
        ctx->sched = strcmp(sc, "static") == 0 ? 1 : strcmp(sc, "dynamic") == 0 ? 2 : 0;
    if (const char *pr = getenv("ARA_MAP_PROBE")) ctx->probe = atoi(pr) != 0;
    if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_err, 4);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        e = cudaEventCreateWithFlags(&ctx->ev_copy[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_done[i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        ara_destroy(ctx);
        return e == cudaErrorMemoryAllocation ? ARA_ERR_OOM : ARA_ERR_CUDA;
    }
    *out = ctx;
    return ARA_OK;
}

ara_status ara_set_precision(ara_ctx *ctx, uint32_t bits)
{
    return guarded(ctx, __func__, [&]() -> ara_status {
        if (bits != 32 && bits != 64)
            return fail(ctx, ARA_ERR_ARG, "precision %u bits: 32 or 64 expected", bits);
        if ((int)bits != ctx->bits) {
            ARA_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
            free_layers(ctx);
            ctx->bits = (int)bits;
        }
        return ARA_OK;
    });
}

ara_status ara_set_stream(ara_ctx *ctx, void *cuda_stream)
{
    return guarded(ctx, __func__, [&]() -> ara_status {
        ARA_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        ctx->stream = (cudaStream_t)cuda_stream;
        return ARA_OK;
    });
}

void ara_destroy(ara_ctx *ctx)
{
    if (!ctx) return;
    DeviceGuard g(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    free_layers(ctx);
    cudaFree(ctx->d_err);
    cudaFree(ctx->d_ticket);
    cudaFree(ctx->d_probe);
    cudaFreeHost(ctx->h_probe);
    if (ctx->ev_probe) cudaEventDestroy(ctx->ev_probe);
    cudaFreeHost(ctx->h_err);
    cudaFree(ctx->metrics.d_buf);
    cudaFree(ctx->metrics.d_shard);
    cudaFree(ctx->ep.d_buf);
    cudaFree(ctx->sort.d_buf);
    for (int i = 0; i < 2; ++i) {
        cudaFree(ctx->d_ids_stage[i]);
        cudaFree(ctx->d_off_stage[i]);
        if (ctx->ev_copy[i]) cudaEventDestroy(ctx->ev_copy[i]);
        if (ctx->ev_done[i]) cudaEventDestroy(ctx->ev_done[i]);
    }
    cudaFree(ctx->d_ylt_stage);
    cudaFree(ctx->d_row_stage);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    delete ctx;
}

const char *ara_last_error(const ara_ctx *ctx) { return ctx ? ctx->err.c_str() : "NULL context"; }

ara_status ara_load_elts(ara_ctx *ctx, uint32_t catalogue_size, uint32_t n_elts,
                         const uint64_t *rec_offsets, const uint32_t *rec_event_ids,
                         const double *rec_losses, const ara_fin_terms *fin)
{
    return guarded(ctx, __func__, [&]() -> ara_status {
        if (catalogue_size == 0 || catalogue_size == UINT32_MAX)
            return fail(ctx, ARA_ERR_ARG, "catalogue_size %u outside [1, 2^32-2]", catalogue_size);
        if (n_elts == 0) return fail(ctx, ARA_ERR_ARG, "n_elts is 0");
        if (!rec_offsets || !fin) return fail(ctx, ARA_ERR_ARG, "rec_offsets or fin is NULL");
        for (uint32_t j = 0; j < n_elts; ++j)
            if (rec_offsets[j + 1] < rec_offsets[j])
                return fail(ctx, ARA_ERR_VALIDATION, "rec_offsets decrease at ELT %u", j);
        const uint64_t base = rec_offsets[0];
        const uint64_t n_rec = rec_offsets[n_elts] - base;
        if (n_rec && (!rec_event_ids || !rec_losses))
            return fail(ctx, ARA_ERR_ARG, "record arrays are NULL");
        for (uint32_t j = 0; j < n_elts; ++j) {
            const ara_fin_terms &f = fin[j];
            if (!(isfinite(f.rate) && f.rate > 0.0))
                return fail(ctx, ARA_ERR_VALIDATION, "ELT %u: rate %g is not finite and > 0", j,
                            f.rate);
            if (!finite_nonneg(f.retention))
                return fail(ctx, ARA_ERR_VALIDATION, "ELT %u: retention %g is not finite and >= 0",
                            j, f.retention);
            if (!limit_ok(f.limit))
                return fail(ctx, ARA_ERR_VALIDATION, "ELT %u: limit %g is not >= 0 (or +inf)", j,
                            f.limit);
        }
        std::vector<uint32_t> stamp((size_t)catalogue_size + 1, 0);
        for (uint32_t j = 0; j < n_elts; ++j) {
            for (uint64_t r = rec_offsets[j] - base; r < rec_offsets[j + 1] - base; ++r) {
                const uint32_t id = rec_event_ids[r];
                if (id == 0 || id > catalogue_size)
                    return fail(ctx, ARA_ERR_RANGE,
                                "ELT %u record %llu: event id %u outside [1, %u]", j,
                                (unsigned long long)(r - (rec_offsets[j] - base)), id,
                                catalogue_size);
                if (stamp[id] == j + 1)
                    return fail(ctx, ARA_ERR_VALIDATION, "ELT %u: duplicate event id %u", j, id);
                stamp[id] = j + 1;
                if (!finite_nonneg(rec_losses[r]))
                    return fail(ctx, ARA_ERR_VALIDATION,
                                "ELT %u record %llu: loss %g is not finite and >= 0", j,
                                (unsigned long long)(r - (rec_offsets[j] - base)), rec_losses[r]);
            }
        }
        ARA_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        free_layers(ctx);
        ctx->C = catalogue_size;
        ctx->n_elts = n_elts;
        ctx->rec_off.assign(rec_offsets, rec_offsets + n_elts + 1);
        for (auto &o : ctx->rec_off) o -= base;
        ctx->rec_ids.assign(rec_event_ids, rec_event_ids + n_rec);
        ctx->rec_losses.assign(rec_losses, rec_losses + n_rec);
        ctx->fin.assign(fin, fin + n_elts);
        ctx->have_elts = true;
        return ARA_OK;
    });
}

ara_status ara_set_layers(ara_ctx *ctx, uint32_t n_layers, const ara_layer_terms *terms,
                          const uint32_t *elt_offsets, const uint32_t *elt_index)
{
    return guarded(ctx, __func__, [&]() -> ara_status {
        if (!ctx->have_elts) return fail(ctx, ARA_ERR_STATE, "ara_load_elts has not succeeded");
        if (n_layers == 0) return fail(ctx, ARA_ERR_ARG, "n_layers is 0");
        if (!terms || !elt_offsets || !elt_index)
            return fail(ctx, ARA_ERR_ARG, "terms, elt_offsets or elt_index is NULL");
        std::vector<uint32_t> stamp(ctx->n_elts, 0);
        for (uint32_t l = 0; l < n_layers; ++l) {
            const ara_layer_terms &t = terms[l];
            if (!finite_nonneg(t.occ_retention) || !finite_nonneg(t.agg_retention))
                return fail(ctx, ARA_ERR_VALIDATION, "layer %u: retentions must be finite and >= 0",
                            l);
            if (!limit_ok(t.occ_limit) || !limit_ok(t.agg_limit))
                return fail(ctx, ARA_ERR_VALIDATION, "layer %u: limits must be >= 0 (or +inf)", l);
            if (elt_offsets[l + 1] < elt_offsets[l])
                return fail(ctx, ARA_ERR_VALIDATION, "elt_offsets decrease at layer %u", l);
            const uint32_t E = elt_offsets[l + 1] - elt_offsets[l];
            if (E == 0) return fail(ctx, ARA_ERR_VALIDATION, "layer %u covers no ELT", l);
            if (E > ARA_MAX_ELTS_PER_LAYER)
                return fail(ctx, ARA_ERR_UNSUPPORTED, "layer %u covers %u ELTs (max %d)", l, E,
                            ARA_MAX_ELTS_PER_LAYER);
            for (uint32_t c = elt_offsets[l]; c < elt_offsets[l + 1]; ++c) {
                const uint32_t j = elt_index[c];
                if (j >= ctx->n_elts)
                    return fail(ctx, ARA_ERR_VALIDATION, "layer %u: ELT index %u >= n_elts %u", l,
                                j, ctx->n_elts);
                if (stamp[j] == l + 1)
                    return fail(ctx, ARA_ERR_VALIDATION, "layer %u lists ELT %u twice", l, j);
                stamp[j] = l + 1;
            }
        }
        ARA_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        free_layers(ctx);

        // A1: union of all layers' events (ascending id -> dense rows 1..U), one shared map, and
        // event-major rows holding each layer's columns back to back (layer l at l * W).
        const uint32_t C = ctx->C;
        ara::DeviceStore &st = ctx->store;
        st.n_layers = n_layers;
        uint32_t maxE = 0;
        for (uint32_t l = 0; l < n_layers; ++l) {
            st.n_cols.push_back(elt_offsets[l + 1] - elt_offsets[l]);
            maxE = std::max(maxE, st.n_cols.back());
        }
        st.bits = ctx->bits;
        if (const char *g = getenv("ARA_SCAN_GROUP")) st.group_override = atoi(g);
        if (const char *m = getenv("ARA_SCAN_MINB")) st.min_blocks = atoi(m);
        if (const char *d = getenv("ARA_SCAN_DEPTH")) st.depth = atoi(d);
        if (const char *q = getenv("ARA_PAIR_SCAN")) st.pair_scan = atoi(q) != 0;
        if (const char *q = getenv("ARA_PAIR_WIDE")) st.pair_wide = atoi(q) != 0;
        if (const char *q = getenv("ARA_PAIR_G2")) st.pair_g2 = atoi(q) != 0;
        if (const char *q = getenv("ARA_PAIR_EV2")) st.pair_ev2 = atoi(q) != 0;
        st.scaled = ctx->bits == 64 && scaled_terms_ok(ctx, n_layers, terms, elt_offsets,
                                                       elt_index);
        uint32_t W = ctx->bits == 32 ? ara::row_width_for_f32(maxE) : ara::row_width_for(maxE);
        // 17-24 ELTs: 24-column rows for the 3-lane pair scan instead of padding to 32 (only
        // that kernel reads them; the compare-select scan.cu serves W = 32)
        if (W == 32 && maxE <= 24 && st.scaled && st.pair_scan && ctx->sched != 1) W = 24;
        st.width = W;
        // lanes per trial of the kernel that reads the rows (the interleave, ara_internal.h):
        // W >= 32 four lanes (ARA_PAIR_G2=1, tuning: 25-32 ELTs on the 2-lane pair scan)
        st.ilv = (ctx->bits != 64 || W <= 16) ? 0
                 : W == 24                     ? 3
                 : (W == 32 && st.scaled && st.pair_scan && st.pair_g2 && ctx->sched != 1) ? 2
                                               : 4;
        std::vector<uint32_t> map((size_t)C + 1, 0u);
        std::vector<uint32_t> uni;
        for (uint32_t c = elt_offsets[0]; c < elt_offsets[n_layers]; ++c) {
            const uint32_t j = elt_index[c];
            for (uint64_t r = ctx->rec_off[j]; r < ctx->rec_off[j + 1]; ++r) {
                const uint32_t id = ctx->rec_ids[r];
                if (!map[id]) {
                    map[id] = 1;
                    uni.push_back(id);
                }
            }
        }
        std::sort(uni.begin(), uni.end());
        st.n_union = (uint32_t)uni.size();
        st.zero_base = st.n_union + 1;
        for (uint32_t u = 0; u < st.n_union; ++u) map[uni[u]] = u + 1;
        size_t row_bytes = 0, term_bytes = 0;
        std::vector<char> rows_buf, terms_buf;
        if (ctx->bits == 32)
            build_rows<float>(ctx, st, map, terms, elt_offsets, elt_index, rows_buf, terms_buf);
        else
            build_rows<double>(ctx, st, map, terms, elt_offsets, elt_index, rows_buf, terms_buf);
        row_bytes = rows_buf.size();
        term_bytes = terms_buf.size();
        const size_t map_bytes = ((size_t)C + 1) * 4;
        cudaError_t e = cudaMalloc(&st.d_map, map_bytes);
        if (e == cudaSuccess) e = cudaMalloc(&st.d_rows, row_bytes);
        if (e == cudaSuccess) e = cudaMalloc(&st.d_terms, term_bytes);
        if (e == cudaSuccess) e = cudaMemcpy(st.d_map, map.data(), map_bytes, cudaMemcpyHostToDevice);
        if (e == cudaSuccess)
            e = cudaMemcpy(st.d_rows, rows_buf.data(), row_bytes, cudaMemcpyHostToDevice);
        if (e == cudaSuccess)
            e = cudaMemcpy(st.d_terms, terms_buf.data(), term_bytes, cudaMemcpyHostToDevice);
        if (e == cudaSuccess && st.n_union)
            e = cudaMalloc(&st.d_union_ids, (size_t)st.n_union * 4);
        if (e == cudaSuccess && st.n_union)
            e = cudaMemcpy(st.d_union_ids, uni.data(), (size_t)st.n_union * 4,
                           cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            free_layers(ctx);
            return cuda_fail(ctx, e, "device ELT store");
        }
        ctx->store_bytes = map_bytes + row_bytes + term_bytes;
        ara_status us = build_union(ctx, map, terms, elt_offsets, elt_index);
        if (us == ARA_OK) us = build_direct(ctx);
        if (us != ARA_OK) {
            free_layers(ctx);
            return us;
        }
        ctx->have_layers = true;
        return ARA_OK;
    });
}

ara_status ara_run_outputs(ara_ctx *ctx, uint64_t n_trials, const uint64_t *d_trial_offsets,
                           const uint32_t *d_event_ids, const ara_outputs *out, uint32_t flags)
{
    return guarded(ctx, __func__, [&]() -> ara_status {
        if (!ctx->have_layers) return fail(ctx, ARA_ERR_STATE, "ara_set_layers has not succeeded");
        if (flags & ~(ARA_RUN_SYNC | ARA_RUN_VALIDATE | ARA_RUN_BALANCE | ARA_RUN_HOIST))
            return fail(ctx, ARA_ERR_ARG, "unknown flags 0x%x", flags);
        if (!out) return fail(ctx, ARA_ERR_ARG, "outputs is NULL");
        if (n_trials == 0) return ARA_OK;
        if (!d_trial_offsets || !d_event_ids || !out->ylt)
            return fail(ctx, ARA_ERR_ARG, "device pointer is NULL");
        ara_outputs o = *out;
        if (!o.ylt_ld) o.ylt_ld = n_trials;
        if (!o.max_occ_ld) o.max_occ_ld = n_trials;
        if (o.ylt_ld < n_trials || (o.max_occ && o.max_occ_ld < n_trials))
            return fail(ctx, ARA_ERR_ARG, "leading dimension < n_trials");
        // the YET's event count (increments, validation): two 8-byte reads of the offsets
        uint64_t ends[2] = {0, 0};
        if (o.event_inc || (flags & ARA_RUN_VALIDATE)) {
            ARA_CUDA(ctx, cudaMemcpyAsync(&ends[0], d_trial_offsets, 8, cudaMemcpyDeviceToHost,
                                          ctx->stream));
            ARA_CUDA(ctx, cudaMemcpyAsync(&ends[1], d_trial_offsets + n_trials, 8,
                                          cudaMemcpyDeviceToHost, ctx->stream));
            ARA_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
            if (ends[1] < ends[0])
                return fail(ctx, ARA_ERR_VALIDATION,
                            "trial offsets decrease (offsets[n] = %llu < offsets[0] = %llu)",
                            (unsigned long long)ends[1], (unsigned long long)ends[0]);
        }
        if (o.event_inc) {
            const uint64_t n_ev = ends[1] - ends[0];
            if (!o.event_inc_ld) o.event_inc_ld = n_ev;
            if (o.event_inc_ld < n_ev)
                return fail(ctx, ARA_ERR_ARG, "event_inc_ld %llu < %llu events",
                            (unsigned long long)o.event_inc_ld, (unsigned long long)n_ev);
        }
        if (flags & ARA_RUN_VALIDATE) {
            ara_status s = check_device_error(ctx);  // report earlier deferred errors first
            if (s != ARA_OK) return s;
            cudaError_t e = ara::launch_validate(d_trial_offsets, d_event_ids, n_trials,
                                                 ends[1] - ends[0], ctx->C, ctx->d_err,
                                                 ctx->sm_count, ctx->stream, &ctx->launches);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "validate kernel launch");
            s = check_device_error(ctx);
            if (s != ARA_OK) return s;
        }
        const bool extra = o.max_occ || o.event_inc;
        if ((flags & ARA_RUN_HOIST) && !extra) {
            ara_status h = prepare_hoist(ctx);
            if (h != ARA_OK) return h;
        }
        ara_status s = launch_layers(ctx, n_trials, d_trial_offsets, d_event_ids, o.ylt, o.ylt_ld,
                                     flags, extra ? &o : nullptr);
        if (s != ARA_OK) return s;
        if (flags & (ARA_RUN_SYNC | ARA_RUN_VALIDATE)) return check_device_error(ctx);
        return ARA_OK;
    });
}

ara_status ara_run(ara_ctx *ctx, uint64_t n_trials, const uint64_t *d_trial_offsets,
                   const uint32_t *d_event_ids, double *d_ylt, uint64_t ylt_ld, uint32_t flags)
{
    const ara_outputs o{d_ylt, ylt_ld, nullptr, 0, nullptr, 0};
    return ara_run_outputs(ctx, n_trials, d_trial_offsets, d_event_ids, &o, flags);
}

ara_status ara_synchronize(ara_ctx *ctx)
{
    return guarded(ctx, __func__, [&]() -> ara_status {
        ARA_CUDA(ctx, cudaGetLastError());
        return check_device_error(ctx);
    });
}

ara_status ara_run_host(ara_ctx *ctx, uint64_t n_trials, const uint64_t *h_trial_offsets,
                        const uint32_t *h_event_ids, double *h_ylt, uint64_t ylt_ld,
                        uint32_t flags)
{
    return guarded(ctx, __func__, [&]() -> ara_status {
        if (!ctx->have_layers) return fail(ctx, ARA_ERR_STATE, "ara_set_layers has not succeeded");
        if (flags & ~(ARA_RUN_SYNC | ARA_RUN_VALIDATE | ARA_RUN_BALANCE | ARA_RUN_HOIST))
            return fail(ctx, ARA_ERR_ARG, "unknown flags 0x%x", flags);
        if (n_trials == 0) return ARA_OK;
        if (!h_trial_offsets || !h_ylt) return fail(ctx, ARA_ERR_ARG, "host pointer is NULL");
        const uint64_t ld = ylt_ld ? ylt_ld : n_trials;
        if (ld < n_trials) return fail(ctx, ARA_ERR_ARG, "ylt_ld < n_trials");
        // one pass over the offsets: monotonicity and the longest trial (sizes the staging)
        uint64_t max_trial = 0;
        for (uint64_t t = 0; t < n_trials; ++t) {
            if (h_trial_offsets[t + 1] < h_trial_offsets[t])
                return fail(ctx, ARA_ERR_VALIDATION, "trial offsets decrease at trial %llu",
                            (unsigned long long)t);
            max_trial = std::max<uint64_t>(max_trial, h_trial_offsets[t + 1] - h_trial_offsets[t]);
        }
        const uint64_t base = h_trial_offsets[0];
        if (h_trial_offsets[n_trials] > base && !h_event_ids)
            return fail(ctx, ARA_ERR_ARG, "h_event_ids is NULL");
        ara_status s = check_device_error(ctx);
        if (s != ARA_OK) return s;

        const size_t n_layers = ctx->store.n_layers;
        // device YLT staging
        if (ctx->ylt_stage_cap < n_layers * n_trials) {
            cudaFree(ctx->d_ylt_stage);
            ctx->d_ylt_stage = nullptr;
            ctx->ylt_stage_cap = 0;
            ARA_CUDA(ctx, cudaMalloc(&ctx->d_ylt_stage, n_layers * n_trials * 8));
            ctx->ylt_stage_cap = n_layers * n_trials;
        }
        if (flags & ARA_RUN_HOIST) {  // the per-event table once for all chunks
            s = prepare_hoist(ctx);
            if (s != ARA_OK) return s;
        }
        // chunking at trial boundaries: ~64 MiB of ids per chunk (>= 1 trial)
        const size_t kChunkIds = (size_t)16 << 20;
        const size_t ids_cap = std::max<size_t>(kChunkIds, max_trial);
        const size_t off_cap = ids_cap + 2;  // a chunk holds at most ids_cap non-empty trials...
        if (ctx->ids_stage_cap < ids_cap || ctx->off_stage_cap < off_cap) {
            for (int i = 0; i < 2; ++i) {
                cudaFree(ctx->d_ids_stage[i]);
                cudaFree(ctx->d_off_stage[i]);
                ctx->d_ids_stage[i] = nullptr;
                ctx->d_off_stage[i] = nullptr;
            }
            ctx->ids_stage_cap = ctx->off_stage_cap = 0;
            for (int i = 0; i < 2; ++i) {
                ARA_CUDA(ctx, cudaMalloc(&ctx->d_ids_stage[i], ids_cap * 4));
                ARA_CUDA(ctx, cudaMalloc(&ctx->d_off_stage[i], off_cap * 8));
            }
            ctx->ids_stage_cap = ids_cap;
            ctx->off_stage_cap = off_cap;
        }
        // ... and at most off_cap - 1 trials (empty trials)
        uint64_t t0 = 0;
        int buf = 0;
        bool used[2] = {false, false};
        while (t0 < n_trials) {
            uint64_t t1 = t0 + 1;
            while (t1 < n_trials && t1 - t0 < off_cap - 1 &&
                   h_trial_offsets[t1 + 1] - h_trial_offsets[t0] <= ids_cap)
                ++t1;
            const uint64_t n_ev = h_trial_offsets[t1] - h_trial_offsets[t0];
            if (used[buf]) ARA_CUDA(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_done[buf], 0));
            ARA_CUDA(ctx, cudaMemcpyAsync(ctx->d_off_stage[buf], h_trial_offsets + t0,
                                          (t1 - t0 + 1) * 8, cudaMemcpyHostToDevice,
                                          ctx->copy_stream));
            if (n_ev)
                ARA_CUDA(ctx, cudaMemcpyAsync(ctx->d_ids_stage[buf],
                                              h_event_ids + (h_trial_offsets[t0] - base),
                                              n_ev * 4, cudaMemcpyHostToDevice, ctx->copy_stream));
            ARA_CUDA(ctx, cudaEventRecord(ctx->ev_copy[buf], ctx->copy_stream));
            ARA_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_copy[buf], 0));
            if (flags & ARA_RUN_VALIDATE) {  // ids of this chunk (the offsets were checked above)
                cudaError_t e = ara::launch_validate(ctx->d_off_stage[buf], ctx->d_ids_stage[buf],
                                                     t1 - t0, n_ev, ctx->C, ctx->d_err,
                                                     ctx->sm_count, ctx->stream, &ctx->launches);
                if (e != cudaSuccess) return cuda_fail(ctx, e, "validate kernel launch");
            }
            s = launch_layers(ctx, t1 - t0, ctx->d_off_stage[buf], ctx->d_ids_stage[buf],
                              ctx->d_ylt_stage + t0, n_trials, flags);
            if (s != ARA_OK) return s;
            ARA_CUDA(ctx, cudaEventRecord(ctx->ev_done[buf], ctx->stream));
            used[buf] = true;
            buf ^= 1;
            t0 = t1;
        }
        // device errors (ids out of range) are reported before anything reaches h_ylt
        s = check_device_error(ctx);
        if (s != ARA_OK) return s;
        ARA_CUDA(ctx, cudaMemcpy2DAsync(h_ylt, ld * 8, ctx->d_ylt_stage, n_trials * 8,
                                        n_trials * 8, n_layers, cudaMemcpyDeviceToHost,
                                        ctx->stream));
        ARA_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        return ARA_OK;
    });
}

ara_status ara_ep_curve(ara_ctx *ctx, const double *d_row, uint64_t n, double *d_curve)
{
    return guarded(ctx, __func__, [&]() -> ara_status {
        if (n == 0) return fail(ctx, ARA_ERR_EMPTY, "n is 0");
        if (!d_row || !d_curve) return fail(ctx, ARA_ERR_ARG, "device pointer is NULL");
        if (d_row < d_curve + n && d_curve < d_row + n)
            return fail(ctx, ARA_ERR_ARG, "d_row and d_curve overlap");
        cudaError_t e = ara::launch_ep_curve(d_row, n, d_curve, ctx->ep, ctx->sm_count,
                                             ctx->stream, &ctx->launches);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "exceedance curve");
        return ARA_OK;
    });
}

ara_status ara_metrics(ara_ctx *ctx, const double *d_ylt_row, uint64_t n, uint32_t n_p,
                       const double *p, double *pml_out, double *tvar_out)
{
    return guarded(ctx, __func__, [&]() -> ara_status {
        if (n == 0) return fail(ctx, ARA_ERR_EMPTY, "metrics over zero trials");
        ara_status s = validate_p(ctx, n_p, p);
        if (s != ARA_OK) return s;
        if (!d_ylt_row || !pml_out || !tvar_out) return fail(ctx, ARA_ERR_ARG, "NULL pointer");
        cudaError_t e = ara::launch_metrics(d_ylt_row, n, 1, n, n_p, p, pml_out, tvar_out,
                                            ctx->metrics, ctx->sm_count, ctx->device, ctx->stream,
                                            &ctx->launches);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "metrics kernel");
        return ARA_OK;
    });
}

ara_status ara_metrics_rows(ara_ctx *ctx, const double *d_rows, uint32_t n_rows, uint64_t ld,
                            uint64_t n, uint32_t n_p, const double *p, double *pml_out,
                            double *tvar_out)
{
    return guarded(ctx, __func__, [&]() -> ara_status {
        if (n == 0) return fail(ctx, ARA_ERR_EMPTY, "metrics over zero trials");
        ara_status s = validate_p(ctx, n_p, p);
        if (s != ARA_OK) return s;
        if (n_rows == 0) return ARA_OK;
        if (!d_rows || !pml_out || !tvar_out) return fail(ctx, ARA_ERR_ARG, "NULL pointer");
        const uint64_t stride = ld ? ld : n;
        if (stride < n) return fail(ctx, ARA_ERR_ARG, "ld < n");
        cudaError_t e = ara::launch_metrics(d_rows, stride, n_rows, n, n_p, p, pml_out, tvar_out,
                                            ctx->metrics, ctx->sm_count, ctx->device, ctx->stream,
                                            &ctx->launches);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "metrics kernel");
        return ARA_OK;
    });
}

ara_status ara_portfolio_ylt(ara_ctx *ctx, const double *d_ylt, uint64_t n_trials,
                             uint64_t ylt_ld, double *d_out, uint32_t flags)
{
    return guarded(ctx, __func__, [&]() -> ara_status {
        if (!ctx->have_layers) return fail(ctx, ARA_ERR_STATE, "ara_set_layers has not succeeded");
        if (flags & ~ARA_RUN_SYNC) return fail(ctx, ARA_ERR_ARG, "unknown flags 0x%x", flags);
        if (n_trials == 0) return ARA_OK;
        if (!d_ylt || !d_out) return fail(ctx, ARA_ERR_ARG, "device pointer is NULL");
        const uint64_t ld = ylt_ld ? ylt_ld : n_trials;
        if (ld < n_trials) return fail(ctx, ARA_ERR_ARG, "ylt_ld < n_trials");
        cudaError_t e = ara::launch_portfolio_row(d_ylt, ctx->store.n_layers, n_trials, ld, d_out,
                                                  ctx->sm_count, ctx->stream, &ctx->launches);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "portfolio row kernel");
        if (flags & ARA_RUN_SYNC) ARA_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        return ARA_OK;
    });
}

ara_status ara_metrics_sharded(ara_ctx *ctx, const double *d_ylt_slice, uint64_t n_local,
                               uint64_t n_global, uint32_t n_p, const double *p, double *pml_out,
                               double *tvar_out, void *d_xbuf, uint64_t xbuf_bytes,
                               ara_shard_reduce reduce, void *user)
{
    return guarded(ctx, __func__, [&]() -> ara_status {
        if (n_global == 0) return fail(ctx, ARA_ERR_EMPTY, "metrics over zero trials");
        ara_status s = validate_p(ctx, n_p, p);
        if (s != ARA_OK) return s;
        if ((n_local && !d_ylt_slice) || !pml_out || !tvar_out || !d_xbuf || !reduce)
            return fail(ctx, ARA_ERR_ARG, "NULL pointer");
        if (n_local > n_global) return fail(ctx, ARA_ERR_ARG, "n_local > n_global");
        if (xbuf_bytes < (uint64_t)ARA_MAX_P * 256 * 8)
            return fail(ctx, ARA_ERR_ARG, "exchange buffer smaller than %d bytes",
                        ARA_MAX_P * 256 * 8);
        cudaError_t e = ara::launch_metrics_sharded(
            d_ylt_slice, n_local, n_global, n_p, p, pml_out, tvar_out, (char *)d_xbuf,
            (ara::ShardReduce)reduce, user, ctx->metrics, ctx->sm_count, ctx->stream,
            &ctx->launches);
        if (e == cudaErrorUnknown) return fail(ctx, ARA_ERR_ARG, "the reduction callback failed");
        if (e != cudaSuccess) return cuda_fail(ctx, e, "sharded metrics");
        return ARA_OK;
    });
}

ara_status ara_metrics_host(ara_ctx *ctx, const double *h_ylt_row, uint64_t n, uint32_t n_p,
                            const double *p, double *pml_out, double *tvar_out)
{
    return guarded(ctx, __func__, [&]() -> ara_status {
        if (n == 0) return fail(ctx, ARA_ERR_EMPTY, "metrics over zero trials");
        ara_status s = validate_p(ctx, n_p, p);
        if (s != ARA_OK) return s;
        if (!h_ylt_row || !pml_out || !tvar_out) return fail(ctx, ARA_ERR_ARG, "NULL pointer");
        if (ctx->row_stage_cap < n) {
            cudaFree(ctx->d_row_stage);
            ctx->d_row_stage = nullptr;
            ctx->row_stage_cap = 0;
            ARA_CUDA(ctx, cudaMalloc(&ctx->d_row_stage, n * 8));
            ctx->row_stage_cap = n;
        }
        ARA_CUDA(ctx, cudaMemcpyAsync(ctx->d_row_stage, h_ylt_row, n * 8, cudaMemcpyHostToDevice,
                                      ctx->stream));
        cudaError_t e = ara::launch_metrics(ctx->d_row_stage, n, 1, n, n_p, p, pml_out, tvar_out,
                                            ctx->metrics, ctx->sm_count, ctx->device,
                                            ctx->stream, &ctx->launches);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "metrics kernel");
        return ARA_OK;
    });
}

ara_status ara_get_info(const ara_ctx *ctx, ara_info *out)
{
    if (!ctx || !out) return ARA_ERR_ARG;
    out->catalogue_size = ctx->C;
    out->n_elts = ctx->n_elts;
    out->n_layers = ctx->have_layers ? ctx->store.n_layers : 0;
    out->max_row_width = ctx->have_layers ? ctx->store.width : 0;
    out->store_bytes = ctx->store_bytes;
    out->kernel_launches = ctx->launches;
    out->device = ctx->device;
    out->sm_count = ctx->sm_count;
    out->row_addressing = ctx->have_layers ? ctx->store.map_mode : 0;
    out->layer_kernel = !ctx->have_layers || !ctx->store.uni.enabled ? 0
                        : ctx->store.uni.shfl == 3 ? 3 : 1 + (ctx->store.uni.shfl != 0);
    out->gather_row_bytes = !ctx->have_layers ? 0
                            : ctx->store.uni.enabled
                                ? 8 * 8 * ctx->store.uni.GU
                                : ctx->store.n_layers * ctx->store.width * (ctx->store.bits / 8);
    snprintf(out->last_kernel, sizeof(out->last_kernel), "%s", ctx->last_kernel.c_str());
    return ARA_OK;
}

ara_status ara_layer_store_shape(const ara_ctx *ctx, uint32_t layer, uint32_t *n_union,
                                 uint32_t *row_width)
{
    if (!ctx) return ARA_ERR_ARG;
    if (!ctx->have_layers) return ARA_ERR_STATE;
    if (layer >= ctx->store.n_layers) return ARA_ERR_ARG;
    if (n_union) *n_union = ctx->store.n_union;
    if (row_width) *row_width = ctx->store.width;
    return ARA_OK;
}

ara_status ara_export_store(ara_ctx *ctx, uint32_t layer, uint32_t *h_map, double *h_rows)
{
    return guarded(ctx, __func__, [&]() -> ara_status {
        if (!ctx->have_layers) return fail(ctx, ARA_ERR_STATE, "no layers");
        const ara::DeviceStore &st = ctx->store;
        if (layer >= st.n_layers) return fail(ctx, ARA_ERR_ARG, "layer %u out of range", layer);
        ARA_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        if (h_map)
            ARA_CUDA(ctx, cudaMemcpy(h_map, st.d_map, ((size_t)ctx->C + 1) * 4, cudaMemcpyDeviceToHost));
        if (h_rows) {  // this layer's W columns of every union row, widened to double
            const size_t es = st.bits == 32 ? 4 : 8;
            std::vector<char> tmp((size_t)(st.n_union + 1) * st.width * es);
            ARA_CUDA(ctx, cudaMemcpy2D(tmp.data(), (size_t)st.width * es,
                                       (const char *)st.d_rows + (size_t)layer * st.width * es,
                                       (size_t)st.n_layers * st.width * es, (size_t)st.width * es,
                                       st.n_union + 1, cudaMemcpyDeviceToHost));
            // logical column order (the device rows of W >= 32 are lane-interleaved)
            for (size_t u = 0; u <= st.n_union; ++u)
                for (uint32_t j = 0; j < st.width; ++j) {
                    const size_t i = u * st.width + ara::row_phys_col(j, st.width, st.ilv);
                    h_rows[u * st.width + j] = st.bits == 32
                                                   ? (double)((const float *)tmp.data())[i]
                                                   : ((const double *)tmp.data())[i];
                }
        }
        return ARA_OK;
    });
}

}  // extern "C"
