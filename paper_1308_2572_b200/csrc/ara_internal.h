// ara_internal.h -- shared declarations of libara's host code (ara.cpp) and kernels
// (scan.cu, metrics.cu).  Not installed; the public ABI is include/ara.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

#include "ara.h"

namespace ara {

constexpr int kMaxCols = ARA_MAX_ELTS_PER_LAYER;  // row width limit W (doubles)

// Per-layer terms in device memory, one record per layer; every lane copies its own columns'
// financial terms and its layer's occurrence / aggregate terms into registers at kernel start.
// Padded columns j >= E carry the neutral terms (rate 1, retention 0, limit +inf) and zero
// losses, so F_j = +0 and lo + (+0) = lo exactly (reading R12).
template <typename R>
struct LayerTermsT {
    R rate[kMaxCols];
    R ret[kMaxCols];
    R lim[kMaxCols];
    R occ_ret, occ_lim, agg_ret, agg_lim;
};
using LayerTermsDev = LayerTermsT<double>;

// Scan decomposition for a row width: G lanes per trial, each owning CH 32-byte chunks
// (4 doubles each), W = 4 * G * CH.  The paper's 15-16 ELT layers give W = 16 and G = 2: a
// 128-byte row is gathered by two lanes (two 256-bit loads each) and the ELT-sum chain has one
// shuffle hop.  Measured on B200 at the headline (profiles/r1_tune_scan.jsonl): G = 2 12.9 ms,
// G = 4 17.2 ms (3 hops: issue-bound), G = 1 22.9 ms (uncoalesced gathers: L1-request-bound).
struct ScanShape {
    int G, CH;
};

// Row width (elements) of the event-major store for a layer of E ELTs: whole 32-byte chunks.
// fp32 store (F3): 8 floats per chunk -> 8, 16, 32 or 64.
inline uint32_t row_width_for_f32(uint32_t E)
{
    const uint32_t nc = (E + 7) / 8;
    return nc <= 1 ? 8 : nc == 2 ? 16 : nc <= 4 ? 32 : 64;
}

// fp64 store: 4 doubles per chunk.
inline uint32_t row_width_for(uint32_t E)
{
    const uint32_t nc = (E + 3) / 4;  // 32-byte chunks needed
    if (nc <= 1) return 4;
    if (nc == 2) return 8;
    return 16 * ((nc + 3) / 4);       // multiples of 16 doubles
}

// Column order inside a layer's W-element row segment (DeviceStore::ilv).  ilv = 0 (W <= 16, and
// every fp32 store): logical, column j at j.  ilv = g > 0 (fp64 stores of W >= 24): LANE-
// INTERLEAVED for the kernel that reads the store with g lanes per trial, lane c owning the
// CH = W / (4 g) logical 32-byte chunks [CH c, CH c + CH) (4 columns each, in ELT-sum order):
// physical chunk k g + c holds lane c's k-th chunk.  A group's k-th 256-bit load instruction then
// reads g contiguous chunks (a whole 128-byte line for g = 4) instead of one sector in each of g
// lines: 1 L1 wavefront and 1 L2 request per line instead of g (W = 64: 4 instead of 16 per
// event; profiles/r2_tune_interleave.jsonl).  g = 3 for W = 24; for W = 32, 2 when the 2-lane
// pair scan reads it, else 4; g = 4 for W = 48, 64.
__host__ __device__ inline uint32_t row_phys_col(uint32_t j, uint32_t W, uint32_t ilv)
{
    if (ilv == 0) return j;
    const uint32_t ch = W / (4 * ilv);                 // chunks per lane
    const uint32_t c = j / (4 * ch), k = (j / 4) % ch;  // owning lane, its chunk
    return 4 * (k * ilv + c) + j % 4;
}

// Decomposition for a store of width W; override (1, 2 or 4) selects G for W = 16 only.
inline ScanShape scan_shape_for_width(uint32_t W, int override_g)
{
    if (W == 4) return {1, 1};
    if (W == 8) return {2, 1};
    if (W == 16) {
        if (override_g == 1 || override_g == 4) return {override_g, 4 / override_g};
        return {2, 2};
    }
    return {4, (int)(W / 16)};
}

// Union-row store for multi-layer portfolios (F1, portfolio.cu): the distinct ELTs J of all
// layers (|J| <= 64) are the columns of one row per event; each layer lists its columns in its
// own summation order.  Used when 2 <= n_layers <= 8, every layer has <= 16 ELTs and the store is
// fp64; otherwise the per-layer rows below serve the scan.
constexpr int kUnionMaxLayers = 8;
constexpr int kUnionMaxE = 16;
struct UnionTermsDev {
    double rate[kMaxCols], ret[kMaxCols], lim[kMaxCols];  // per union column (padding neutral)
    double occ_ret[kUnionMaxLayers], occ_lim[kUnionMaxLayers];
    double agg_ret[kUnionMaxLayers], agg_lim[kUnionMaxLayers];
    uint32_t slot2[kUnionMaxLayers][kUnionMaxE / 2];  // packed 16-bit shared-memory F slots
    uint32_t n_layers;
    // register-shuffle layout (portfolio.cu, shfl != 0): the F value of a layer's i-th ELT sits
    // in register i mod 8 of lane src(l, i) of the group; src5 packs the 16 source lanes of a
    // layer as 5-bit fields, six per word
    uint32_t src5[kUnionMaxLayers][3];
    // block layout (shfl == 3): layer l's positions 0-7 are registers 0-7 of lane l, positions
    // 8-15 registers 0-7 of lane src2[l]
    uint32_t src2[kUnionMaxLayers];
    uint32_t n_cols[kUnionMaxLayers];    // ELTs of each layer
};
struct UnionStore {
    bool enabled = false;
    double *d_rows_direct = nullptr;     // [(C+1+kZeroRows) * WU] rows by catalogue id (mode >= 1)
    uint32_t zero_base = 0;              // U + 1: zero-row block of d_rows
    uint32_t zero_base_direct = 0;       // C + 1: zero-row block of d_rows_direct
    uint32_t GU = 0;         // lanes per trial (2, 4 or 8); union row width WU = 8 * GU doubles
    int shfl = 0;            // layer sums: 0 = shared-memory F row; 1 = register shuffles
                             // (general); 2 = register shuffles, every layer has 16 ELTs;
                             // 3 = blocks: half of every layer in its own lane's registers
    uint32_t n_cols = 0;     // |J|
    bool scaled = false;     // DeviceStore::scaled (the scaled-clamp instantiation may run)
    double *d_rows = nullptr;            // [(U+1+kZeroRows) * WU]
    UnionTermsDev *d_terms = nullptr;
};

// Device ELT store of all layers: one catalogue map shared by the
// layers and event-major rows that hold every layer's columns back to back, so one id read and
// one map lookup per event serve all layers (F1, the layer-fused portfolio pass).
struct DeviceStore {
    uint32_t n_layers = 0;
    uint32_t n_union = 0;        // U: distinct events over all layers' ELTs
    uint32_t width = 0;          // W = row width (elements) per layer
    int bits = 64;               // 64: fp64 store and arithmetic; 32: fp32 (F3)
    std::vector<uint32_t> n_cols;  // E of each layer
    int group_override = 0;      // tuning: G for W = 16 (env ARA_SCAN_GROUP), 0 = default
    int min_blocks = 0;          // tuning: __launch_bounds__ min blocks (env ARA_SCAN_MINB)
    int depth = 0;               // tuning: rows in flight per group (env ARA_SCAN_DEPTH)
    // scan_pair.cu (fp64, W = 16 / 32): every loss * rate, retention, finite limit and
    // layer term is below 2^960, so the exactly scaled clamps cannot overflow
    bool scaled = false;
    bool pair_scan = true;       // tuning: ARA_PAIR_SCAN=0 runs scan.cu's kernel instead
    bool pair_wide = true;       // tuning: ARA_PAIR_WIDE=0 keeps W = 48 / 64 on scan.cu
    bool pair_g2 = false;        // tuning: ARA_PAIR_G2=1 runs W = 32 on 2 lanes x 16 columns
                                 // (half the chain adds, but 255 registers: 29.3 vs 26.1 ms)
    bool pair_ev2 = true;        // W = 32 / 48 plain scan: two events per step (ARA_PAIR_EV2=0: one)
    uint32_t ilv = 0;            // row layout: 0 logical, g = lane-interleaved for g lanes
    uint32_t *d_map = nullptr;   // [C+1] catalogue id -> row (0 = absent)
    // Row addressing of the scan: 0 = through d_map (dense rows);
    // 1 = direct (rows indexed by catalogue id, no map read); 2 = direct behind a presence
    // bitmap held in shared memory (absent ids read the zero row instead of a cold line).
    int map_mode = 0;
    void *d_rows_direct = nullptr;  // [(C+1+kZeroRows) * n_layers * W]: row id = dense map[id]
    uint32_t *d_bitmap = nullptr;   // [2^bitmap_log2 bits]: bit h(id) set when map[id] != 0
    uint32_t bitmap_log2 = 0;
    void *d_rows = nullptr;      // [(U+1+kZeroRows) * n_layers * W] double or float; row 0 and
                                 // rows U+1.. (the zero-row block) are zero
    uint32_t zero_base = 0;      // U + 1
    uint32_t zero_base_direct = 0;  // C + 1 (d_rows_direct)
    void *d_terms = nullptr;     // [n_layers] LayerTermsT<double or float>
    UnionStore uni;              // F1 union rows (when eligible)
    // hoisted scan (hoist.cu, ARA_RUN_HOIST): per-event layer losses oc[row][l], allocated on
    // the first hoisted run; rows are catalogue ids (oc_direct, map modes 1-2) or dense rows
    uint32_t *d_union_ids = nullptr;  // [U]: dense row u+1 -> catalogue id
    void *d_oc = nullptr;             // [(C+1) or (U+1)] x oc_lp, R; absent rows stay +0
    int oc_direct = 0;
    uint32_t oc_lp = 0;               // layers padded to 1, 2, 4 or 8
    uint32_t *d_oc_bitmap = nullptr;  // map mode 2: 2^kBitmapLog2Hoist-bit presence bitmap
};

// Every row store ends with a block of kZeroRows all-zero rows (at DeviceStore / UnionStore
// zero_base): an absent or out-of-range id reads zero row zero_base + (id mod kZeroRows), so the
// reads of absent events spread over many L2 lines instead of all hitting row 0's line (the row
// gathers bypass L1, so a single shared zero line would be one hot L2 slice).
constexpr uint32_t kZeroRows = 1024;

// Presence bitmap of map mode 2: 2^b bits, bit h(id) = Fibonacci hash of the catalogue id.  A
// clear bit proves the id absent; a set bit may be a collision (then the direct row, all zeros,
// is read).  b = 19 (64 KB of shared memory per block, three blocks per SM) for the scan kernel,
// b = 18 for the union-row kernel (its blocks also hold their F rows in shared memory).
constexpr int kBitmapLog2Scan = 19;
constexpr int kBitmapLog2Union = 18;
constexpr int kBitmapLog2Hoist = 18;  // hoisted scan (hoist.cu): 32 KB, 2 blocks of 512 per SM
__host__ __device__ inline uint32_t bitmap_hash(uint32_t id, uint32_t log2_bits)
{
    return (id * 0x9E3779B1u) >> (32 - log2_bits);
}
inline size_t bitmap_bytes(uint32_t log2_bits) { return (size_t)1 << (log2_bits - 3); }

struct ScanLaunch {
    const uint64_t *offsets;  // [n+1], device
    const uint32_t *ids;      // device, indexed by offsets[t] - offsets[0]
    double *ylt;              // [n_layers][ld], device
    uint64_t ylt_ld;          // YLT row stride (elements)
    uint64_t n_trials;
    uint32_t catalogue_size;
    uint32_t *err;            // device error word (bit 0: id out of range)
    uint32_t zero_base;       // first row of the zero-row block of the rows the kernel reads
    uint32_t bitmap_log2;     // map mode 2: log2 of the presence bitmap's bit count
    unsigned long long *counter;  // dynamic ticket counter (NULL: static assignment)
    unsigned int *done;           // finished-block counter (resets `counter`)
    double *max_occ;              // F4: [n_layers][max_occ_ld] or NULL
    uint64_t max_occ_ld;
    double *event_inc;            // F4: [n_layers][event_inc_ld] or NULL (YET positions)
    uint64_t event_inc_ld;
    const uint32_t *perm;         // length-sorted trial order (ARA_RUN_BALANCE) or NULL
    const unsigned long long *probe;  // map mode 2: hit-probe counts {present, sampled} or NULL
};

// Scratch of the length sort (ARA_RUN_BALANCE): keys, indices, CUB temporary storage.
struct SortScratch {
    void *d_buf = nullptr;
    size_t bytes = 0;
    const uint32_t *perm = nullptr;  // result of the last sort (inside d_buf)
};
// The sort also raises *differ when trial lengths are not all equal; launch_length_check does
// that check alone (when the sort is skipped).
cudaError_t launch_length_sort(const uint64_t *offsets, uint64_t n, SortScratch &sc, int sm_count,
                               cudaStream_t stream, uint64_t *launches,
                               unsigned long long *differ);
cudaError_t launch_length_check(const uint64_t *offsets, uint64_t n, SortScratch &sc,
                                unsigned long long *differ, int sm_count, cudaStream_t stream,
                                uint64_t *launches);

// scan.cu
// Map modes >= 1: expand the dense rows to rows by catalogue id (direct[id] = dense[map[id]]) and
// build the presence bitmap (mode 2).
cudaError_t launch_expand_rows(const uint32_t *d_map, uint32_t C, const void *dense,
                               void *direct, size_t row_bytes, cudaStream_t stream);
cudaError_t launch_build_bitmap(const uint32_t *d_map, uint32_t C, uint32_t *bitmap,
                                uint32_t log2_bits, cudaStream_t stream);
cudaError_t launch_scan(const DeviceStore &st, const ScanLaunch &s, int sm_count,
                        cudaStream_t stream, uint64_t *launches);
// scan_pair.cu: the pair-skewed, exactly scaled fp64 scan (warp-batched tickets only)
bool pair_scan_eligible(const DeviceStore &st, const ScanLaunch &s);
cudaError_t launch_pair_scan(const DeviceStore &st, const ScanLaunch &s, int sm_count,
                             cudaStream_t stream, uint64_t *launches);
// hoist.cu
cudaError_t launch_hoist_oc(const DeviceStore &st, cudaStream_t stream, uint64_t *launches);
cudaError_t launch_hoisted_scan(const DeviceStore &st, const ScanLaunch &s, int sm_count,
                                cudaStream_t stream, uint64_t *launches);
cudaError_t launch_portfolio(const UnionStore &us, const uint32_t *d_map, int map_mode,
                             const uint32_t *d_bitmap, const ScanLaunch &s, int sm_count,
                             cudaStream_t stream, uint64_t *launches);
// Map mode 2: sample up to kProbeSamples of the YET's event ids (evenly strided) and count how
// many are in the store (probe[0]) of how many sampled (probe[1]); the scans skip their
// presence-bitmap test when at least 99% are (probe_use_bitmap).  probe[] must be zeroed first.
constexpr uint32_t kProbeSamples = 65536;
cudaError_t launch_hit_probe(const uint64_t *offsets, const uint32_t *ids, uint64_t n_trials,
                             const uint32_t *d_map, uint32_t C, unsigned long long *probe,
                             cudaStream_t stream, uint64_t *launches);
cudaError_t launch_validate(const uint64_t *offsets, const uint32_t *ids, uint64_t n_trials,
                            uint64_t n_ev, uint32_t catalogue_size, uint32_t *err, int sm_count,
                            cudaStream_t stream, uint64_t *launches);

// metrics.cu
struct MetricsScratch {
    void *d_buf = nullptr;
    size_t bytes = 0;
    int grid = 0;
    void *d_shard = nullptr;  // sharded metrics: state + per-block tail partials
    size_t shard_bytes = 0;
};
cudaError_t launch_portfolio_row(const double *d_ylt, uint32_t n_layers, uint64_t n, uint64_t ld,
                                 double *d_out, int sm_count, cudaStream_t stream,
                                 uint64_t *launches);
// Caller-supplied reduction for the sharded metrics: element-wise SUM across all ranks, in
// place, of `count` values (int64 if !is_f64, else fp64) at byte offset `offset` of the caller's
// device exchange buffer, ordered on the context's stream.  Returns 0 on success.
typedef int (*ShardReduce)(uint64_t offset, uint64_t count, int is_f64, void *user);
cudaError_t launch_metrics_sharded(const double *d_slice, uint64_t n_local, uint64_t n_global,
                                   uint32_t n_p, const double *p, double *pml_out,
                                   double *tvar_out, char *d_xbuf, ShardReduce reduce,
                                   void *user, MetricsScratch &scratch, int sm_count,
                                   cudaStream_t stream, uint64_t *launches);
// F4 exceedance curve (ara_ep_curve): the row sorted descending, stream-ordered.
struct EpScratch {
    void *d_buf = nullptr;
    size_t bytes = 0;
};
cudaError_t launch_ep_curve(const double *d_row, uint64_t n, double *d_out, EpScratch &sc,
                            int sm_count, cudaStream_t stream, uint64_t *launches);
// PML/TVaR of n_rows rows (row r at d_rows + r * ld, n entries each) in shared passes;
// pml_out / tvar_out are [n_rows][n_p].
cudaError_t launch_metrics(const double *d_rows, uint64_t ld, uint32_t n_rows, uint64_t n,
                           uint32_t n_p, const double *p, double *pml_out, double *tvar_out,
                           MetricsScratch &scratch, int sm_count, int device, cudaStream_t stream,
                           uint64_t *launches);

// Name of the last scan-kernel instantiation launched by this host thread, as ncu prints it
// (e.g. "pair_scan_kernel<1, 3, 1, 0>"); ara_run copies it into ara_info.last_kernel, and the
// bench keys its committed ncu counters by it.  Set by the launchers.
extern thread_local const char *t_last_kernel;
inline std::string kernel_arg(int v) { return std::to_string(v); }
inline std::string kernel_arg(bool v) { return v ? "1" : "0"; }
inline std::string kernel_arg(const char *v) { return v; }
template <typename... A>
std::string kernel_name(const char *base, A... args)
{
    std::string s = std::string(base) + "<";
    bool first = true;
    ((s += (first ? "" : ", ") + kernel_arg(args), first = false), ...);
    return s + ">";
}

// Resident blocks per SM of kernel `func` (`threads` threads, `smem` bytes of dynamic shared
// memory) on the current device.  The dynamic shared memory attribute is per device, so it is
// set on each device's first launch; `cache` is the launcher's per-instantiation static array.
constexpr int kMaxDevices = 64;
inline cudaError_t blocks_per_sm(const void *func, int threads, size_t smem,
                                 std::atomic<int> (&cache)[kMaxDevices], int &occ)
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const bool cached = dev >= 0 && dev < kMaxDevices;
    occ = cached ? cache[dev].load(std::memory_order_relaxed) : 0;
    if (occ > 0) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, func, threads, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    if (cached) cache[dev].store(occ, std::memory_order_relaxed);
    return cudaSuccess;
}

constexpr uint32_t kErrRange = 1u;
constexpr uint32_t kErrOffsets = 2u;

}  // namespace ara
