// metrics.cu -- YLT post-pass (A9): PML and TVaR of one YLT row on the device.
//
// PML(p) = v[ceil(p n) - 1] of the ascending row (nearest rank), TVaR(p) = mean of all v >=
// PML(p) (reading R11; the paper only names the metrics,
// PAPER.md L32).  Instead of sorting, one cooperative kernel finds all n_p order statistics
// at once by MSB radix select on order-preserving u64 keys (8 passes of 8 bits; each pass
// reads the L2-resident row once and builds per-probability 256-bin histograms of the
// elements still matching that probability's key prefix), then sums the tails.  Partial
// tail sums are combined in block order, so the result is deterministic for a given grid.
#include <cooperative_groups.h>
#include <string.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "ara_internal.h"

namespace cg = cooperative_groups;

namespace ara {
namespace {

constexpr int kThreads = 256;
constexpr int kBins = 256;
constexpr int kPasses = 8;

// A batch of R rows (row r at v + r * ld, n entries each) is processed in the same passes: slot
// s = r * n_p + i is (row r, probability i); R * n_p <= kMaxSlots.  One row is ara_metrics.
constexpr int kMaxSlots = 64;
// Early finish: once every slot's remaining key prefix holds at most kCand elements (and all of
// them together at most kCandTotal), one pass collects those elements and every block finds the
// ranks by sorting them in shared memory, instead of the remaining radix passes and their
// grid-wide barriers (the headline's 1M-entry row: 3 passes instead of 8).
constexpr int kCand = 1024;  // 2048 and 4096 measured the same (1M-8M entries)
constexpr int kCandTotal = 2 * kCand;

struct MetricsParams {
    const double *v;
    uint64_t ld;                   // row stride (elements)
    uint64_t n;                    // entries per row
    uint32_t n_rows;
    uint32_t n_p;
    uint64_t rank[ARA_MAX_P];      // 0-based target ranks ceil(p n) - 1 (same for every row)
    uint32_t *hist;                // [kPasses][kMaxSlots][kBins]
    double *part_sum;              // [grid][kMaxSlots]
    unsigned long long *part_cnt;  // [grid][kMaxSlots]
    double *out;                   // [2][n_rows * n_p]: pml, tvar
    uint64_t *cand;                // [kMaxSlots][kCand] candidate keys (early finish)
    unsigned int *cand_n;          // [kMaxSlots] candidates collected per distinct pair
};

// Order-preserving map of finite doubles to u64 (-0 canonicalised to +0).
__device__ __forceinline__ uint64_t to_key(double x)
{
    uint64_t b = (uint64_t)__double_as_longlong(x);
    if (b == 0x8000000000000000ull) b = 0;
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ double from_key(uint64_t k)
{
    uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)b);
}

// Distinct (row, key prefix under mask) pairs of the slots, row-major, so that the pairs of row r
// are u in [ubeg[r], ubeg[r + 1]).  Two distinct prefixes of one row are disjoint, so every
// element adds to at most one histogram.
__device__ __forceinline__ uint32_t dedup_rows(const uint64_t *prefix, uint32_t n_rows,
                                               uint32_t n_p, uint64_t mask, uint64_t *uprefix,
                                               uint32_t *uof, uint32_t *ubeg)
{
    uint32_t nu = 0;
    for (uint32_t r = 0; r < n_rows; ++r) {
        ubeg[r] = nu;
        for (uint32_t i = 0; i < n_p; ++i) {
            const uint32_t sl = r * n_p + i;
            uint32_t u = ubeg[r];
            while (u < nu && uprefix[u] != (prefix[sl] & mask)) ++u;
            if (u == nu) uprefix[nu++] = prefix[sl] & mask;
            uof[sl] = u;
        }
    }
    ubeg[n_rows] = nu;
    return nu;
}

__global__ void __launch_bounds__(kThreads) metrics_kernel(const __grid_constant__ MetricsParams P)
{
    cg::grid_group grid = cg::this_grid();
    extern __shared__ uint32_t sh[];          // [distinct pairs][kBins]
    __shared__ uint64_t s_prefix[kMaxSlots];  // per slot: key prefix found so far
    __shared__ uint64_t s_rank[kMaxSlots];    // per slot: rank within that prefix
    __shared__ uint64_t s_uprefix[kMaxSlots]; // distinct (row, prefix) pairs of this pass
    __shared__ uint32_t s_uof[kMaxSlots];     // slot -> its distinct pair
    __shared__ uint32_t s_ubeg[kMaxSlots + 1];
    __shared__ uint32_t s_nu;
    __shared__ uint64_t s_prefix_n[kMaxSlots];
    __shared__ uint64_t s_rank_n[kMaxSlots];
    __shared__ uint64_t s_cnt_n[kMaxSlots];   // elements under the new prefix
    __shared__ int s_done;                    // early finish taken

    const uint32_t n_p = P.n_p, R = P.n_rows, S = R * n_p;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;

    for (uint64_t i = gtid; i < (uint64_t)kPasses * kMaxSlots * kBins; i += gstride)
        P.hist[i] = 0;
    for (uint64_t i = gtid; i < (uint64_t)kMaxSlots; i += gstride) P.cand_n[i] = 0;
    if (threadIdx.x < S) {
        s_prefix[threadIdx.x] = 0;
        s_rank[threadIdx.x] = P.rank[threadIdx.x % n_p];
    }
    if (threadIdx.x == 0) s_done = 0;
    grid.sync();  // (zeroing with stream-ordered memsets instead measured 0.018 ms slower)

    for (int pass = 0; pass < kPasses && !s_done; ++pass) {
        const int shift = 56 - 8 * pass;
        const uint64_t mask = pass == 0 ? 0ull : (~0ull << (shift + 8));
        // Probabilities whose prefixes agree share one histogram (early passes: all of a row's)
        if (threadIdx.x == 0) s_nu = dedup_rows(s_prefix, R, n_p, mask, s_uprefix, s_uof, s_ubeg);
        __syncthreads();
        const uint32_t nu = s_nu;
        for (uint32_t i = threadIdx.x; i < nu * kBins; i += blockDim.x) sh[i] = 0;
        __syncthreads();
        for (uint32_t r = 0; r < R; ++r) {
            const double *v = P.v + (size_t)r * P.ld;
            const uint32_t u0 = s_ubeg[r], u1 = s_ubeg[r + 1];
            for (uint64_t e0 = gtid - lane; e0 < P.n; e0 += gstride) {  // warp-uniform trips
                const uint64_t e = e0 + lane;
                uint32_t slot = 0xffffffffu;  // (distinct pair, digit) or none
                if (e < P.n) {
                    const uint64_t key = to_key(v[e]);
                    for (uint32_t u = u0; u < u1; ++u)
                        if ((key & mask) == s_uprefix[u]) slot = u * kBins + ((key >> shift) & 0xff);
                }
                // warp-aggregated histogram update: one atomic per distinct slot in the warp
                // (after the first passes most warps hold no element of a surviving prefix)
                if (__any_sync(0xffffffffu, slot != 0xffffffffu)) {
                    const uint32_t peers = __match_any_sync(0xffffffffu, slot);
                    if (slot != 0xffffffffu && lane == (uint32_t)(__ffs(peers) - 1))
                        atomicAdd(sh + slot, (uint32_t)__popc(peers));
                }
            }
        }
        __syncthreads();
        uint32_t *gh = P.hist + (size_t)pass * kMaxSlots * kBins;
        for (uint32_t i = threadIdx.x; i < nu * kBins; i += blockDim.x) {
            const uint32_t c = sh[i];
            if (c) atomicAdd(gh + i, c);
        }
        grid.sync();
        // Every block reads the merged histograms and each slot finds the bin holding its rank:
        // one warp per distinct pair (8 bins per lane, a warp-shuffle scan of the lane totals),
        // no block-wide barriers inside and no serial walk over dependent L2 loads.
        static_assert(kBins == 32 * 8, "8 bins per lane");
        {
            const uint32_t warp = threadIdx.x >> 5;
            for (uint32_t u = warp; u < nu; u += kThreads / 32) {
                uint32_t row = 0;
                while (s_ubeg[row + 1] <= u) ++row;  // pairs are row-major
                const uint32_t *hu = gh + (size_t)u * kBins + lane * 8;
                uint64_t c[8], tot = 0;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    c[k] = __ldcg(hu + k);
                    tot += c[k];
                }
                uint64_t incl = tot;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= (uint32_t)o) incl += y;
                }
                const uint64_t excl = incl - tot;
                for (uint32_t i = row * n_p; i < (row + 1) * n_p; ++i) {
                    const uint64_t r = s_rank[i];
                    if (s_uof[i] == u && r >= excl && r < incl) {  // exactly one lane
                        uint64_t acc = excl;
                        for (int k = 0; k < 8; ++k) {
                            if (r < acc + c[k]) {
                                s_prefix_n[i] = s_prefix[i] | ((uint64_t)(lane * 8 + k) << shift);
                                s_rank_n[i] = r - acc;
                                s_cnt_n[i] = c[k];
                                break;
                            }
                            acc += c[k];
                        }
                    }
                }
            }
        }
        __syncthreads();
        if (threadIdx.x < S) {
            s_prefix[threadIdx.x] = s_prefix_n[threadIdx.x];
            s_rank[threadIdx.x] = s_rank_n[threadIdx.x];
        }
        __syncthreads();
        // early finish (every block takes the same decision: same merged histograms)
        if (pass >= 1 && pass + 1 < kPasses) {
            const uint64_t fmask = ~0ull << shift;  // bits fixed so far
            if (threadIdx.x == 0) {
                s_nu = dedup_rows(s_prefix, R, n_p, fmask, s_uprefix, s_uof, s_ubeg);
                uint64_t tot = 0;
                bool ok = true;
                for (uint32_t u = 0; u < s_nu; ++u) {
                    uint64_t cu = 0;  // the count of any slot of this pair
                    for (uint32_t i = 0; i < S; ++i)
                        if (s_uof[i] == u) cu = s_cnt_n[i];
                    ok = ok && cu <= (uint64_t)kCand;
                    tot += cu;
                }
                s_done = ok && tot <= (uint64_t)kCandTotal;
            }
            __syncthreads();
            if (s_done) {
                // collect every element under a surviving prefix
                const uint32_t nu = s_nu;
                for (uint32_t r = 0; r < R; ++r) {
                    const double *v = P.v + (size_t)r * P.ld;
                    const uint32_t u0 = s_ubeg[r], u1 = s_ubeg[r + 1];
                    for (uint64_t e = gtid; e < P.n; e += gstride) {
                        const uint64_t key = to_key(v[e]);
                        for (uint32_t u = u0; u < u1; ++u)
                            if ((key & fmask) == s_uprefix[u]) {
                                const unsigned int at = atomicAdd(P.cand_n + u, 1u);
                                if (at < (unsigned int)kCand) P.cand[(size_t)u * kCand + at] = key;
                            }
                    }
                }
                grid.sync();
                // each block sorts each pair's candidates in shared memory (bitonic, padded with
                // ~0) and reads its slots' ranks off the sorted keys
                uint64_t *sk = (uint64_t *)sh;  // kCand keys (8 KB of the dynamic buffer)
                for (uint32_t u = 0; u < nu; ++u) {
                    const uint32_t cu = __ldcg(P.cand_n + u);
                    uint32_t m = 1;
                    while (m < cu) m <<= 1;
                    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x)
                        sk[i] = i < cu ? __ldcg(P.cand + (size_t)u * kCand + i) : ~0ull;
                    __syncthreads();
                    for (uint32_t k = 2; k <= m; k <<= 1)
                        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                            for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
                                const uint32_t ij = i ^ j;
                                if (ij > i) {
                                    const uint64_t a = sk[i], b = sk[ij];
                                    if (((i & k) == 0) == (a > b)) {
                                        sk[i] = b;
                                        sk[ij] = a;
                                    }
                                }
                            }
                            __syncthreads();
                        }
                    if (threadIdx.x < S && s_uof[threadIdx.x] == u)
                        s_prefix[threadIdx.x] = sk[s_rank[threadIdx.x]];  // the full key
                    __syncthreads();
                }
            }
        }
    }

    // Tail sums over this block's contiguous chunk of each row in a fixed order, once per
    // distinct PML of the row (equal order statistics have equal tails).  The sum is of
    // (v - PML) >= 0, so TVaR = PML + mean(v - PML) >= PML holds exactly and the rounding error
    // scales with the tail's spread.
    if (threadIdx.x == 0) s_nu = dedup_rows(s_prefix, R, n_p, ~0ull, s_uprefix, s_uof, s_ubeg);
    __syncthreads();
    const uint64_t chunk = (P.n + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = (uint64_t)blockIdx.x * chunk;
    const uint64_t hi = lo + chunk < P.n ? lo + chunk : P.n;
    const uint32_t warp = threadIdx.x >> 5, nu_t = s_nu;
    // one warp per distinct (row, PML) pair: a fixed assignment and a fixed order, so the
    // partial sums are deterministic; no block-wide barriers
    for (uint32_t u = warp; u < nu_t; u += kThreads / 32) {
        uint32_t row = 0;
        while (s_ubeg[row + 1] <= u) ++row;
        const double *v = P.v + (size_t)row * P.ld;
        const uint64_t q = s_uprefix[u];
        const double qv = from_key(q);
        double sum = 0.0;
        unsigned long long c = 0;
        for (uint64_t e = lo + lane; e < hi; e += 32) {
            const double x = v[e];
            if (to_key(x) >= q) {
                sum += x - qv;
                ++c;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            sum += __shfl_down_sync(0xffffffffu, sum, o);
            c += __shfl_down_sync(0xffffffffu, c, o);
        }
        if (lane == 0) {
            P.part_sum[(size_t)blockIdx.x * kMaxSlots + u] = sum;
            P.part_cnt[(size_t)blockIdx.x * kMaxSlots + u] = c;
        }
    }
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x < S) {
        const uint32_t i = threadIdx.x, u = s_uof[i];
        double sum = 0.0;
        unsigned long long c = 0;
        for (uint32_t b = 0; b < gridDim.x; ++b) {
            sum += __ldcg(P.part_sum + (size_t)b * kMaxSlots + u);
            c += __ldcg(P.part_cnt + (size_t)b * kMaxSlots + u);
        }
        const double q = from_key(s_prefix[i]);
        P.out[i] = q;
        P.out[S + i] = q + sum / (double)c;
    }
}

// ---------------------------------------------------------------------------------------------
// Sharded PML/TVaR (launch_metrics_sharded): the YLT row is split over ranks; the same MSB radix
// select runs as separate per-pass kernels, and between passes the caller's reduction sums the
// per-rank histograms (a real exchange step: 8 x n_p x 256 counts instead of gathering the
// row).  Every rank holds identical state after each reduction, so the distinct-prefix
// numbering -- and with it the histogram layout -- agrees across ranks.
struct ShardState {
    unsigned long long prefix[ARA_MAX_P];  // key prefix found so far, per probability
    unsigned long long rank[ARA_MAX_P];    // global rank within that prefix
};

// distinct prefixes (under mask) of the probabilities, in first-appearance order
__device__ __forceinline__ uint32_t distinct_prefixes(const ShardState &S, uint32_t n_p,
                                                      uint64_t mask, uint64_t *uprefix,
                                                      uint32_t *uof)
{
    uint32_t nu = 0;
    for (uint32_t i = 0; i < n_p; ++i) {
        uint32_t u = 0;
        while (u < nu && uprefix[u] != (S.prefix[i] & mask)) ++u;
        if (u == nu) uprefix[nu++] = S.prefix[i] & mask;
        uof[i] = u;
    }
    return nu;
}

__global__ void __launch_bounds__(kThreads)
    shard_hist_kernel(const double *__restrict__ v, uint64_t n, uint32_t n_p, int pass,
                      const ShardState *__restrict__ st, long long *__restrict__ hist)
{
    __shared__ uint32_t sh[ARA_MAX_P * kBins];
    __shared__ uint64_t s_uprefix[ARA_MAX_P];
    __shared__ uint32_t s_uof[ARA_MAX_P];
    __shared__ uint32_t s_nu;
    const int shift = 56 - 8 * pass;
    const uint64_t mask = pass == 0 ? 0ull : (~0ull << (shift + 8));
    if (threadIdx.x == 0) s_nu = distinct_prefixes(*st, n_p, mask, s_uprefix, s_uof);
    for (uint32_t i = threadIdx.x; i < ARA_MAX_P * kBins; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const uint32_t nu = s_nu, lane = threadIdx.x & 31u;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x - lane; e0 < n;
         e0 += stride) {  // warp-uniform trip count
        const uint64_t e = e0 + lane;
        uint32_t slot = 0xffffffffu;
        if (e < n) {
            const uint64_t key = to_key(v[e]);
            for (uint32_t u = 0; u < nu; ++u)
                if ((key & mask) == s_uprefix[u]) slot = u * kBins + ((key >> shift) & 0xff);
        }
        if (__any_sync(0xffffffffu, slot != 0xffffffffu)) {
            const uint32_t peers = __match_any_sync(0xffffffffu, slot);
            if (slot != 0xffffffffu && lane == (uint32_t)(__ffs(peers) - 1))
                atomicAdd(sh + slot, (uint32_t)__popc(peers));
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nu * kBins; i += blockDim.x)
        if (sh[i]) atomicAdd((unsigned long long *)(hist + i), (unsigned long long)sh[i]);
}

// One block: every probability finds the bin of the (globally reduced) histogram that holds its
// rank and extends its prefix by that digit.
__global__ void __launch_bounds__(kThreads)
    shard_select_kernel(uint32_t n_p, int pass, ShardState *st, const long long *__restrict__ hist)
{
    __shared__ uint64_t s_uprefix[ARA_MAX_P];
    __shared__ uint32_t s_uof[ARA_MAX_P];
    __shared__ uint32_t s_nu;
    __shared__ unsigned long long s_wsum[kThreads / 32];
    __shared__ unsigned long long s_prefix_n[ARA_MAX_P], s_rank_n[ARA_MAX_P];
    const int shift = 56 - 8 * pass;
    const uint64_t mask = pass == 0 ? 0ull : (~0ull << (shift + 8));
    if (threadIdx.x == 0) s_nu = distinct_prefixes(*st, n_p, mask, s_uprefix, s_uof);
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31u;
    static_assert(kThreads == kBins, "one bin per thread");
    for (uint32_t u = 0; u < s_nu; ++u) {
        const unsigned long long cnt = (unsigned long long)hist[u * kBins + threadIdx.x];
        unsigned long long incl = cnt;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (uint32_t)o) incl += y;
        }
        if (lane == 31) s_wsum[threadIdx.x >> 5] = incl;
        __syncthreads();
        unsigned long long before = 0;
        for (uint32_t w = 0; w < (threadIdx.x >> 5); ++w) before += s_wsum[w];
        incl += before;
        const unsigned long long excl = incl - cnt;
        for (uint32_t i = 0; i < n_p; ++i) {
            const unsigned long long r = st->rank[i];
            if (s_uof[i] == u && r >= excl && r < incl) {
                s_prefix_n[i] = st->prefix[i] | ((unsigned long long)threadIdx.x << shift);
                s_rank_n[i] = r - excl;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x < n_p) {
        st->prefix[threadIdx.x] = s_prefix_n[threadIdx.x];
        st->rank[threadIdx.x] = s_rank_n[threadIdx.x];
    }
}

// Tail sums of (v - PML) over v >= PML for each distinct PML, per block, then combined in block
// order by shard_tail_combine_kernel: deterministic for a given grid.
__global__ void __launch_bounds__(kThreads)
    shard_tail_kernel(const double *__restrict__ v, uint64_t n, uint32_t n_p,
                      const ShardState *__restrict__ st, double *part_sum,
                      unsigned long long *part_cnt)
{
    __shared__ uint64_t s_uprefix[ARA_MAX_P];
    __shared__ uint32_t s_uof[ARA_MAX_P];
    __shared__ uint32_t s_nu;
    __shared__ double s_red[kThreads / 32];
    __shared__ unsigned long long s_redc[kThreads / 32];
    if (threadIdx.x == 0) s_nu = distinct_prefixes(*st, n_p, ~0ull, s_uprefix, s_uof);
    __syncthreads();
    const uint64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = (uint64_t)blockIdx.x * chunk, hi = lo + chunk < n ? lo + chunk : n;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint32_t u = 0; u < s_nu; ++u) {
        const uint64_t q = s_uprefix[u];
        const double qv = from_key(q);
        double sum = 0.0;
        unsigned long long c = 0;
        for (uint64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
            const double x = v[e];
            if (to_key(x) >= q) {
                sum += x - qv;
                ++c;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            sum += __shfl_down_sync(0xffffffffu, sum, o);
            c += __shfl_down_sync(0xffffffffu, c, o);
        }
        if (lane == 0) {
            s_red[warp] = sum;
            s_redc[warp] = c;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double bs = 0.0;
            unsigned long long bc = 0;
            for (int w = 0; w < kThreads / 32; ++w) {
                bs += s_red[w];
                bc += s_redc[w];
            }
            part_sum[(size_t)blockIdx.x * ARA_MAX_P + u] = bs;
            part_cnt[(size_t)blockIdx.x * ARA_MAX_P + u] = bc;
        }
        __syncthreads();
    }
}

__global__ void shard_tail_combine_kernel(uint32_t n_p, int blocks, const ShardState *st,
                                          const double *part_sum,
                                          const unsigned long long *part_cnt, double *sum_out,
                                          long long *cnt_out)
{
    __shared__ uint64_t s_uprefix[ARA_MAX_P];
    __shared__ uint32_t s_uof[ARA_MAX_P];
    if (threadIdx.x == 0) distinct_prefixes(*st, n_p, ~0ull, s_uprefix, s_uof);
    __syncthreads();
    if (threadIdx.x < n_p) {
        const uint32_t u = s_uof[threadIdx.x];
        double sum = 0.0;
        unsigned long long c = 0;
        for (int b = 0; b < blocks; ++b) {
            sum += part_sum[(size_t)b * ARA_MAX_P + u];
            c += part_cnt[(size_t)b * ARA_MAX_P + u];
        }
        sum_out[threadIdx.x] = sum;
        cnt_out[threadIdx.x] = (long long)c;
    }
}

// Portfolio-scope trial losses: out[t] = ((0 + ylt[0][t]) +
// ylt[1][t]) + ... in layer order -- coalesced reads of the L layer rows, one write.
__global__ void portfolio_row_kernel(const double *__restrict__ ylt, uint32_t n_layers,
                                     uint64_t n, uint64_t ld, double *__restrict__ out)
{
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
         t += (uint64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (uint32_t l = 0; l < n_layers; ++l) s = __dadd_rn(s, ylt[(size_t)l * ld + t]);
        out[t] = s;
    }
}

}  // namespace

cudaError_t launch_metrics(const double *d_rows, uint64_t ld, uint32_t n_rows, uint64_t n,
                           uint32_t n_p, const double *p, double *pml_out, double *tvar_out,
                           MetricsScratch &scratch, int sm_count, int device, cudaStream_t stream,
                           uint64_t *launches)
{
    cudaError_t e;
    int per_sm = 4;  // blocks per SM (tuning: ARA_METRICS_BLOCKS_PER_SM; 4 measured best)
    if (const char *bps = getenv("ARA_METRICS_BLOCKS_PER_SM")) per_sm = atoi(bps);
    if (per_sm < 1) per_sm = 1;
    if (scratch.d_buf == nullptr) {
        int coop = 0;
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
        if (!coop) return cudaErrorNotSupported;
        e = cudaFuncSetAttribute(metrics_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kMaxSlots * kBins * 4);
        if (e != cudaSuccess) return e;
        scratch.grid = sm_count * per_sm;  // upper bound; the launch clamps to co-residency
        scratch.bytes = (size_t)kPasses * kMaxSlots * kBins * 4 +
                        (size_t)scratch.grid * kMaxSlots * 16 + 2 * kMaxSlots * 8 +
                        (size_t)kMaxSlots * kCand * 8 + kMaxSlots * 4;
        e = cudaMalloc(&scratch.d_buf, scratch.bytes);
        if (e != cudaSuccess) return e;
    }
    uint64_t rank[ARA_MAX_P];
    for (uint32_t i = 0; i < n_p; ++i) {
        // nearest rank, computed in fp64 exactly as the reading states: ceil(p * n)
        uint64_t r = (uint64_t)ceil(p[i] * (double)n);
        if (r < 1) r = 1;
        if (r > n) r = n;
        rank[i] = r - 1;
    }
    const uint32_t rows_per = kMaxSlots / n_p;  // rows per launch (n_p <= ARA_MAX_P <= 64)
    for (uint32_t r0 = 0; r0 < n_rows; r0 += rows_per) {
        const uint32_t R = std::min(rows_per, n_rows - r0), S = R * n_p;
        MetricsParams P{};
        P.v = d_rows + (size_t)r0 * ld;
        P.ld = ld;
        P.n = n;
        P.n_rows = R;
        P.n_p = n_p;
        for (uint32_t i = 0; i < n_p; ++i) P.rank[i] = rank[i];
        char *b = (char *)scratch.d_buf;
        P.hist = (uint32_t *)b;
        b += (size_t)kPasses * kMaxSlots * kBins * 4;
        P.part_sum = (double *)b;
        b += (size_t)scratch.grid * kMaxSlots * 8;
        P.part_cnt = (unsigned long long *)b;
        b += (size_t)scratch.grid * kMaxSlots * 8;
        P.out = (double *)b;
        b += 2 * kMaxSlots * 8;
        P.cand = (uint64_t *)b;
        b += (size_t)kMaxSlots * kCand * 8;
        P.cand_n = (unsigned int *)b;
        // one histogram per distinct pair (<= S); at least kCand keys for the early finish sort
        const size_t smem = std::max((size_t)S * kBins * 4, (size_t)kCand * 8);
        int occ = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, metrics_kernel, kThreads, smem);
        if (e != cudaSuccess) return e;
        if (occ < 1) return cudaErrorNotSupported;
        int grid = sm_count * std::min(occ, per_sm);
        if (grid > scratch.grid) grid = scratch.grid;
        const uint64_t want = (n + kThreads - 1) / kThreads;
        if ((uint64_t)grid > want) grid = (int)want;
        void *args[] = {&P};
        ++*launches;
        e = cudaLaunchCooperativeKernel((void *)metrics_kernel, grid, kThreads, args, smem,
                                        stream);
        if (e != cudaSuccess) return e;
        double host[2 * kMaxSlots];
        e = cudaMemcpyAsync(host, P.out, 2 * S * sizeof(double), cudaMemcpyDeviceToHost, stream);
        if (e != cudaSuccess) return e;
        e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) return e;
        for (uint32_t i = 0; i < S; ++i) {
            pml_out[(size_t)r0 * n_p + i] = host[i];
            tvar_out[(size_t)r0 * n_p + i] = host[S + i];
        }
    }
    return cudaSuccess;
}

cudaError_t launch_metrics_sharded(const double *d_slice, uint64_t n_local, uint64_t n_global,
                                   uint32_t n_p, const double *p, double *pml_out,
                                   double *tvar_out, char *d_xbuf, ShardReduce reduce,
                                   void *user, MetricsScratch &scratch, int sm_count,
                                   cudaStream_t stream, uint64_t *launches)
{
    // scratch: the shard state and the per-block tail partials (the cooperative kernel's buffer
    // is large enough: kPasses x ARA_MAX_P x kBins x 4 bytes)
    cudaError_t e;
    const int blocks = sm_count * 4;
    const size_t need = sizeof(ShardState) + (size_t)blocks * ARA_MAX_P * 16;
    if (scratch.shard_bytes < need) {
        cudaFree(scratch.d_shard);
        scratch.d_shard = nullptr;
        scratch.shard_bytes = 0;
        e = cudaMalloc(&scratch.d_shard, need);
        if (e != cudaSuccess) return e;
        scratch.shard_bytes = need;
    }
    ShardState h{};
    for (uint32_t i = 0; i < n_p; ++i) {
        uint64_t r = (uint64_t)ceil(p[i] * (double)n_global);  // nearest rank, fp64 (R11)
        if (r < 1) r = 1;
        if (r > n_global) r = n_global;
        h.rank[i] = r - 1;
    }
    ShardState *st = (ShardState *)scratch.d_shard;
    double *part_sum = (double *)((char *)scratch.d_shard + sizeof(ShardState));
    unsigned long long *part_cnt = (unsigned long long *)(part_sum + (size_t)blocks * ARA_MAX_P);
    e = cudaMemcpyAsync(st, &h, sizeof(h), cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return e;
    long long *hist = (long long *)d_xbuf;  // [ARA_MAX_P][kBins], reduced across ranks
    const unsigned hb = n_local ? (unsigned)std::min<uint64_t>((n_local + kThreads - 1) / kThreads,
                                                                (uint64_t)blocks)
                                : 1u;
    for (int pass = 0; pass < kPasses; ++pass) {
        e = cudaMemsetAsync(hist, 0, (size_t)n_p * kBins * 8, stream);
        if (e != cudaSuccess) return e;
        ++*launches;
        shard_hist_kernel<<<hb, kThreads, 0, stream>>>(d_slice, n_local, n_p, pass, st, hist);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        if (reduce(0, (uint64_t)n_p * kBins, 0, user) != 0) return cudaErrorUnknown;
        ++*launches;
        shard_select_kernel<<<1, kThreads, 0, stream>>>(n_p, pass, st, hist);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    // tails: per-rank sums of (v - PML) and counts, reduced across ranks
    double *sums = (double *)d_xbuf;                      // [n_p] f64
    long long *cnts = (long long *)(d_xbuf + 8 * ARA_MAX_P);  // [n_p] i64
    ++*launches;
    shard_tail_kernel<<<hb, kThreads, 0, stream>>>(d_slice, n_local, n_p, st, part_sum, part_cnt);
    ++*launches;
    shard_tail_combine_kernel<<<1, 32, 0, stream>>>(n_p, (int)hb, st, part_sum, part_cnt, sums,
                                                    cnts);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (reduce(0, n_p, 1, user) != 0) return cudaErrorUnknown;
    if (reduce(8 * ARA_MAX_P, n_p, 0, user) != 0) return cudaErrorUnknown;
    double hs[ARA_MAX_P];
    long long hc[ARA_MAX_P];
    e = cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hs, sums, 8 * n_p, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hc, cnts, 8 * n_p, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return e;
    for (uint32_t i = 0; i < n_p; ++i) {
        uint64_t k = h.prefix[i];
        const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
        double q;
        memcpy(&q, &b, 8);
        pml_out[i] = q;
        tvar_out[i] = q + hs[i] / (double)hc[i];
    }
    return cudaSuccess;
}

cudaError_t launch_portfolio_row(const double *d_ylt, uint32_t n_layers, uint64_t n, uint64_t ld,
                                 double *d_out, int sm_count, cudaStream_t stream,
                                 uint64_t *launches)
{
    if (n == 0) return cudaSuccess;
    ++*launches;
    const uint64_t want = (n + 255) / 256;
    const unsigned blocks = (unsigned)std::min<uint64_t>(want, (uint64_t)sm_count * 8);
    portfolio_row_kernel<<<blocks, 256, 0, stream>>>(d_ylt, n_layers, n, ld, d_out);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// F4: exceedance-probability curves (reading R15).  The row's order-preserving keys
// (to_key: -0 canonicalised to +0) are sorted descending with CUB's radix sort (a library sort;
// the keys and the decode are this file's kernels) and decoded back: out[i] = the (i+1)-th
// largest value, exceedance probability (i+1)/n.
namespace {
__global__ void ep_keys_kernel(const double *__restrict__ v, uint64_t n, uint64_t *keys)
{
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        keys[i] = to_key(v[i]);
}

__global__ void ep_decode_kernel(const uint64_t *__restrict__ keys, uint64_t n, double *out)
{
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = from_key(keys[i]);
}
}  // namespace

cudaError_t launch_ep_curve(const double *d_row, uint64_t n, double *d_out, EpScratch &sc,
                            int sm_count, cudaStream_t stream, uint64_t *launches)
{
    if (n == 0) return cudaSuccess;
    size_t temp = 0;
    cudaError_t e = cub::DeviceRadixSort::SortKeysDescending(
        nullptr, temp, (const uint64_t *)nullptr, (uint64_t *)nullptr, (int64_t)n, 0, 64, stream);
    if (e != cudaSuccess) return e;
    const size_t need = 2 * n * sizeof(uint64_t) + temp + 256;
    if (sc.bytes < need) {
        cudaFree(sc.d_buf);  // synchronising: no earlier curve still uses the old buffer
        sc.d_buf = nullptr;
        sc.bytes = 0;
        e = cudaMalloc(&sc.d_buf, need);
        if (e != cudaSuccess) return e;
        sc.bytes = need;
    }
    uint64_t *keys = (uint64_t *)sc.d_buf, *sorted = keys + n;
    void *tmp = (void *)(((uintptr_t)(sorted + n) + 255) & ~(uintptr_t)255);
    const unsigned blocks = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)sm_count * 8);
    *launches += 3;  // keys, the CUB sort (a few internal kernels counted once), decode
    ep_keys_kernel<<<blocks, 256, 0, stream>>>(d_row, n, keys);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    e = cub::DeviceRadixSort::SortKeysDescending(tmp, temp, keys, sorted, (int64_t)n, 0, 64,
                                                 stream);
    if (e != cudaSuccess) return e;
    ep_decode_kernel<<<blocks, 256, 0, stream>>>(sorted, n, d_out);
    return cudaGetLastError();
}

}  // namespace ara
