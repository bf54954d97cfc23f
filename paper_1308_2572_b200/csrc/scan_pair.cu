// scan_pair.cu -- the fp64 YET scan (Algorithm 1 lines 3-29) for sm_100a on
// rows of W = 16, 32 or 64 columns: pair-skewed lane groups and exactly scaled clamps.
//
// Decomposition.  A row of W = 16 P doubles is P 128-byte lines.  A group of G = 2 P lanes owns
// one (trial, layer) ticket; lane c owns the 8 columns [8c, 8c + 8) of the layer's row (two
// 256-bit loads per event, both lines of a row in the same instructions).  The ELT sum of lines
// 11-13 must be the oracle's ((0 + F_0) + F_1) + ... + F_{W-1} (SURVEY.md finding 3), i.e. a
// chain through the lanes in column order: lane 0 sums its 8 columns, each further lane adds its
// 8 columns to its left neighbour's partial after one 64-bit shuffle (G - 1 hops; in SIMT every
// lane issues every hop).  P = 1 (the paper's 15-16 ELT layers) is the headline kernel; P = 2
// serves 17-32 ELTs.  (A skewed variant -- pair p one or two events behind pair p - 1, so every
// step needs only two hops -- computed fewer adds but ran 1.4-1.6x slower: its gathers were
// scheduled too late under register pressure; profiles/r2_tune_pair.jsonl.)
//
// Two events per step (EV = 2; the plain scan of 25-48 ELTs, ARA_PAIR_EV2=0 turns it off): the
// ELT sums of events j and j + 1 are independent, so pair_step2 runs both chains (and both hops)
// interleaved and then lines 15-29 for j and j + 1 in order -- the wide rows are bound by the
// latency of their serial chains (ncu: `wait` stalls first), and two chains per group hide half
// of it (E = 32: 26.1 -> 24.5 ms, E = 48: 36.9 -> 35.0 ms at 1M x 1000; W = 16 and 24 are
// faster with one event per step, W = 64 spills; profiles/r2_tune_ev2.jsonl).
//
// Exactly scaled clamps.  sm_100a has no fp64 min/max instruction; max(x, 0) as a compare-select
// costs DSETP + 2 FSEL.  Instead the kernel carries power-of-two multiples of the oracle's values:
//   2 max(x, 0) = x + |x|  exactly (x > 0: 2x is exact; x <= 0: x + |x| = +0 under RN),
// and scaling by 2^m commutes with every RN add/sub/compare as long as nothing overflows (sums of
// subnormals are exact, so underflow cannot differ either).  Per event:
//   F2_j  = min(x_j + |x_j|, 2 lim_j)                       = 2 F_j      (line 9)
//   lo2   = ((F2_0 + F2_1) + ...)                           = 2 lo      (lines 11-13)
//   t2    = lo2 - 2 OccR;  oc4 = min(t2 + |t2|, 4 OccL)     = 4 oc      (line 16)
//   S4   += oc4                                             = 4 S       (line 19)
//   u4    = S4 - 4 AggR;   C8  = min(u4 + |u4|, 8 AggL)     = 8 C_d     (line 22)
//   inc8  = C8 - C8_prev;  lr8 += inc8                      = 8 lr      (lines 25, 28)
// and the YLT entry is lr8 * 0.125 (exact).  ara_set_layers enables this path only when every
// loss * rate, retention, finite limit and layer term is below 2^960, so that 8 (k (E + 1) + 1)
// times that bound cannot overflow for any YET the device can hold (k < 2^36, E <= 64); other
// portfolios run scan.cu's compare-select kernel.  The result is bit-identical to the oracle's
// unscaled sequence (tests/test_parity_gpu.py).  (0 + F_0 = F_0 for F_0 >= +0, and F2 is never
// -0, so the chain may start at F2_0.)
#include <cuda_runtime.h>
#include <stdint.h>

#include "ara_internal.h"
#include "scan_common.cuh"

namespace ara {
namespace {

using namespace scan_detail;

constexpr unsigned kFull = 0xffffffffu;

// Bounds-checking debug builds (-DARA_DEBUG_BOUNDS, a tuning-library variant; compute-sanitizer
// is not available on every pool): every row index, trial range and YLT index is checked and a
// violation traps (a sticky launch error).  Product builds compile the checks away.
#ifdef ARA_DEBUG_BOUNDS
__constant__ uint64_t c_dbg_rows;  // rows of the store this launch reads
#define ARA_DBG_CHECK(cond) \
    do {                    \
        if (!(cond)) __trap(); \
    } while (0)
#else
#define ARA_DBG_CHECK(cond) \
    do {                    \
    } while (0)
#endif


template <int N>
struct ScaledTerms {
    double rate[N], ret[N], lim2[N];  // this lane's N = 4 CH columns
    double occ_ret2, occ_lim4, agg_ret4, agg_lim8;
};

// 2 max(x, 0), exact (see the file comment)
__device__ __forceinline__ double twice_max0(double x) { return __dadd_rn(x, fabs(x)); }

__device__ __forceinline__ double cmin(double m, double lim) { return (lim < m) ? lim : m; }

// Trial state of the group's last lane (lane G - 1 ends every step with the full ELT sum of its
// event); the other lanes carry the same registers with meaningless values.
struct TrialState {
    double S4, C8, lr8, max4;
};

// One step of lane c on its row segment r: financial terms of its 8 columns, the ELT chain,
// then (meaningful in lane G - 1) the occurrence and aggregate terms.  own is the lane's partial
// of its own columns (the gather pin).  Returns inc8 (lane G - 1).
// Chain hop: lane c > 0 receives lane c - 1's partial (src_up = its lane index; lane 0 its own).
// Groups of 2 or 4 lanes use the segmented up-shuffle, 3-lane groups (10 per warp) an indexed one.
template <int G>
__device__ __forceinline__ double hop_up(uint32_t gmask, double v, uint32_t src_up)
{
    if constexpr (G == 2 || G == 4) return __shfl_up_sync(gmask, v, 1, G);
    else return __shfl_sync(gmask, v, src_up);
}

template <int G, int CH, int X>
__device__ __forceinline__ double pair_step(const Chunk<double> (&r)[CH],
                                            const ScaledTerms<4 * CH> &T, uint32_t gmask,
                                            uint32_t src_up, double &own,
                                            TrialState &st)
{
    constexpr int N = 4 * CH;
    double f[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const double x = rsub(rmul(r[j >> 2].v[j & 3], T.rate[j]), T.ret[j]);  // line 9
        f[j] = cmin(twice_max0(x), T.lim2[j]);
    }
    // lines 11-13: lane 0 starts at F2_0 (= 0 + F2_0), lane h continues lane h - 1's partial
    double a = f[0];
#pragma unroll
    for (int j = 1; j < N; ++j) a = radd(a, f[j]);
    own = a;
#pragma unroll
    for (int h = 1; h < G; ++h) {
        double x = hop_up<G>(gmask, a, src_up);
#pragma unroll
        for (int j = 0; j < N; ++j) x = radd(x, f[j]);
        a = x;
    }
    // lines 15-29 on lo2 = a (lane G - 1)
    const double t2 = rsub(a, T.occ_ret2);
    const double oc4 = cmin(twice_max0(t2), T.occ_lim4);
    st.S4 = radd(st.S4, oc4);
    const double u4 = rsub(st.S4, T.agg_ret4);
    const double C8 = cmin(twice_max0(u4), T.agg_lim8);
    const double inc8 = rsub(C8, st.C8);
    st.lr8 = radd(st.lr8, inc8);
    st.C8 = C8;
    st.max4 = (st.max4 < oc4) ? oc4 : st.max4;  // F4 (dead code unless stored)
    return inc8;
}

// Two events of the trial at once (EV = 2): their ELT sums are independent, so the two chains
// (and their hops) interleave and hide each other's add latency; lines 15-29 then run for the
// first event and the second, in YET order.  Same operations, same order per event as pair_step.
template <int G, int CH, int X>
__device__ __forceinline__ void pair_step2(const Chunk<double> (&r0)[CH],
                                           const Chunk<double> (&r1)[CH],
                                           const ScaledTerms<4 * CH> &T, uint32_t gmask,
                                           uint32_t src_up, double &own0, double &own1,
                                           TrialState &st, double &inc0, double &inc1)
{
    constexpr int N = 4 * CH;
    double f0[N], f1[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const double x0 = rsub(rmul(r0[j >> 2].v[j & 3], T.rate[j]), T.ret[j]);  // line 9
        const double x1 = rsub(rmul(r1[j >> 2].v[j & 3], T.rate[j]), T.ret[j]);
        f0[j] = cmin(twice_max0(x0), T.lim2[j]);
        f1[j] = cmin(twice_max0(x1), T.lim2[j]);
    }
    double a0 = f0[0], a1 = f1[0];
#pragma unroll
    for (int j = 1; j < N; ++j) {
        a0 = radd(a0, f0[j]);
        a1 = radd(a1, f1[j]);
    }
    own0 = a0;
    own1 = a1;
#pragma unroll
    for (int h = 1; h < G; ++h) {
        double x0 = hop_up<G>(gmask, a0, src_up);
        double x1 = hop_up<G>(gmask, a1, src_up);
#pragma unroll
        for (int j = 0; j < N; ++j) {
            x0 = radd(x0, f0[j]);
            x1 = radd(x1, f1[j]);
        }
        a0 = x0;
        a1 = x1;
    }
    double lo2[2] = {a0, a1}, inc[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {  // lines 15-29, first event first
        const double t2 = rsub(lo2[e], T.occ_ret2);
        const double oc4 = cmin(twice_max0(t2), T.occ_lim4);
        st.S4 = radd(st.S4, oc4);
        const double u4 = rsub(st.S4, T.agg_ret4);
        const double C8 = cmin(twice_max0(u4), T.agg_lim8);
        inc[e] = rsub(C8, st.C8);
        st.lr8 = radd(st.lr8, inc[e]);
        st.C8 = C8;
        st.max4 = (st.max4 < oc4) ? oc4 : st.max4;
    }
    inc0 = inc[0];
    inc1 = inc[1];
}

// The lane's two 32-byte chunks: adjacent for G = 2 (16 columns, one line); G chunks apart for
// G = 3 and 4, whose 24- and 32-column rows are lane-interleaved (ara_internal.h row_phys_col),
// so that each of the group's two load instructions reads G contiguous chunks.
template <int G, int CH, bool ILV>
__device__ __forceinline__ void gather2(const double *__restrict__ my_rows, uint32_t stride,
                                        uint32_t idx, Chunk<double> (&r)[CH])
{
    ARA_DBG_CHECK(idx < c_dbg_rows);
    const double *p = my_rows + (size_t)idx * stride;
#pragma unroll
    for (int k = 0; k < CH; ++k) load_row_chunk(p + (ILV ? 4 * G : 4) * k, r[k]);
}

// F4 increments of an aligned 8-event chunk: the last lane (the one that carries the trial
// state) keeps each half chunk's 4 increments in registers and stores them as one 32-byte
// segment, L2 evict-first (scan_common.cuh store_v4): no shared memory, no warp barriers, no
// extra shuffles (profiles/r2_tune_interleave.jsonl: 15.4 ms with round 1's shared-memory
// staging, 14.7 ms with a broadcast of lo to the group and one 64-byte store per group, 13.6 ms).
__device__ __forceinline__ void store_inc4(double *d, const double (&slot)[4])
{
    if ((((uintptr_t)d) & 31u) == 0) {
        store_v4(d, slot[0], slot[1], slot[2], slot[3]);
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) d[q] = slot[q];
    }
}

// Row index of the event at step J of the current 8-event chunk (J = 8, 9: the next chunk; past
// the last full chunk the prefetch reads a zero row -- the tail redoes those steps).
template <int MM>
__device__ __forceinline__ uint32_t chunk_row(int J, const uint32_t (&idc)[8],
                                              const uint32_t (&idn)[8], bool more,
                                              const RowLookup &look, bool &bad)
{
    if (J < 8) return row_index<MM>(look, idc[J < 8 ? J : 0], bad);
    return more ? row_index<MM>(look, idn[J - 8 < 8 ? J - 8 : 0], bad) : look.zero_base;
}

template <int G, int CH, int MM, int X, int EV>
__device__ __forceinline__ void pair_body(const ScanLaunch &s, const uint32_t *__restrict__ map,
                                          const uint32_t *__restrict__ bitmap,
                                          const double *__restrict__ rows,
                                          const LayerTermsT<double> *__restrict__ terms,
                                          uint32_t n_layers)
{
    extern __shared__ __align__(16) uint32_t sbits[];  // map mode 2 only
    load_bitmap<MM>(sbits, bitmap, s.bitmap_log2);
    constexpr uint32_t W = 4 * G * CH;
    constexpr int N = 4 * CH;  // columns per lane
    constexpr bool ILV = W >= 24;  // lane-interleaved rows (ara_internal.h row_phys_col, ilv = G)
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t c = lane % G;
    // group mask: the groups of a warp run different trials (ragged lengths, head/tail loops)
    const uint32_t gmask = (G == 32) ? kFull : (((1u << G) - 1u) << (lane - c));
    const bool writer = c == G - 1;
    // groups per warp, this group's index in it (G = 3: 10 groups, lanes 30 and 31 idle)
    const uint32_t B = 32 / G, gw = lane / G;
    const bool active = gw < B;
    const uint32_t src_up = c ? lane - 1 : lane;
    const uint64_t warp_g = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) / 32;
    const uint64_t n_tickets = s.n_trials * n_layers;
    const uint32_t row_stride = n_layers * W;
    const uint32_t zb = s.zero_base;
    const RowLookup look{map, sbits, s.catalogue_size, zb, s.bitmap_log2};
    const uint64_t base = s.offsets[0];

    ScaledTerms<N> T;
    const double *__restrict__ my_rows = rows;
    double *ylt_row = s.ylt, *mo_row = nullptr, *inc_row = nullptr;
    uint32_t cur_layer = 0xffffffffu;
    bool bad = false;

    // Warp-batched tickets in length order (s.perm): ticket q = (trial perm[q / L], layer q % L);
    // a warp takes B consecutive tickets at a time from the device counter.
    for (uint64_t ticket = warp_g * B + gw;;) {
        if (ticket - gw >= n_tickets) break;  // warp-uniform
        if (active && ticket < n_tickets) {
            const uint64_t q = ticket / n_layers;
            const uint64_t t = s.perm ? (uint64_t)s.perm[q] : q;
            const uint32_t layer = (uint32_t)(ticket - q * n_layers);
            if (layer != cur_layer) {
                const LayerTermsT<double> &L = terms[layer];
#pragma unroll
                for (int j = 0; j < N; ++j) {
                    T.rate[j] = L.rate[N * c + j];
                    T.ret[j] = L.ret[N * c + j];
                    T.lim2[j] = 2.0 * L.lim[N * c + j];
                }
                T.occ_ret2 = 2.0 * L.occ_ret;
                T.occ_lim4 = 4.0 * L.occ_lim;
                T.agg_ret4 = 4.0 * L.agg_ret;
                T.agg_lim8 = 8.0 * L.agg_lim;
                my_rows = rows + (size_t)layer * W + (ILV ? 4 * c : N * c);
                ylt_row = s.ylt + (size_t)layer * s.ylt_ld;
                if (X) {
                    mo_row = s.max_occ ? s.max_occ + (size_t)layer * s.max_occ_ld : nullptr;
                    inc_row = X == 2 && s.event_inc ? s.event_inc + (size_t)layer * s.event_inc_ld
                                                    : nullptr;
                }
                cur_layer = layer;
            }
            const uint64_t beg = s.offsets[t] - base;
            const uint64_t k = s.offsets[t + 1] - base - beg;
            ARA_DBG_CHECK(t < s.n_trials && t < s.ylt_ld && s.offsets[t] >= base &&
                          beg + k <= s.offsets[s.n_trials] - base);
            const uint32_t *const tr = s.ids + beg;  // the trial's event ids
            TrialState st{0.0, 0.0, 0.0, 0.0};
            double own = 0.0;
            auto out = [&](double inc8, uint64_t e) {  // F4: the increment of event e
                if constexpr (X == 2)
                    if (inc_row && writer) inc_row[beg + e] = inc8 * 0.125;
            };
            auto single = [&](uint64_t e) {
                Chunk<double> r[CH];
                gather2<G, CH, ILV>(my_rows, row_stride, row_index<MM>(look, load_id(tr + e), bad), r);
                out(pair_step<G, CH, X>(r, T, gmask, src_up, own, st), e);
            };
            uint64_t e = 0;
            // head: single events until the id pointer is 32-byte aligned
            while (e < k && (((uintptr_t)(tr + e)) & 31u) != 0) single(e++);
            // body: chunks of 8 events; the ids of chunk i + 1 are in flight during chunk i, the
            // gather of event j + 1 while event j is computed
            const uint64_t n_chunks = (k - e) / 8;
            double slot[4];    // X == 2: the writer lane's increments of half a chunk
            uint64_t e0w = 0;  // YET position of the current chunk
            auto out8 = [&](double inc8, int j) {  // body events: kept in registers
                if constexpr (X == 2) {
                    slot[j & 3] = inc8 * 0.125;  // meaningful in the writer lane
                    if ((j & 3) == 3 && inc_row && writer) store_inc4(inc_row + beg + e0w + (j - 3), slot);
                }
            };
            if (n_chunks) {
                uint32_t id_c[8], id_n[8];
                load_ids8(tr + e, id_c);
                if (n_chunks > 1) load_ids8(tr + e + 8, id_n);
                Chunk<double> ra[CH], rb[CH];
                gather2<G, CH, ILV>(my_rows, row_stride, chunk_row<MM>(0, id_c, id_n, true, look, bad), ra);
                if constexpr (EV == 2) {
                    // two events per step: (ra, ra1) computed while (rb, rb1) load
                    Chunk<double> ra1[CH], rb1[CH];
                    double own1 = 0.0;
                    gather2<G, CH, ILV>(my_rows, row_stride, chunk_row<MM>(1, id_c, id_n, true, look, bad), ra1);
#pragma unroll 1
                    for (uint64_t i = 0; i < n_chunks; ++i) {
                        const bool more = i + 1 < n_chunks;
                        e0w = e + 8 * i;
#pragma unroll
                        for (int j = 0; j < 8; j += 4) {
                            double i0, i1;
                            gather2<G, CH, ILV>(my_rows, row_stride, pin(chunk_row<MM>(j + 2, id_c, id_n, more, look, bad), own), rb);
                            gather2<G, CH, ILV>(my_rows, row_stride, pin(chunk_row<MM>(j + 3, id_c, id_n, more, look, bad), own1), rb1);
                            pair_step2<G, CH, X>(ra, ra1, T, gmask, src_up, own, own1, st, i0, i1);
                            out8(i0, j);
                            out8(i1, j + 1);
                            gather2<G, CH, ILV>(my_rows, row_stride, pin(chunk_row<MM>(j + 4, id_c, id_n, more, look, bad), own), ra);
                            gather2<G, CH, ILV>(my_rows, row_stride, pin(chunk_row<MM>(j + 5, id_c, id_n, more, look, bad), own1), ra1);
                            pair_step2<G, CH, X>(rb, rb1, T, gmask, src_up, own, own1, st, i0, i1);
                            out8(i0, j + 2);
                            out8(i1, j + 3);
                        }
#pragma unroll
                        for (int j = 0; j < 8; ++j) id_c[j] = id_n[j];
                        if (i + 2 < n_chunks) load_ids8(tr + e + 8 * (i + 2), id_n);
                    }
                } else {
#pragma unroll 1
                for (uint64_t i = 0; i < n_chunks; ++i) {
                    const bool more = i + 1 < n_chunks;
                    const uint64_t e0 = e + 8 * i;
                    e0w = e0;
#pragma unroll
                    for (int j = 0; j < 8; j += 2) {
                        const uint32_t ib = chunk_row<MM>(j + 1, id_c, id_n, more, look, bad);
                        gather2<G, CH, ILV>(my_rows, row_stride, pin(ib, own), rb);
                        out8(pair_step<G, CH, X>(ra, T, gmask, src_up, own, st), j);
                        const uint32_t ic = chunk_row<MM>(j + 2, id_c, id_n, more, look, bad);
                        gather2<G, CH, ILV>(my_rows, row_stride, pin(ic, own), ra);
                        out8(pair_step<G, CH, X>(rb, T, gmask, src_up, own, st), j + 1);
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) id_c[j] = id_n[j];
                    if (i + 2 < n_chunks) load_ids8(tr + e + 8 * (i + 2), id_n);
                }
                }
                e += 8 * n_chunks;
            }
            while (e < k) single(e++);  // tail
            if (writer) {
                ylt_row[t] = st.lr8 * 0.125;  // A8 (exact rescale)
                if (X && mo_row) mo_row[t] = st.max4 * 0.25;
            }
        }
        __syncwarp();
        uint64_t b = 0;
        if (lane == 0) b = warps + atomicAdd(s.counter, 1ull);
        ticket = __shfl_sync(kFull, b, 0) * B + gw;
    }
    if (bad) atomicOr(s.err, kErrRange);
    __syncthreads();  // the last block to finish resets the ticket counter for the next launch
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(s.done, 1u) == gridDim.x - 1) {
            *s.counter = 0;
            *s.done = 0;
            __threadfence();
        }
    }
}

template <int G, int CH, int MINB, int MM, int X, int EV>
__global__ void __launch_bounds__(kScanThreads, MINB)
    pair_scan_kernel(const ScanLaunch s, const uint32_t *__restrict__ map,
                     const uint32_t *__restrict__ bitmap, const double *__restrict__ rows,
                     const LayerTermsT<double> *__restrict__ terms, uint32_t n_layers)
{
    if constexpr (MM == 2) {
        if (!probe_use_bitmap(s.probe)) {
            pair_body<G, CH, 1, X, EV>(s, map, bitmap, rows, terms, n_layers);
            return;
        }
    }
    pair_body<G, CH, MM, X, EV>(s, map, bitmap, rows, terms, n_layers);
}

template <int G, int CH, int MINB, int MM, int X, int EV = 1>
cudaError_t launch_pair(const DeviceStore &st, const ScanLaunch &s, int sm_count,
                        cudaStream_t stream)
{
    auto kern = pair_scan_kernel<G, CH, MINB, MM, X, EV>;
    const size_t smem = MM == 2 ? bitmap_bytes(kBitmapLog2Scan) : 0;
    static std::atomic<int> occ_cache[kMaxDevices];
    int occ = 0;
    cudaError_t e = blocks_per_sm((const void *)kern, kScanThreads, smem, occ_cache, occ);
    if (e != cudaSuccess) return e;
    // One wave of resident blocks; the warp-batched tickets balance the work.  Fewer blocks when
    // the tickets cannot fill them.
    constexpr uint64_t groups_per_block = (kScanThreads / 32) * (32 / G);
    const uint64_t n_tickets = s.n_trials * st.n_layers;
    uint64_t blocks = (uint64_t)sm_count * occ;
    const uint64_t need = (n_tickets + groups_per_block - 1) / groups_per_block;
    if (need < blocks) blocks = need;
    if (blocks == 0) blocks = 1;
    ScanLaunch sl = s;
    sl.zero_base = MM ? st.zero_base_direct : st.zero_base;
    sl.bitmap_log2 = kBitmapLog2Scan;
#ifdef ARA_DEBUG_BOUNDS
    const uint64_t rows_lim = (uint64_t)sl.zero_base + kZeroRows;
    e = cudaMemcpyToSymbolAsync(c_dbg_rows, &rows_lim, sizeof(rows_lim), 0,
                                cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return e;
#endif
    static const std::string name = kernel_name("pair_scan_kernel", G, CH, MINB, MM, X, EV);
    t_last_kernel = name.c_str();
    kern<<<(unsigned)blocks, kScanThreads, smem, stream>>>(
        sl, st.d_map, st.d_bitmap, (const double *)(MM ? st.d_rows_direct : st.d_rows),
        (const LayerTermsT<double> *)st.d_terms, st.n_layers);
    return cudaGetLastError();
}

template <int G, int CH, int MINB, int X, int EV = 1>
cudaError_t launch_pair_mm(const DeviceStore &st, const ScanLaunch &s, int sm_count,
                           cudaStream_t stream)
{
    if (!st.d_rows_direct) return launch_pair<G, CH, MINB, 0, X, EV>(st, s, sm_count, stream);
    if (st.map_mode == 1 || (X && st.map_mode == 2))
        return launch_pair<G, CH, MINB, 1, X, EV>(st, s, sm_count, stream);
    if constexpr (X == 0)
        if (st.map_mode == 2) return launch_pair<G, CH, MINB, 2, 0, EV>(st, s, sm_count, stream);
    return launch_pair<G, CH, MINB, 0, X, EV>(st, s, sm_count, stream);
}

// EV2MINB > 0: the plain scan (no F4 outputs) runs two events per step with that MINB
// (ARA_PAIR_EV2=0 keeps one event per step)
template <int G, int CH, int MINB, int EV2MINB = 0, int INCMINB = MINB>
cudaError_t launch_pair_x(const DeviceStore &st, const ScanLaunch &s, int sm_count,
                          cudaStream_t stream)
{
    if (s.event_inc) return launch_pair_mm<G, CH, INCMINB, 2>(st, s, sm_count, stream);
    if (s.max_occ) return launch_pair_mm<G, CH, MINB, 1>(st, s, sm_count, stream);
    if constexpr (EV2MINB > 0)  // (not behind the presence bitmap: map mode 2 spills there)
        if (st.pair_ev2 && !(st.d_rows_direct && st.map_mode == 2))
            return launch_pair_mm<G, CH, EV2MINB, 0, 2>(st, s, sm_count, stream);
    return launch_pair_mm<G, CH, MINB, 0>(st, s, sm_count, stream);
}

}  // namespace

#ifndef ARA_PAIR_INC_MINB16
#define ARA_PAIR_INC_MINB16 3
#endif
#ifndef ARA_PAIR_WIDE_MINB
#define ARA_PAIR_WIDE_MINB 2
#endif
bool pair_scan_eligible(const DeviceStore &st, const ScanLaunch &s)
{
    // W = 64: scan.cu's G = 4 lanes x 16 columns is faster (61.8 vs 72.7 ms for 1M x 1000,
    // profiles/r2_tune_pair.jsonl): 8 lanes x 8 columns issue twice the chain adds
    return st.bits == 64 && st.scaled && s.counter && s.done && st.pair_scan &&
           (st.width == 16 || st.width == 24 || st.width == 32 ||
            (st.pair_wide && (st.width == 48 || st.width == 64)));
}

cudaError_t launch_pair_scan(const DeviceStore &st, const ScanLaunch &s, int sm_count,
                             cudaStream_t stream, uint64_t *launches)
{
    if (s.n_trials == 0) return cudaSuccess;
    ++*launches;
    switch (st.width) {
        case 16: return launch_pair_x<2, 2, 3, 0, ARA_PAIR_INC_MINB16>(st, s, sm_count, stream);
        case 24: return launch_pair_x<3, 2, 3>(st, s, sm_count, stream);
        case 32:
            if (st.ilv == 2) return launch_pair_x<2, 4, ARA_PAIR_WIDE_MINB>(st, s, sm_count, stream);
            return launch_pair_x<4, 2, 3, 3>(st, s, sm_count, stream);
        case 48: return launch_pair_x<4, 3, ARA_PAIR_WIDE_MINB, 2>(st, s, sm_count, stream);
        case 64: return launch_pair_x<4, 4, ARA_PAIR_WIDE_MINB>(st, s, sm_count, stream);
        default: --*launches; return cudaErrorInvalidValue;
    }
}

}  // namespace ara
