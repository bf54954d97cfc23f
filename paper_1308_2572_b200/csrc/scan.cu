// scan.cu -- the YET scan kernel (Algorithm 1 lines 3-29 for one layer) for sm_100a.
//
// Decomposition: trial-per-group.  A group of G lanes (G = 2 for the paper's 15-16 ELT layers)
// owns one trial; lane c of the group owns the CH consecutive 32-byte chunks
// [c*CH, (c+1)*CH) of every event-major row, i.e. columns [4*CH*c, 4*CH*(c+1)), and keeps
// those columns' financial terms in its own registers.  Per event:
//   A2  all G lanes read the event id (256-bit loads of 8 ids, no L1 allocation, L2
//       evict-first: the YET is streamed once),
//   A3  map the catalogue id to a dense row (u32 map, L2-resident) and gather the row
//       together: one 256-bit load per lane and chunk, the group covering whole 128-byte lines
//       (measured 3x the event rate of one-lane-per-row gathers: profiles/README.md),
//   A4  each lane applies the financial terms to its columns; the ELT sum of lines 11-13 runs
//       as a chain through the group in column order (lane 0 adds its columns to +0 and
//       passes the partial to lane 1 by shuffle, ...), so lo = ((0 + F_0) + F_1) + ... in the
//       layer's ELT order, exactly the oracle's sequence,
//   A5-A7 lane G-1 applies the occurrence terms, adds to the running sum S, applies the
//       aggregate terms, differences against C_{d-1} and adds to lr,
//   A8  lane G-1 writes lr to the YLT.
// Every product / difference / sum is a separately rounded fp64 op (__dmul_rn, __dsub_rn,
// __dadd_rn; the file is also built with -fmad=false), min/max are the oracle's compares.
// The event loop is a rolled software pipeline: row(d+1) and map(d+2) are in flight while
// event d is computed.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <cub/device/device_radix_sort.cuh>

#include "ara_internal.h"
#include "scan_common.cuh"

// ARA_ABLATION (tuning builds only, tools/tune_scan.py with ARA_LIB_VARIANT): time the scan with
// phases removed, for a Fig. graph11-style breakdown:
// 1 = ids + row index + ELT sum of placeholders (no row gather), 2 = + row gather, 3 = +
// financial terms, unset = + occurrence / aggregate terms (the real kernel).  The YLT of an
// ablation build is meaningless.
#ifndef ARA_ABLATION
#define ARA_ABLATION 0
#endif

namespace ara {

thread_local const char *t_last_kernel = nullptr;

namespace {

using namespace scan_detail;

// A2-A8 for one event with its row chunks in r[] (see the file comment).
template <int G, int CH, typename R>
__device__ __forceinline__ void event_step(const Chunk<R> (&r)[CH],
                                           const R (&rate)[Chunk<R>::N * CH],
                                           const R (&ret)[Chunk<R>::N * CH],
                                           const R (&lim)[Chunk<R>::N * CH], uint32_t gmask,
                                           R occ_ret, R occ_lim, R agg_ret, R agg_lim, R &S,
                                           R &Cprev, R &lr, R &oc_out, R &inc_out, R &own)
{
    constexpr int PER = Chunk<R>::N;
    constexpr int NCOL = PER * CH;
    // A4, line 9 on this lane's columns: min(max(x*rate - ret, 0), lim)
    R f[NCOL];
#pragma unroll
    for (int i = 0; i < CH; ++i)
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int j = PER * i + q;
#if ARA_ABLATION == 1 || ARA_ABLATION == 2  // phase ablation (timing only): no financial terms
            f[j] = r[i].v[q];
#else
            const R l = rsub(rmul(r[i].v[q], rate[j]), ret[j]);
            f[j] = dmin(dmax0(l), lim[j]);
#endif
        }
    // lines 11-13: lo = ((0 + F_0) + F_1) + ... through the group in column order
    R part = R(0);
#pragma unroll
    for (int j = 0; j < NCOL; ++j) part = radd(part, f[j]);
    own = part;  // this lane's columns only: available before the chain through the group
#pragma unroll
    for (int h = 1; h < G; ++h) {
        R x = __shfl_up_sync(gmask, part, 1, G);  // lane h reads lane h-1
#pragma unroll
        for (int j = 0; j < NCOL; ++j) x = radd(x, f[j]);
        part = x;  // valid in lane h after hop h
    }
    // A5-A7 (valid in lane G-1)
#if ARA_ABLATION >= 1 && ARA_ABLATION <= 3  // phase ablation: no occurrence / aggregate terms
    S = radd(S, part);
    lr = S;
    oc_out = part;
    inc_out = part;
    return;
#endif
    const R oc = dmin(dmax0(rsub(part, occ_ret)), occ_lim);  // line 16
    S = radd(S, oc);                                          // line 19
    const R Cd = dmin(dmax0(rsub(S, agg_ret)), agg_lim);      // line 22
    const R inc = rsub(Cd, Cprev);                            // line 25
    lr = radd(lr, inc);                                       // line 28
    Cprev = Cd;
    oc_out = oc;
    inc_out = inc;
}

// F4 outputs of one event (X: compiled in only when requested): the trial's maximum
// occurrence loss and the event's incremental aggregate loss at its YET position.
template <int X, typename R>
__device__ __forceinline__ void event_out(R oc, R inc, R &max_oc, double *inc_row, uint64_t pos,
                                          bool writer)
{
    if (X) {
        max_oc = (max_oc < oc) ? oc : max_oc;
        if (X == 2 && inc_row && writer) inc_row[pos] = (double)inc;
    }
}

// F4 increments of an aligned 8-event chunk (X == 2, the pipelined loop): the writer lane
// stages inc_d in shared memory and the group stores the chunk's 8 increments as one 64-byte
// segment (one full 32-byte sector per lane for G = 2) instead of 8 scattered 8-byte stores.
template <int X, typename R>
__device__ __forceinline__ void event_out_staged(R oc, R inc, R &max_oc, double *stage, int j,
                                                 bool writer)
{
    max_oc = (max_oc < oc) ? oc : max_oc;
    if (X == 2 && stage && writer) stage[j] = (double)inc;
}

template <int G>
__device__ __forceinline__ void flush_inc(const double *stage, double *dst, uint32_t c,
                                          uint32_t gmask)
{
    constexpr int PER = 8 / G;  // increments stored by each lane of the group
    __syncwarp(gmask);          // the writer's staged values are visible to the group
    const double *src = stage + c * PER;
    double *d = dst + c * PER;
    if ((((uintptr_t)dst) & 63u) == 0) {
        if constexpr (PER == 8) {
            store_v4(d, src[0], src[1], src[2], src[3]);
            store_v4(d + 4, src[4], src[5], src[6], src[7]);
        } else if constexpr (PER == 4) {
            store_v4(d, src[0], src[1], src[2], src[3]);
        } else if constexpr (PER == 2) {
            store_v2(d, src[0], src[1]);
        } else {
#pragma unroll
            for (int k = 0; k < PER; ++k) d[k] = src[k];
        }
    } else {
#pragma unroll
        for (int k = 0; k < PER; ++k) d[k] = src[k];
    }
    __syncwarp(gmask);  // the stage is read before the next chunk overwrites it
}

// Chunk i of the lane's columns sits CS chunks after chunk i - 1 (CS = 1: logical rows; CS = G:
// lane-interleaved rows, ara_internal.h row_phys_col).
template <int CH, typename R, int CS = 1>
__device__ __forceinline__ void gather(const R *__restrict__ my_rows, uint32_t stride,
                                       uint32_t idx, Chunk<R> (&r)[CH])
{
    const R *p = my_rows + (size_t)idx * stride;
#if ARA_ABLATION == 1  // phase ablation (timing only): ids and row indices, no row gather
#pragma unroll
    for (int i = 0; i < CH; ++i)
#pragma unroll
        for (int q = 0; q < Chunk<R>::N; ++q) r[i].v[q] = (R)((idx >> q) & 7u);
    (void)p;
#else
#pragma unroll
    for (int i = 0; i < CH; ++i) load_row_chunk(p + Chunk<R>::N * CS * i, r[i]);
#endif
}

template <int G, int CH, int X, typename R, bool BAL, int MM, int D>
__device__ __forceinline__ void scan_body(const ScanLaunch &s, const uint32_t *__restrict__ map,
                                          const uint32_t *__restrict__ bitmap,
                                          const R *__restrict__ rows,
                                          const LayerTermsT<R> *__restrict__ terms,
                                          uint32_t n_layers)
{
    extern __shared__ __align__(16) uint32_t sbits[];  // map mode 2 only
    load_bitmap<MM>(sbits, bitmap, s.bitmap_log2);
    __shared__ __align__(16) double s_inc[X == 2 ? (kScanThreads / G) * kStageStride : 2];  // F4 staging
    constexpr int PER = Chunk<R>::N;
    constexpr int W = PER * G * CH;  // row width per layer (elements)
    constexpr int NCOL = PER * CH;   // columns per lane
    // lane-interleaved rows (fp64, W >= 32): the lane's chunks are G chunks apart
    constexpr bool ILV = sizeof(R) == 8 && W >= 32;
    static_assert(!ILV || G == 4, "interleaved rows are laid out for 4 lanes per trial");
    constexpr int CS = ILV ? G : 1;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t c = lane % G;   // this lane's position in its group
    const uint32_t gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane - c));

    // Work is handed out as tickets: ticket q = (trial q / L, layer q % L), so consecutive
    // groups of one trial share its id and map requests.  Group g starts with ticket g; then
    // either ticket += groups (static: the launch makes groups a multiple of L, so a lane keeps
    // its layer) or the group leader draws the next ticket from a device counter (dynamic:
    // balances variable-length trials; the last block to finish resets the counter).
    const uint64_t g = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const uint64_t groups = ((uint64_t)gridDim.x * blockDim.x) / G;
    const uint32_t leader = lane - c;
    const uint32_t row_stride = n_layers * W;  // elements per union row
    const uint32_t zb = s.zero_base;
    const RowLookup look{map, sbits, s.catalogue_size, zb, s.bitmap_log2};

    R rate[NCOL], ret[NCOL], lim[NCOL];  // terms I_j of this lane's columns
    R occ_ret = 0, occ_lim = 0, agg_ret = 0, agg_lim = 0;
    const R *__restrict__ my_rows = rows;
    double *ylt_row = s.ylt;
    double *mo_row = nullptr, *inc_row = nullptr;  // F4 outputs (X only)
    uint32_t cur_layer = 0xffffffffu;

    // Length-bucketed mode (s.perm, ARA_RUN_BALANCE): tickets index trials in the order of
    // s.perm (sorted by length) and are taken a warp-sized batch at a time, so the groups of a
    // warp run trials of nearly equal length and stay converged.
    constexpr bool batched = BAL;  // s.perm != nullptr
    const uint32_t B = 32 / G, gw = lane / G;  // groups per warp, this group's index in it
    const uint64_t warp_g = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) / 32;
    const uint64_t n_tickets = s.n_trials * n_layers;

    const uint64_t base = s.offsets[0];
    bool bad = false;
    for (uint64_t ticket = batched ? warp_g * B + gw : g;;) {
        if (batched ? ticket - gw >= n_tickets : ticket >= n_tickets) break;  // warp-uniform
        if (ticket < n_tickets) {
        const uint64_t q = ticket / n_layers;
        const uint64_t t = batched ? (uint64_t)s.perm[q] : q;
        const uint32_t layer = (uint32_t)(ticket - q * n_layers);
        if (layer != cur_layer) {
            const LayerTermsT<R> &T = terms[layer];
#pragma unroll
            for (int j = 0; j < NCOL; ++j) {
                rate[j] = T.rate[NCOL * c + j];
                ret[j] = T.ret[NCOL * c + j];
                lim[j] = T.lim[NCOL * c + j];
            }
            occ_ret = T.occ_ret;
            occ_lim = T.occ_lim;
            agg_ret = T.agg_ret;
            agg_lim = T.agg_lim;
            my_rows = rows + (size_t)layer * W + (ILV ? PER * c : NCOL * c);
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
        const uint32_t *ev = s.ids + beg;
        const uint32_t *const ev_end = ev + k;
        R S = 0, Cprev = 0, lr = 0;  // lines 19, 25 (C_0 = 0), 28
        R max_oc = 0, oc, inc;       // F4
        R own = 0;                   // last event's own-column partial (gather pin)
        const bool writer = c == G - 1;

        // head: single events until the id pointer is 32-byte aligned
        while (ev < ev_end && ((uintptr_t)ev & 31u) != 0) {
            Chunk<R> r[CH];
            gather<CH, R, CS>(my_rows, row_stride, row_index<MM>(look, load_id(ev), bad), r);
            event_step<G, CH, R>(r, rate, ret, lim, gmask, occ_ret, occ_lim, agg_ret, agg_lim, S,
                              Cprev, lr, oc, inc, own);
            event_out<X, R>(oc, inc, max_oc, inc_row, ev - s.ids, writer);
            ++ev;
        }
        // body: chunks of 8 events.  Pipeline per group: the ids of chunk i+1 are in flight
        // during chunk i (one 32-byte load per chunk), the map lookup of event j+2 and the row
        // gather of event j+1 are in flight while event j is computed.
        const uint64_t n_chunks = (uint64_t)(ev_end - ev) / 8;
        if constexpr (D > 2) {
            // Deep pipeline: a ring of D row buffers; event j is computed from slot j % D, which
            // is then refilled with the row of event j + D (zero row past the trial's end).
            static_assert(8 % D == 0, "D divides the 8-event chunk");
            if (n_chunks) {
                uint32_t id_c[8], id_n[8];
                load_ids8(ev, id_c);
                if (n_chunks > 1) load_ids8(ev + 8, id_n);
                Chunk<R> ring[D][CH];
#pragma unroll
                for (int e = 0; e < D; ++e)
                    gather<CH, R, CS>(my_rows, row_stride, row_index<MM>(look, id_c[e], bad),
                                  ring[e]);
#pragma unroll 1
                for (uint64_t i = 0; i < n_chunks; ++i) {
                    const bool more = i + 1 < n_chunks;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        event_step<G, CH, R>(ring[j % D], rate, ret, lim, gmask, occ_ret, occ_lim,
                                             agg_ret, agg_lim, S, Cprev, lr, oc, inc, own);
                        event_out<X, R>(oc, inc, max_oc, inc_row, (ev - s.ids) + 8 * i + j, writer);
                        const int e2 = j + D;  // refill: event j + D of this chunk or the next
                        const uint32_t id2 = e2 < 8 ? id_c[e2 < 8 ? e2 : 0] : id_n[e2 < 8 ? 0 : e2 - 8];
                        const bool ok2 = e2 < 8 || more;
                        const uint32_t idx2 = ok2 ? row_index<MM>(look, id2, bad) : zb;
                        gather<CH, R, CS>(my_rows, row_stride, pin(idx2, own), ring[j % D]);
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) id_c[j] = id_n[j];
                    if (i + 2 < n_chunks) load_ids8(ev + 8 * (i + 2), id_n);
                }
                ev += 8 * n_chunks;
            }
        } else if (n_chunks) {
            double *const stage = (X == 2 && inc_row) ? s_inc + (threadIdx.x / G) * kStageStride : nullptr;
            uint32_t id_c[8], id_n[8];
            load_ids8(ev, id_c);
            if (n_chunks > 1) load_ids8(ev + 8, id_n);
            uint32_t idx0 = row_index<MM>(look, id_c[0], bad);
            uint32_t idx1 = row_index<MM>(look, id_c[1], bad);
            Chunk<R> ra[CH];
            gather<CH, R, CS>(my_rows, row_stride, idx0, ra);
#pragma unroll 1
            for (uint64_t i = 0; i < n_chunks; ++i) {
                const bool more = i + 1 < n_chunks;
#pragma unroll
                for (int j = 0; j < 8; j += 2) {
                    // events j (in ra) and j+1: lookups of j+2, j+3 and gathers of j+1, j+2
                    uint32_t id2 = j + 2 < 8 ? id_c[j + 2] : id_n[0];
                    uint32_t id3 = j + 3 < 8 ? id_c[j + 3] : id_n[1];
                    const bool ok2 = j + 2 < 8 || more;
                    uint32_t idx2 = ok2 ? row_index<MM>(look, id2, bad) : zb;
                    Chunk<R> rb[CH];
                    gather<CH, R, CS>(my_rows, row_stride, pin(idx1, own), rb);
                    event_step<G, CH, R>(ra, rate, ret, lim, gmask, occ_ret, occ_lim, agg_ret,
                                      agg_lim, S, Cprev, lr, oc, inc, own);
                    if constexpr (X == 2)
                        event_out_staged<X, R>(oc, inc, max_oc, stage, j, writer);
                    else
                        event_out<X, R>(oc, inc, max_oc, inc_row, (ev - s.ids) + 8 * i + j, writer);
                    uint32_t idx3 = ok2 ? row_index<MM>(look, id3, bad) : zb;
                    gather<CH, R, CS>(my_rows, row_stride, pin(idx2, own), ra);  // event j+2 (zero row past end)
                    event_step<G, CH, R>(rb, rate, ret, lim, gmask, occ_ret, occ_lim, agg_ret,
                                      agg_lim, S, Cprev, lr, oc, inc, own);
                    if constexpr (X == 2)
                        event_out_staged<X, R>(oc, inc, max_oc, stage, j + 1, writer);
                    else
                        event_out<X, R>(oc, inc, max_oc, inc_row, (ev - s.ids) + 8 * i + j + 1,
                                        writer);
                    idx1 = idx3;
                }
                if constexpr (X == 2)
                    if (stage) flush_inc<G>(stage, inc_row + (ev - s.ids) + 8 * i, c, gmask);
#pragma unroll
                for (int j = 0; j < 8; ++j) id_c[j] = id_n[j];
                if (i + 2 < n_chunks) load_ids8(ev + 8 * (i + 2), id_n);
            }
            ev += 8 * n_chunks;
        }
        // tail: remaining events one by one
        while (ev < ev_end) {
            Chunk<R> r[CH];
            gather<CH, R, CS>(my_rows, row_stride, row_index<MM>(look, load_id(ev), bad), r);
            event_step<G, CH, R>(r, rate, ret, lim, gmask, occ_ret, occ_lim, agg_ret, agg_lim, S,
                              Cprev, lr, oc, inc, own);
            event_out<X, R>(oc, inc, max_oc, inc_row, ev - s.ids, writer);
            ++ev;
        }
        if (writer) {
            ylt_row[t] = (double)lr;  // A8
            if (X && mo_row) mo_row[t] = (double)max_oc;
        }
        }  // ticket < n_tickets
        if (batched) {
            __syncwarp();
            uint64_t b = 0;
            if (lane == 0) b = warps + atomicAdd(s.counter, 1ull);
            ticket = __shfl_sync(0xffffffffu, b, 0) * B + gw;
        } else if (s.counter) {
            uint64_t next = 0;
            if (c == 0) next = groups + atomicAdd(s.counter, 1ull);
            ticket = __shfl_sync(gmask, next, leader);
        } else {
            ticket += groups;
        }
    }
    if (bad) atomicOr(s.err, kErrRange);
    if (s.counter) {  // the last block to finish resets the ticket counter for the next launch
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(s.done, 1u) == gridDim.x - 1) {
                *s.counter = 0;
                *s.done = 0;
                __threadfence();
            }
        }
    }
}

// The kernel: map mode 2 runs its mode-1 body when the hit probe found (nearly) every sampled
// id in the store (probe_use_bitmap), chosen once per launch.
template <int G, int CH, int MINB, int X, typename R, bool BAL, int MM, int D = 2>
__global__ void __launch_bounds__(kScanThreads, MINB)
    scan_kernel(const ScanLaunch s, const uint32_t *__restrict__ map,
                const uint32_t *__restrict__ bitmap, const R *__restrict__ rows,
                const LayerTermsT<R> *__restrict__ terms, uint32_t n_layers)
{
    if constexpr (MM == 2) {
        if (!probe_use_bitmap(s.probe)) {
            scan_body<G, CH, X, R, BAL, 1, D>(s, map, bitmap, rows, terms, n_layers);
            return;
        }
    }
    scan_body<G, CH, X, R, BAL, MM, D>(s, map, bitmap, rows, terms, n_layers);
}

// Device-side validation (ARA_RUN_VALIDATE): offsets non-decreasing, ids in [1, C].  n_ev =
// offsets[n] - offsets[0] comes from the host, which has checked offsets[n] >= offsets[0]: the
// id pass never reads past the YET whatever the interior offsets hold.
__global__ void validate_kernel(const uint64_t *__restrict__ offsets,
                                const uint32_t *__restrict__ ids, uint64_t n_trials,
                                uint64_t n_ev, uint32_t C, uint32_t *err)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t e = 0;
    for (uint64_t t = tid; t < n_trials; t += stride)
        if (offsets[t + 1] < offsets[t]) e |= kErrOffsets;
    for (uint64_t i = tid; i < n_ev; i += stride)
        if (ids[i] - 1u >= C) e |= kErrRange;
    if (e) atomicOr(err, e);
}

// Map-mode-2 hit probe (launch_hit_probe): one thread per sampled id, evenly strided over the
// YET (the samples are independent DRAM reads: one per thread keeps them all in flight).
// probe[0] = sampled ids present in the store, probe[1] = ids sampled (zeroed before launch).
__global__ void __launch_bounds__(256) hit_probe_kernel(const uint64_t *__restrict__ offsets,
                                                        const uint32_t *__restrict__ ids,
                                                        uint64_t n_trials,
                                                        const uint32_t *__restrict__ map,
                                                        uint32_t C, unsigned long long *probe)
{
    const uint64_t n_ev = offsets[n_trials] - offsets[0];
    const uint64_t m = n_ev < kProbeSamples ? n_ev : kProbeSamples;
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool hit = false;
    if (i < m) {
        const uint32_t id = ids[i * (n_ev / m)];
        hit = (id - 1u) < C && map[id] != 0u;
    }
    const uint32_t nh = __popc(__ballot_sync(0xffffffffu, hit));
    const uint32_t nc = __popc(__ballot_sync(0xffffffffu, i < m));
    if ((threadIdx.x & 31u) == 0 && nc) {
        atomicAdd(probe, (unsigned long long)nh);
        atomicAdd(probe + 1, (unsigned long long)nc);
    }
}

// Keys for the length sort: trial lengths (saturated to 32 bits) and trial indices.
// Also raises *differ when some trial's length differs from trial 0's (keys == nullptr: the
// check alone plus the identity order, used when the sort is skipped).
__global__ void length_keys_kernel(const uint64_t *__restrict__ offsets, uint64_t n,
                                   uint32_t *keys, uint32_t *idx, unsigned long long *differ)
{
    const uint64_t len0 = offsets[1] - offsets[0];
    bool d = false;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t len = offsets[t + 1] - offsets[t];
        d |= len != len0;
        if (keys) keys[t] = len > 0xffffffffull ? 0xffffffffu : (uint32_t)len;
        idx[t] = (uint32_t)t;
    }
    if (differ && __any_sync(0xffffffffu, d) && (threadIdx.x & 31u) == 0) atomicOr(differ, 1ull);
}

template <int G, int CH, int MINB, int X, typename R, bool BAL, int MM, int D>
cudaError_t launch_gcm(const DeviceStore &st, const ScanLaunch &s, int sm_count,
                       cudaStream_t stream)
{
    const size_t smem = MM == 2 ? bitmap_bytes(kBitmapLog2Scan) : 0;
    static std::atomic<int> occ_cache[kMaxDevices];  // resident blocks per SM, per device
    int occ = 0;
    cudaError_t oe = blocks_per_sm((const void *)scan_kernel<G, CH, MINB, X, R, BAL, MM, D>,
                                   kScanThreads, smem, occ_cache, occ);
    if (oe != cudaSuccess) return oe;
    // Balanced single wave over (trial, layer) groups: every trial slot gets ceil(n / slots)
    // or one fewer trials; the number of groups is a multiple of L (a lane keeps its layer) and,
    // where possible, the grid is a multiple of the SM count.
    const uint64_t L = st.n_layers;
    const uint64_t per_block = kScanThreads / G;
    uint64_t m = L;  // blocks must be a multiple of m = L / gcd(L, per_block)
    for (uint64_t a = L, b = per_block; b;) { const uint64_t r = a % b; a = b; b = r; m = L / a; }
    const uint64_t max_blocks = (uint64_t)sm_count * occ / m * m;
    if (max_blocks == 0) return cudaErrorInvalidConfiguration;
    const uint64_t slots_max = max_blocks * per_block / L;
    const uint64_t rounds = (s.n_trials + slots_max - 1) / slots_max;
    const uint64_t slots = (s.n_trials + rounds - 1) / rounds;
    uint64_t blocks = (slots * L + per_block - 1) / per_block;
    blocks = (blocks + m - 1) / m * m;
    uint64_t lcm = m;
    while (lcm % (uint64_t)sm_count) lcm += m;
    if (blocks >= (uint64_t)sm_count && (blocks + lcm - 1) / lcm * lcm <= max_blocks)
        blocks = (blocks + lcm - 1) / lcm * lcm;
    if (blocks > max_blocks) blocks = max_blocks;
    ScanLaunch sl = s;
    sl.zero_base = MM ? st.zero_base_direct : st.zero_base;
    sl.bitmap_log2 = kBitmapLog2Scan;
    static const std::string name = kernel_name("scan_kernel", G, CH, MINB, X,
                                                sizeof(R) == 8 ? "double" : "float", BAL, MM, D);
    t_last_kernel = name.c_str();
    scan_kernel<G, CH, MINB, X, R, BAL, MM, D><<<(unsigned)blocks, kScanThreads, smem, stream>>>(
        sl, st.d_map, st.d_bitmap, (const R *)(MM ? st.d_rows_direct : st.d_rows),
        (const LayerTermsT<R> *)st.d_terms, st.n_layers);
    return cudaGetLastError();
}

// Map mode dispatch.
template <int G, int CH, int MINB = 1, int X = 0, typename R = double, bool BAL = false,
          int D = 2>
cudaError_t launch_gc(const DeviceStore &st, const ScanLaunch &s, int sm_count,
                      cudaStream_t stream)
{
    // The per-layer direct rows exist only when the union-row store does not serve the layers
    // (then the F4 outputs, which always use the per-layer kernel, read the dense rows through
    // the map); the F4 outputs read direct rows without the bitmap (mode 1).
    if (!st.d_rows_direct)
        return launch_gcm<G, CH, MINB, X, R, BAL, 0, D>(st, s, sm_count, stream);
    if (st.map_mode == 1 || (X && st.map_mode == 2))
        return launch_gcm<G, CH, MINB, X, R, BAL, 1, D>(st, s, sm_count, stream);
    if (!X && st.map_mode == 2)
        return launch_gcm<G, CH, MINB, X, R, BAL, X ? 0 : 2, D>(st, s, sm_count, stream);
    return launch_gcm<G, CH, MINB, X, R, BAL, 0, D>(st, s, sm_count, stream);
}

}  // namespace

__global__ void expand_rows_kernel(const uint32_t *__restrict__ map, uint32_t C,
                                   const uint4 *__restrict__ dense, uint4 *__restrict__ direct,
                                   uint32_t row_vecs)
{
    // rows 0..C: direct[id] = dense[map[id]]; rows C+1..C+kZeroRows: the zero-row block
    const uint64_t n = ((uint64_t)C + 1 + kZeroRows) * row_vecs;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t id = i / row_vecs, v = i - id * row_vecs;
        direct[i] = id <= C ? dense[(uint64_t)map[id] * row_vecs + v] : make_uint4(0, 0, 0, 0);
    }
}

__global__ void build_bitmap_kernel(const uint32_t *__restrict__ map, uint32_t C, uint32_t *bits,
                                    uint32_t log2_bits)
{
    for (uint32_t id = blockIdx.x * blockDim.x + threadIdx.x + 1; id <= C && id != 0;
         id += gridDim.x * blockDim.x)
        if (map[id]) {
            const uint32_t h = bitmap_hash(id, log2_bits);
            atomicOr(bits + (h >> 5), 1u << (h & 31u));
        }
}

cudaError_t launch_expand_rows(const uint32_t *d_map, uint32_t C, const void *dense,
                               void *direct, size_t row_bytes, cudaStream_t stream)
{
    if (row_bytes % 16) return cudaErrorInvalidValue;
    expand_rows_kernel<<<1184, 256, 0, stream>>>(d_map, C, (const uint4 *)dense, (uint4 *)direct,
                                                 (uint32_t)(row_bytes / 16));
    return cudaGetLastError();
}

cudaError_t launch_build_bitmap(const uint32_t *d_map, uint32_t C, uint32_t *bitmap,
                                uint32_t log2_bits, cudaStream_t stream)
{
    cudaError_t e = cudaMemsetAsync(bitmap, 0, bitmap_bytes(log2_bits), stream);
    if (e != cudaSuccess) return e;
    build_bitmap_kernel<<<592, 256, 0, stream>>>(d_map, C, bitmap, log2_bits);
    return cudaGetLastError();
}

cudaError_t launch_scan(const DeviceStore &st, const ScanLaunch &s, int sm_count,
                        cudaStream_t stream, uint64_t *launches)
{
    if (s.n_trials == 0) return cudaSuccess;
    // this kernel reads logical rows (W <= 16) or rows interleaved for its 4 lanes (W >= 32)
    if (st.ilv != 0 && st.ilv != 4) return cudaErrorInvalidValue;
    ++*launches;
    if (s.perm && (s.max_occ || s.event_inc)) {  // F4 outputs, length-bucketed (fp64 store)
        if (st.bits != 64) { --*launches; return cudaErrorInvalidValue; }
        // X = 1: the per-trial maximum only (no increment code in the loop); X = 2: both
        const bool inc = s.event_inc != nullptr;
        switch (st.width) {
#define ARA_F4_BAL(G_, CH_, MINB_)                                                          \
    return inc ? launch_gc<G_, CH_, MINB_, 2, double, true>(st, s, sm_count, stream)        \
               : launch_gc<G_, CH_, MINB_, 1, double, true>(st, s, sm_count, stream)
            case 4: ARA_F4_BAL(1, 1, 1);
            case 8: ARA_F4_BAL(2, 1, 4);
            case 16: ARA_F4_BAL(2, 2, 3);
            case 32: ARA_F4_BAL(4, 2, 3);
            case 48: ARA_F4_BAL(4, 3, 1);
            case 64: ARA_F4_BAL(4, 4, 1);
#undef ARA_F4_BAL
            default: --*launches; return cudaErrorInvalidValue;
        }
    }
    if (s.perm) {  // length-bucketed (ARA_RUN_BALANCE)
        if (st.bits == 32) {
            switch (st.width) {
                // register caps (__launch_bounds__ min blocks): without them ptxas spends up to
                // 254 registers on deeper pipelining and halves the resident warps
                case 8: return launch_gc<1, 1, 4, 0, float, true>(st, s, sm_count, stream);
                case 16: return launch_gc<2, 1, 4, 0, float, true>(st, s, sm_count, stream);
                case 32: return launch_gc<2, 2, 2, 0, float, true>(st, s, sm_count, stream);
                case 64: return launch_gc<4, 2, 2, 0, float, true>(st, s, sm_count, stream);
                default: --*launches; return cudaErrorInvalidValue;
            }
        }
        switch (st.width) {
            case 4: return launch_gc<1, 1, 1, 0, double, true>(st, s, sm_count, stream);
            case 8: return launch_gc<2, 1, 4, 0, double, true>(st, s, sm_count, stream);
            case 16:  // tuning variants: ARA_SCAN_GROUP (G), ARA_SCAN_DEPTH (D), ARA_SCAN_MINB
                if (st.group_override == 4) {
                    if (st.depth == 8)
                        return launch_gc<4, 1, 3, 0, double, true, 8>(st, s, sm_count, stream);
                    if (st.min_blocks == 4)
                        return launch_gc<4, 1, 4, 0, double, true, 4>(st, s, sm_count, stream);
                    return launch_gc<4, 1, 3, 0, double, true, 4>(st, s, sm_count, stream);
                }
                if (st.depth == 4 && st.min_blocks == 3)
                    return launch_gc<2, 2, 3, 0, double, true, 4>(st, s, sm_count, stream);
                if (st.depth == 4)
                    return launch_gc<2, 2, 2, 0, double, true, 4>(st, s, sm_count, stream);
                if (st.min_blocks == 2)
                    return launch_gc<2, 2, 2, 0, double, true>(st, s, sm_count, stream);
                return launch_gc<2, 2, 3, 0, double, true>(st, s, sm_count, stream);
            case 32: return launch_gc<4, 2, 3, 0, double, true>(st, s, sm_count, stream);
            case 48: return launch_gc<4, 3, 1, 0, double, true>(st, s, sm_count, stream);
            case 64: return launch_gc<4, 4, 1, 0, double, true>(st, s, sm_count, stream);
            default: --*launches; return cudaErrorInvalidValue;
        }
    }
    if (st.bits == 32) {  // F3: fp32 store (widths in floats: 8, 16, 32, 64)
        const bool x = s.max_occ || s.event_inc;
        switch (st.width) {
            case 8: return x ? launch_gc<1, 1, 1, 2, float>(st, s, sm_count, stream)
                             : launch_gc<1, 1, 1, 0, float>(st, s, sm_count, stream);
            case 16: return x ? launch_gc<2, 1, 1, 2, float>(st, s, sm_count, stream)
                              : launch_gc<2, 1, 1, 0, float>(st, s, sm_count, stream);
            case 32: return x ? launch_gc<2, 2, 1, 2, float>(st, s, sm_count, stream)
                              : launch_gc<2, 2, 1, 0, float>(st, s, sm_count, stream);
            case 64: return x ? launch_gc<4, 2, 1, 2, float>(st, s, sm_count, stream)
                              : launch_gc<4, 2, 1, 0, float>(st, s, sm_count, stream);
            default: --*launches; return cudaErrorInvalidValue;
        }
    }
    if (s.max_occ || s.event_inc) {  // F4 outputs, per-group tickets (fp32 store, > 2^32 trials)
        switch (st.width) {
            case 4: return launch_gc<1, 1, 1, 2>(st, s, sm_count, stream);
            case 8: return launch_gc<2, 1, 1, 2>(st, s, sm_count, stream);
            case 16: return launch_gc<2, 2, 3, 2>(st, s, sm_count, stream);
            case 32: return launch_gc<4, 2, 1, 2>(st, s, sm_count, stream);
            case 48: return launch_gc<4, 3, 1, 2>(st, s, sm_count, stream);
            case 64: return launch_gc<4, 4, 1, 2>(st, s, sm_count, stream);
            default: --*launches; return cudaErrorInvalidValue;
        }
    }
    const ScanShape sh = scan_shape_for_width(st.width, st.group_override);
    switch (sh.G * 16 + sh.CH) {
        case 1 * 16 + 1: return launch_gc<1, 1>(st, s, sm_count, stream);
        case 2 * 16 + 1: return launch_gc<2, 1, 4>(st, s, sm_count, stream);
        case 4 * 16 + 1:  // W = 16 with G = 4 (tuning)
            switch (st.min_blocks) {
                case 5: return launch_gc<4, 1, 5>(st, s, sm_count, stream);
                case 6: return launch_gc<4, 1, 6>(st, s, sm_count, stream);
                default: return launch_gc<4, 1>(st, s, sm_count, stream);
            }
        case 4 * 16 + 2: return launch_gc<4, 2, 3>(st, s, sm_count, stream);
        case 4 * 16 + 3: return launch_gc<4, 3>(st, s, sm_count, stream);
        case 4 * 16 + 4: return launch_gc<4, 4>(st, s, sm_count, stream);
        case 2 * 16 + 2:  // W = 16 (default)
            switch (st.min_blocks) {
                case 4: return launch_gc<2, 2, 4>(st, s, sm_count, stream);
                default: return launch_gc<2, 2, 3>(st, s, sm_count, stream);
            }
        case 1 * 16 + 4: return launch_gc<1, 4>(st, s, sm_count, stream);  // W = 16, G = 1
        default: --*launches; return cudaErrorInvalidValue;
    }
}

namespace {
// Scratch of the length sort / check: keys, indices (in/out), CUB temporary storage.
cudaError_t sort_scratch(uint64_t n, SortScratch &sc, size_t &temp, cudaStream_t stream)
{
    temp = 0;
    cudaError_t e = cub::DeviceRadixSort::SortPairsDescending(
        nullptr, temp, (const uint32_t *)nullptr, (uint32_t *)nullptr, (const uint32_t *)nullptr,
        (uint32_t *)nullptr, (int)n, 0, 32, stream);
    if (e != cudaSuccess) return e;
    const size_t need = 4 * (size_t)n * 4 + temp + 256;
    if (sc.bytes < need) {
        cudaFree(sc.d_buf);
        sc.d_buf = nullptr;
        sc.bytes = 0;
        e = cudaMalloc(&sc.d_buf, need);
        if (e != cudaSuccess) return e;
        sc.bytes = need;
    }
    return cudaSuccess;
}
}  // namespace

cudaError_t launch_length_check(const uint64_t *offsets, uint64_t n, SortScratch &sc,
                                unsigned long long *differ, int sm_count, cudaStream_t stream,
                                uint64_t *launches)
{
    if (n == 0) return cudaSuccess;
    if (n > 0x7fffffffull) return cudaErrorInvalidValue;  // CUB's int item count
    size_t temp;
    cudaError_t e = sort_scratch(n, sc, temp, stream);
    if (e != cudaSuccess) return e;
    uint32_t *idx = (uint32_t *)sc.d_buf + 2 * n;  // identity order (trials equally long)
    ++*launches;
    length_keys_kernel<<<sm_count * 4, 256, 0, stream>>>(offsets, n, nullptr, idx, differ);
    sc.perm = idx;
    return cudaGetLastError();
}

cudaError_t launch_length_sort(const uint64_t *offsets, uint64_t n, SortScratch &sc, int sm_count,
                               cudaStream_t stream, uint64_t *launches, unsigned long long *differ)
{
    if (n == 0) return cudaSuccess;
    if (n > 0x7fffffffull) return cudaErrorInvalidValue;  // CUB's int item count
    size_t temp;
    cudaError_t e = sort_scratch(n, sc, temp, stream);
    if (e != cudaSuccess) return e;
    uint32_t *keys_in = (uint32_t *)sc.d_buf, *keys_out = keys_in + n;
    uint32_t *idx_in = keys_out + n, *idx_out = idx_in + n;
    void *tmp = (void *)(((uintptr_t)(idx_out + n) + 255) & ~(uintptr_t)255);
    ++*launches;
    length_keys_kernel<<<sm_count * 4, 256, 0, stream>>>(offsets, n, keys_in, idx_in, differ);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ++*launches;  // the CUB radix sort (a few internal kernels)
    e = cub::DeviceRadixSort::SortPairsDescending(tmp, temp, keys_in, keys_out, idx_in, idx_out,
                                                  (int)n, 0, 32, stream);
    sc.perm = idx_out;
    return e;
}

cudaError_t launch_hit_probe(const uint64_t *offsets, const uint32_t *ids, uint64_t n_trials,
                             const uint32_t *d_map, uint32_t C, unsigned long long *probe,
                             cudaStream_t stream, uint64_t *launches)
{
    if (n_trials == 0) return cudaSuccess;
    ++*launches;
    hit_probe_kernel<<<kProbeSamples / 256, 256, 0, stream>>>(offsets, ids, n_trials, d_map, C,
                                                               probe);
    return cudaGetLastError();
}

cudaError_t launch_validate(const uint64_t *offsets, const uint32_t *ids, uint64_t n_trials,
                            uint64_t n_ev, uint32_t catalogue_size, uint32_t *err, int sm_count,
                            cudaStream_t stream, uint64_t *launches)
{
    if (n_trials == 0) return cudaSuccess;
    ++*launches;
    validate_kernel<<<sm_count * 8, 256, 0, stream>>>(offsets, ids, n_trials, n_ev,
                                                     catalogue_size, err);
    return cudaGetLastError();
}

}  // namespace ara
