// hoist.cu -- the hoisted scan (ARA_RUN_HOIST): SURVEY.md section 7, "Deferred levers (exact;
// report separately)", finding 6.
//
// Algorithm 1 lines 4-17 (look up the event's loss in every ELT of the layer, apply each ELT's
// financial terms, sum over the ELTs in layer order, apply the occurrence terms; PAPER.md
// L72-L84) depend only on the event and the layer, not on the trial.  Every run therefore first
// evaluates them ONCE per distinct event of the layers' union (U ~ 20,000 events, with exactly
// the scan's fp64 operations in the scan's order), writing the per-event occurrence loss
//     oc[e][l] = min(max(((0 + F_0) + F_1) + ... + F_{E-1} - OccR_l, 0), OccL_l)
// to a table, and the trial scan then reads ONE value per (event occurrence, layer) and runs
// lines 18-29 (running sum S, aggregate terms, difference, trial sum).  Every occurrence of
// event e would have computed exactly oc[e][l] (same inputs, same operations, same order), so
// the YLT is bit-identical to the full scan's and the oracle's.  An event absent from every
// ELT has oc = +0 (reading R12), so the table's entries for absent ids are constant zeros.
//
// Tables (DeviceStore::d_oc): indexed by catalogue id ([(C+1) x LP], map modes 1-2; in mode 2
// a 32 KB presence bitmap in shared memory skips the load of absent ids) or by dense row through
// the catalogue map ([(U+1) x LP], map mode 0).  LP = layers padded to 1, 2, 4 or 8 (the padding layers' entries
// stay zero and their YLT rows are not written).
//
// Trial scan decomposition: one lane per trial (and all its layers); ids are read 8 at a time
// (256-bit loads), the per-event oc vectors (LP values) are gathered a sub-batch at a time.
#include <cuda_runtime.h>
#include <stdint.h>

#include "ara_internal.h"
#include "scan_common.cuh"

namespace ara {
namespace {
using namespace scan_detail;

// Threads per block by layer count: one lane per trial needs many resident warps (LP <= 2:
// ~60 registers -> 2 blocks of 512 per SM), wider oc vectors need more registers.
template <int LP>
constexpr int hoist_threads() { return LP <= 2 ? 512 : (LP == 4 ? 256 : 128); }

// Lines 4-17 for one (dense row u >= 1, layer l): the scan's event_step arithmetic, one lane.
template <typename R>
__global__ void __launch_bounds__(256) hoist_oc_kernel(const R *__restrict__ rows,
                                                       const LayerTermsT<R> *__restrict__ terms,
                                                       const uint32_t *__restrict__ union_ids,
                                                       uint32_t n_union, uint32_t n_layers,
                                                       uint32_t W, uint32_t ilv, uint32_t LP,
                                                       int direct, R *__restrict__ oc)
{
    const uint64_t n = (uint64_t)n_union * n_layers;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t u = (uint32_t)(i / n_layers) + 1, l = (uint32_t)(i % n_layers);
        const LayerTermsT<R> &T = terms[l];
        const R *x = rows + (size_t)u * n_layers * W + (size_t)l * W;
        R lo = R(0);  // lines 11-13: ((0 + F_0) + F_1) + ..., padded columns add +0
        for (uint32_t j = 0; j < W; ++j) {
            const R xj = x[row_phys_col(j, W, ilv)];
            const R f = dmin(dmax0(rsub(rmul(xj, T.rate[j]), T.ret[j])), T.lim[j]);  // line 9
            lo = radd(lo, f);
        }
        const R o = dmin(dmax0(rsub(lo, T.occ_ret)), T.occ_lim);  // line 16
        const uint64_t row = direct ? (uint64_t)union_ids[u - 1] : (uint64_t)u;
        oc[row * LP + l] = o;
    }
}

// The LP values of one table row (LP * sizeof(R) bytes, aligned to that size).  Up to 16 bytes
// the loads allocate in L1 (the table's hot sectors partly fit: headline 4.16 -> 3.81 ms,
// profiles/r1_tune_hoist_l1.jsonl); 32/64-byte rows use the scan's L1-bypassing 256-bit loads.
template <int LP, typename R>
__device__ __forceinline__ void load_oc(const R *p, R (&v)[LP])
{
    constexpr int B = LP * (int)sizeof(R);
    if constexpr (B == 4) {
        asm("ld.global.nc.f32 %0, [%1];" : "=f"(*(float *)&v[0]) : "l"(p));
    } else if constexpr (B == 8) {
        if constexpr (sizeof(R) == 8)
            asm("ld.global.nc.f64 %0, [%1];" : "=d"(*(double *)&v[0]) : "l"(p));
        else
            asm("ld.global.nc.v2.f32 {%0,%1}, [%2];"
                : "=f"(*(float *)&v[0]), "=f"(*(float *)&v[1]) : "l"(p));
    } else if constexpr (B == 16) {
        if constexpr (sizeof(R) == 8)
            asm("ld.global.nc.v2.f64 {%0,%1}, [%2];"
                : "=d"(*(double *)&v[0]), "=d"(*(double *)&v[1]) : "l"(p));
        else
            asm("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
                : "=f"(*(float *)&v[0]), "=f"(*(float *)&v[1]), "=f"(*(float *)&v[2]),
                  "=f"(*(float *)&v[3]) : "l"(p));
    } else {  // 32 or 64 bytes: 256-bit loads
        static_assert(B % 32 == 0, "oc rows are 4, 8, 16, 32 or 64 bytes");
#pragma unroll
        for (int h = 0; h < B / 32; ++h) {
            Chunk<R> c;
            load_row_chunk(p + h * Chunk<R>::N, c);
#pragma unroll
            for (int q = 0; q < Chunk<R>::N; ++q) v[h * Chunk<R>::N + q] = c.v[q];
        }
    }
}

// Table row of catalogue id `id` (or none: absent or out of range -> oc = +0 without a load).
template <int MM>
__device__ __forceinline__ bool oc_row(const RowLookup &L, uint32_t id, bool &bad, uint32_t &row)
{
    const bool ok = (id - 1u) < L.C;
    bad |= !ok;
    if (MM == 0) {
        row = ok ? load_map(L.map + id) : 0u;
        return row != 0u;
    }
    row = id;
    if (MM == 1) return ok;
    const uint32_t h = bitmap_hash(id, L.bitmap_log2);
    return ok && ((L.sbits[h >> 5] >> (h & 31u)) & 1u);
}

template <int LP, typename R, bool BAL, int MM>
__device__ __forceinline__ void hoisted_body(const ScanLaunch &s,
                                             const uint32_t *__restrict__ map,
                                             const uint32_t *__restrict__ bitmap,
                                             const R *__restrict__ oc,
                                             const LayerTermsT<R> *__restrict__ terms,
                                             uint32_t n_layers)
{
    extern __shared__ __align__(16) uint32_t sbits[];  // map mode 2 only
    load_bitmap<MM>(sbits, bitmap, s.bitmap_log2);
    constexpr int SB = LP <= 2 ? 8 : (LP == 4 ? 4 : 2);  // events gathered per sub-batch
    const uint32_t lane = threadIdx.x & 31u;
    const RowLookup look{map, sbits, s.catalogue_size, 0u, s.bitmap_log2};

    R agg_ret[LP], agg_lim[LP];
#pragma unroll
    for (int l = 0; l < LP; ++l) {
        const uint32_t lt = (uint32_t)l < n_layers ? (uint32_t)l : 0u;
        agg_ret[l] = terms[lt].agg_ret;
        agg_lim[l] = terms[lt].agg_lim;
    }
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t warp_g = tid / 32, warps = nthreads / 32;
    const uint64_t base = s.offsets[0];
    bool bad = false;

    for (uint64_t ticket = BAL ? warp_g * 32 + lane : tid;;) {
        if (BAL ? ticket - lane >= s.n_trials : ticket >= s.n_trials) break;  // warp-uniform
        if (ticket < s.n_trials) {
            const uint64_t t = BAL ? (uint64_t)s.perm[ticket] : ticket;
            const uint64_t beg = s.offsets[t] - base;
            const uint64_t k = s.offsets[t + 1] - base - beg;
            const uint32_t *ev = s.ids + beg;
            const uint32_t *const ev_end = ev + k;
            R S[LP], Cp[LP], lr[LP];  // lines 19, 25 (C_0 = 0), 28
#pragma unroll
            for (int l = 0; l < LP; ++l) S[l] = Cp[l] = lr[l] = R(0);
            // lines 18-29 for one event given its oc vector
            auto step = [&](const R (&o)[LP]) {
#pragma unroll
                for (int l = 0; l < LP; ++l) {
                    S[l] = radd(S[l], o[l]);                                     // line 19
                    const R Cd = dmin(dmax0(rsub(S[l], agg_ret[l])), agg_lim[l]);  // line 22
                    lr[l] = radd(lr[l], rsub(Cd, Cp[l]));                        // lines 25, 28
                    Cp[l] = Cd;
                }
            };
            auto fetch = [&](uint32_t id, R (&o)[LP]) {
                uint32_t row;
                if (oc_row<MM>(look, id, bad, row)) {
                    load_oc<LP, R>(oc + (size_t)row * LP, o);
                } else {
#pragma unroll
                    for (int l = 0; l < LP; ++l) o[l] = R(0);
                }
            };
            while (ev < ev_end && ((uintptr_t)ev & 31u) != 0) {  // unaligned head
                R o[LP];
                fetch(load_id(ev), o);
                step(o);
                ++ev;
            }
            const uint64_t n_chunks = (uint64_t)(ev_end - ev) / 8;
            if (n_chunks) {
                uint32_t id_c[8], id_n[8];
                load_ids8(ev, id_c);
#pragma unroll 1
                for (uint64_t i = 0; i < n_chunks; ++i) {
                    if (i + 1 < n_chunks) load_ids8(ev + 8 * (i + 1), id_n);
#pragma unroll
                    for (int b = 0; b < 8; b += SB) {
                        R o[SB][LP];
#pragma unroll
                        for (int j = 0; j < SB; ++j) fetch(id_c[b + j], o[j]);
#pragma unroll
                        for (int j = 0; j < SB; ++j) step(o[j]);
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) id_c[j] = id_n[j];
                }
                ev += 8 * n_chunks;
            }
            while (ev < ev_end) {  // tail
                R o[LP];
                fetch(load_id(ev), o);
                step(o);
                ++ev;
            }
#pragma unroll
            for (int l = 0; l < LP; ++l)
                if ((uint32_t)l < n_layers) s.ylt[(size_t)l * s.ylt_ld + t] = (double)lr[l];  // A8
        }
        if (BAL) {
            __syncwarp();
            uint64_t b = 0;
            if (lane == 0) b = warps + atomicAdd(s.counter, 1ull);
            ticket = __shfl_sync(0xffffffffu, b, 0) * 32 + lane;
        } else {
            ticket += nthreads;
        }
    }
    if (bad) atomicOr(s.err, kErrRange);
    if (BAL) {  // the last block to finish resets the ticket counter for the next launch
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

// Map mode 2 runs the mode-1 body when the hit probe found (nearly) every sampled id present.
template <int LP, typename R, bool BAL, int MM>
__global__ void __launch_bounds__(hoist_threads<LP>())
    hoisted_scan_kernel(const ScanLaunch s, const uint32_t *__restrict__ map,
                        const uint32_t *__restrict__ bitmap, const R *__restrict__ oc,
                        const LayerTermsT<R> *__restrict__ terms, uint32_t n_layers)
{
    if constexpr (MM == 2) {
        if (!probe_use_bitmap(s.probe)) {
            hoisted_body<LP, R, BAL, 1>(s, map, bitmap, oc, terms, n_layers);
            return;
        }
    }
    hoisted_body<LP, R, BAL, MM>(s, map, bitmap, oc, terms, n_layers);
}

template <int LP, typename R, bool BAL, int MM>
cudaError_t launch_hs(const DeviceStore &st, const ScanLaunch &s, int sm_count,
                      cudaStream_t stream)
{
    constexpr int T = hoist_threads<LP>();
    const size_t smem = MM == 2 ? bitmap_bytes(kBitmapLog2Hoist) : 0;
    static std::atomic<int> occ_cache[kMaxDevices];  // resident blocks per SM, per device
    int occ = 0;
    cudaError_t oe = blocks_per_sm((const void *)hoisted_scan_kernel<LP, R, BAL, MM>, T, smem,
                                   occ_cache, occ);
    if (oe != cudaSuccess) return oe;
    // one lane per trial: a balanced single wave where possible
    const uint64_t max_blocks = (uint64_t)sm_count * occ;
    const uint64_t rounds = (s.n_trials + max_blocks * T - 1) / (max_blocks * T);
    const uint64_t slots = (s.n_trials + rounds - 1) / rounds;
    uint64_t blocks = (slots + T - 1) / T;
    if (blocks >= (uint64_t)sm_count) blocks = (blocks + sm_count - 1) / sm_count * sm_count;
    if (blocks > max_blocks) blocks = max_blocks;
    ScanLaunch sl = s;
    sl.bitmap_log2 = kBitmapLog2Hoist;
    static const std::string name = kernel_name("hoisted_scan_kernel", LP,
                                                sizeof(R) == 8 ? "double" : "float", BAL, MM);
    t_last_kernel = name.c_str();
    hoisted_scan_kernel<LP, R, BAL, MM><<<(unsigned)blocks, T, smem, stream>>>(
        sl, st.d_map, st.d_oc_bitmap, (const R *)st.d_oc, (const LayerTermsT<R> *)st.d_terms,
        st.n_layers);
    return cudaGetLastError();
}

template <int LP, typename R, bool BAL>
cudaError_t launch_hm(const DeviceStore &st, const ScanLaunch &s, int sm_count,
                      cudaStream_t stream)
{
    if (st.oc_direct && st.d_oc_bitmap) return launch_hs<LP, R, BAL, 2>(st, s, sm_count, stream);
    if (st.oc_direct) return launch_hs<LP, R, BAL, 1>(st, s, sm_count, stream);
    return launch_hs<LP, R, BAL, 0>(st, s, sm_count, stream);
}

template <typename R, bool BAL>
cudaError_t launch_hl(const DeviceStore &st, const ScanLaunch &s, int sm_count,
                      cudaStream_t stream)
{
    switch (st.oc_lp) {
        case 1: return launch_hm<1, R, BAL>(st, s, sm_count, stream);
        case 2: return launch_hm<2, R, BAL>(st, s, sm_count, stream);
        case 4: return launch_hm<4, R, BAL>(st, s, sm_count, stream);
        case 8: return launch_hm<8, R, BAL>(st, s, sm_count, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

cudaError_t launch_hoist_oc(const DeviceStore &st, cudaStream_t stream, uint64_t *launches)
{
    if (st.n_union == 0) return cudaSuccess;
    ++*launches;
    const uint64_t n = (uint64_t)st.n_union * st.n_layers;
    const unsigned blocks = (unsigned)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
    if (st.bits == 32)
        hoist_oc_kernel<float><<<blocks, 256, 0, stream>>>(
            (const float *)st.d_rows, (const LayerTermsT<float> *)st.d_terms, st.d_union_ids,
            st.n_union, st.n_layers, st.width, st.ilv, st.oc_lp, st.oc_direct, (float *)st.d_oc);
    else
        hoist_oc_kernel<double><<<blocks, 256, 0, stream>>>(
            (const double *)st.d_rows, (const LayerTermsT<double> *)st.d_terms, st.d_union_ids,
            st.n_union, st.n_layers, st.width, st.ilv, st.oc_lp, st.oc_direct, (double *)st.d_oc);
    return cudaGetLastError();
}

cudaError_t launch_hoisted_scan(const DeviceStore &st, const ScanLaunch &s, int sm_count,
                                cudaStream_t stream, uint64_t *launches)
{
    if (s.n_trials == 0) return cudaSuccess;
    ++*launches;
    const bool bal = s.perm != nullptr;
    if (st.bits == 32)
        return bal ? launch_hl<float, true>(st, s, sm_count, stream)
                   : launch_hl<float, false>(st, s, sm_count, stream);
    return bal ? launch_hl<double, true>(st, s, sm_count, stream)
               : launch_hl<double, false>(st, s, sm_count, stream);
}

}  // namespace ara
