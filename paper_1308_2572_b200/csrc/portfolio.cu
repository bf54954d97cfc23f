// portfolio.cu -- layer-fused union-row scan for multi-layer portfolios (
// Algorithm 1 line 2).
//
// The ELTs of all layers form one union set J (|J| <= 64).  Per event the kernel reads the id once,
// looks up the shared catalogue map once, gathers ONE union row (the event's losses in every ELT
// of J, 8|J| bytes), applies each ELT's financial terms ONCE (they are per ELT, reading R1), and
// then every layer sums its own columns in its own listed order (lines 11-13), applies its own
// occurrence and aggregate terms (lines 15-29) and writes its YLT entry.  Compared with per-layer
// rows this halves the gathered bytes and the financial-term work when every ELT is shared by two
// layers (configuration P).
//
// Decomposition: a group of GU lanes per trial (GU = 8 for 64 union columns).  Lane c owns the
// 32-byte chunks c and c + GU of the union row (columns 4c..4c+3 and 4(c+GU)..4(c+GU)+3) and their
// financial terms; the two gather instructions of a group each cover 32*GU contiguous bytes.  The
// lanes write their F values to a per-group shared-memory row; after a warp-level barrier lane l
// sums layer l's columns in layer order, ((0 + F_{c_l0}) + F_{c_l1}) + ..., exactly the oracle's
// sequence, and carries layer l's running state.  Padding entries of a layer's column list point
// at a zero slot (+0 is exactly neutral, reading R12).
//
// Block variant (SH = 3): when every layer is two blocks of 8 ELTs and the blocks partition J
// (configuration P: layer l = block l then block l + 1), lane l holds layer l's first block in
// its registers 0-7 and the second comes from one lane by 8 shuffles: half the shuffles of SH = 2
// (the shuffles were the L1 data pipe's largest consumer: 8 wavefronts per trial-event against 4
// for the union row).
//
// Register-shuffle variant (SH = 1, 2; UnionStore::shfl): when every ELT takes positions of one
// residue mod 8 in all layers that hold it (configuration P), ara_set_layers places the ELT of
// residue r in register r of some lane, so position i of EVERY layer is register i mod 8 of a
// lane src(l, i): each position is one 64-bit shuffle per group, with no shared-memory writes,
// reads or barriers (the shared F row cost 2 L1 wavefronts per trial-layer-event, the shuffles
// cost 1).  SH = 2: every layer has 16 ELTs; SH = 1: shorter layers add +0 past their end.
//
// SC = 1: the exactly scaled clamps of scan_pair.cu (reading R16): F2 = min(x + |x|,
// 2 lim), lo2, oc4, S4, C8, lr8, YLT = lr8 * 0.125 -- the oracle's bits with one DADD per clamp
// instead of DSETP + 2 FSEL (inputs below 2^960, UnionStore::scaled).
#include <cuda_runtime.h>
#include <stdint.h>

#include "ara_internal.h"
#include "scan_common.cuh"

namespace ara {
namespace {
using namespace scan_detail;

// Shared-memory F row of one group: 8 doubles per 8 union columns plus 2 padding doubles, then a
// zero pair; the group stride is odd (1 mod 16 doubles) so that the 32 lanes' 8-byte reads of
// configuration P's layer columns hit every bank pair exactly twice (2 wavefronts, the minimum).
__host__ __device__ constexpr int u_slot(int col) { return col + 2 * (col >> 3); }
template <int GU>
__host__ __device__ constexpr int u_row_doubles()
{
    return (u_slot(8 * GU) + 2 + 15) / 16 * 16 + 1;
}

__device__ __forceinline__ double twice_max0(double x) { return __dadd_rn(x, fabs(x)); }
__device__ __forceinline__ double cmin(double m, double lim) { return (lim < m) ? lim : m; }

template <int GU, bool BAL, int MM, int SH, int SC>
__device__ __forceinline__ void portfolio_body(const ScanLaunch &s,
                                               const uint32_t *__restrict__ map,
                                               const uint32_t *__restrict__ bitmap,
                                               const double *__restrict__ urows,
                                               const UnionTermsDev *__restrict__ ut)
{
    extern __shared__ __align__(16) uint32_t sbits[];  // map mode 2 only
    load_bitmap<MM>(sbits, bitmap, s.bitmap_log2);
    constexpr int WU = 8 * GU;              // union row width (doubles)
    constexpr int GS = u_row_doubles<GU>(); // shared F row stride per group (doubles)
    constexpr int ZERO = u_slot(WU);        // index of the zero pair
    __shared__ double sF[SH == 0 ? (kScanThreads / GU) * GS : 2];

    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t c = lane % GU;
    const uint32_t gmask = (GU == 32) ? 0xffffffffu : (((1u << GU) - 1u) << (lane - c));
    const uint32_t gb = threadIdx.x / GU;   // group index in the block
    double *const myF = sF + gb * GS;
    if (SH == 0 && c == 0) {
        myF[ZERO] = 0.0;
        myF[ZERO + 1] = 0.0;
    }

    // financial terms of this lane's 8 union columns
    double rate[8], ret[8], lim[8];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int col = 4 * (c + GU * h) + q;
            rate[4 * h + q] = ut->rate[col];
            ret[4 * h + q] = ut->ret[col];
            lim[4 * h + q] = (SC ? 2.0 : 1.0) * ut->lim[col];  // SC: 2 lim
        }
    // this lane's layer (lane c -> layer c): terms and the shared-memory slots of its columns
    const uint32_t n_layers = ut->n_layers;
    const bool has_layer = c < n_layers;
    const uint32_t ly = has_layer ? c : 0;
    // SC: 2 OccR, 4 OccL, 4 AggR, 8 AggL (the scaled domain of reading R16)
    const double occ_ret = (SC ? 2.0 : 1.0) * ut->occ_ret[ly];
    const double occ_lim = (SC ? 4.0 : 1.0) * ut->occ_lim[ly];
    const double agg_ret = (SC ? 4.0 : 1.0) * ut->agg_ret[ly];
    const double agg_lim = (SC ? 8.0 : 1.0) * ut->agg_lim[ly];
    uint32_t slot2[SH == 0 ? kUnionMaxE / 2 : 1];  // two 16-bit slots per register
    if constexpr (SH == 0) {
#pragma unroll
        for (int i = 0; i < kUnionMaxE / 2; ++i) slot2[i] = ut->slot2[ly][i];
    }
    // register-shuffle layout: source lane of each position (5-bit fields; shfl uses bits 4:0)
    uint32_t src5[3] = {0, 0, 0};
    uint32_t my_n = 0;
    const uint32_t src2 = SH == 3 ? ut->src2[ly] : 0;
    if constexpr (SH == 1 || SH == 2) {
#pragma unroll
        for (int i = 0; i < 3; ++i) src5[i] = ut->src5[ly][i];
        my_n = has_layer ? ut->n_cols[ly] : 0;
    }
    double *const ylt_row = s.ylt + (size_t)ly * s.ylt_ld;
    const double *__restrict__ my_rows = urows + 4 * c;
    const uint32_t zb = s.zero_base;
    const RowLookup look{map, sbits, s.catalogue_size, zb, s.bitmap_log2};
    __syncwarp();

    // one event: F of this lane's columns -> shared row -> this lane's layer sum and state
    auto event = [&](const Chunk<double> (&r)[2], double &S, double &Cprev, double &lr,
                     double &own) {
        double f[8];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = 4 * h + q;
                const double l = rsub(rmul(r[h].v[q], rate[j]), ret[j]);  // line 9
                f[j] = SC ? cmin(twice_max0(l), lim[j]) : dmin(dmax0(l), lim[j]);
            }
        double lo = 0.0;  // lines 11-13 for this lane's layer, in the layer's ELT order
        if constexpr (SH == 0) {
            __syncwarp(gmask);  // the previous event's reads of the shared row are done
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double *dst = myF + u_slot(4 * (c + GU * h));
#pragma unroll
                for (int q = 0; q < 4; ++q) dst[q] = f[4 * h + q];
            }
            __syncwarp(gmask);
#pragma unroll
            for (int i = 0; i < kUnionMaxE; ++i) {
                const uint32_t sl = (slot2[i >> 1] >> (16 * (i & 1))) & 0xffffu;
                lo = radd(lo, myF[sl]);
            }
        } else if constexpr (SH == 3) {
            // block layout: positions 0-7 are this lane's own registers, positions 8-15
            // registers 0-7 of lane src2 -- 8 shuffles per event instead of 16
#pragma unroll
            for (int i = 0; i < 8; ++i) lo = radd(lo, f[i]);
#pragma unroll
            for (int i = 0; i < 8; ++i) lo = radd(lo, __shfl_sync(gmask, f[i], src2, GU));
        } else {
            // position i of every layer lives in register i mod 8 (of lane src(l, i)): one
            // 64-bit shuffle per position serves all layers of the group, no shared memory
#pragma unroll
            for (int i = 0; i < kUnionMaxE; ++i) {
                const uint32_t sl = src5[i / 6] >> (5 * (i % 6));
                if constexpr (SH == 2) {  // shuffle + add in one PTX block (2% faster:
                                          // fewer register-pair moves, r1_tune_portfolio_ptxadd)
                    asm("{\n\t.reg .b32 l32, h32;\n\t.reg .f64 v;\n\t"
                        "mov.b64 {l32, h32}, %2;\n\t"
                        "shfl.sync.idx.b32 l32, l32, %3, %4, %5;\n\t"
                        "shfl.sync.idx.b32 h32, h32, %3, %4, %5;\n\t"
                        "mov.b64 v, {l32, h32};\n\tadd.rn.f64 %0, %1, v;\n\t}"
                        : "=d"(lo) : "d"(lo), "d"(f[i % 8]), "r"(sl),
                          "n"(((32 - GU) << 8) | 0x1f), "r"(gmask));
                    continue;
                }
                double v = __shfl_sync(gmask, f[i % 8], sl, GU);
                if (SH == 1) v = (uint32_t)i < my_n ? v : 0.0;  // past the layer's ELTs: +0
                lo = radd(lo, v);
            }
        }
        own = lo;  // (pinning the gathers on lo instead of S measured 4% slower here)
        const double t = rsub(lo, occ_ret);
        const double oc = SC ? cmin(twice_max0(t), occ_lim) : dmin(dmax0(t), occ_lim);  // l. 16
        S = radd(S, oc);                                                                // l. 19
        const double u = rsub(S, agg_ret);
        const double Cd = SC ? cmin(twice_max0(u), agg_lim) : dmin(dmax0(u), agg_lim);  // l. 22
        lr = radd(lr, rsub(Cd, Cprev));                               // lines 25, 28
        Cprev = Cd;
    };
    auto gather = [&](uint32_t idx, Chunk<double> (&r)[2]) {
        const double *p = my_rows + (size_t)idx * WU;
        load_row_chunk(p, r[0]);
        load_row_chunk(p + 4 * GU, r[1]);
    };

    constexpr uint32_t B = 32 / GU;  // groups per warp
    const uint32_t gw = lane / GU;
    const uint64_t g = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / GU;
    const uint64_t groups = ((uint64_t)gridDim.x * blockDim.x) / GU;
    const uint64_t warp_g = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) / 32;
    const uint64_t base = s.offsets[0];
    bool bad = false;
    for (uint64_t ticket = BAL ? warp_g * B + gw : g;;) {
        if (BAL ? ticket - gw >= s.n_trials : ticket >= s.n_trials) break;  // warp-uniform
        if (ticket < s.n_trials) {
            const uint64_t t = BAL ? (uint64_t)s.perm[ticket] : ticket;
            const uint64_t beg = s.offsets[t] - base;
            const uint64_t k = s.offsets[t + 1] - base - beg;
            const uint32_t *ev = s.ids + beg;
            const uint32_t *const ev_end = ev + k;
            double S = 0.0, Cprev = 0.0, lr = 0.0, own = 0.0;
            while (ev < ev_end && ((uintptr_t)ev & 31u) != 0) {  // unaligned head
                Chunk<double> r[2];
                gather(row_index<MM>(look, load_id(ev), bad), r);
                event(r, S, Cprev, lr, own);
                ++ev;
            }
            const uint64_t n_chunks = (uint64_t)(ev_end - ev) / 8;
            if (n_chunks) {
                uint32_t id_c[8], id_n[8];
                load_ids8(ev, id_c);
                if (n_chunks > 1) load_ids8(ev + 8, id_n);
                uint32_t idx1 = row_index<MM>(look, id_c[1], bad);
                Chunk<double> ra[2];
                gather(row_index<MM>(look, id_c[0], bad), ra);
#pragma unroll 1
                for (uint64_t i = 0; i < n_chunks; ++i) {
                    const bool more = i + 1 < n_chunks;
#pragma unroll
                    for (int j = 0; j < 8; j += 2) {
                        const uint32_t id2 = j + 2 < 8 ? id_c[j + 2] : id_n[0];
                        const uint32_t id3 = j + 3 < 8 ? id_c[j + 3] : id_n[1];
                        const bool ok2 = j + 2 < 8 || more;
                        const uint32_t idx2 = ok2 ? row_index<MM>(look, id2, bad) : zb;
                        Chunk<double> rb[2];
                        gather(pin(idx1, S), rb);
                        event(ra, S, Cprev, lr, own);
                        const uint32_t idx3 = ok2 ? row_index<MM>(look, id3, bad) : zb;
                        gather(pin(idx2, S), ra);
                        event(rb, S, Cprev, lr, own);
                        idx1 = idx3;
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) id_c[j] = id_n[j];
                    if (i + 2 < n_chunks) load_ids8(ev + 8 * (i + 2), id_n);
                }
                ev += 8 * n_chunks;
            }
            while (ev < ev_end) {  // tail
                Chunk<double> r[2];
                gather(row_index<MM>(look, load_id(ev), bad), r);
                event(r, S, Cprev, lr, own);
                ++ev;
            }
            if (has_layer) ylt_row[t] = SC ? lr * 0.125 : lr;  // A8, one entry per layer
        }
        if (BAL) {
            __syncwarp();
            uint64_t b = 0;
            if (lane == 0) b = warps + atomicAdd(s.counter, 1ull);
            ticket = __shfl_sync(0xffffffffu, b, 0) * B + gw;
        } else if (s.counter) {
            uint64_t next = 0;
            if (c == 0) next = groups + atomicAdd(s.counter, 1ull);
            ticket = __shfl_sync(gmask, next, lane - c);
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

// Map mode 2 runs the mode-1 body when the hit probe found (nearly) every sampled id present.
template <int GU, bool BAL, int MM, int SH, int SC>
__global__ void __launch_bounds__(kScanThreads, 3)
    portfolio_kernel(const ScanLaunch s, const uint32_t *__restrict__ map,
                     const uint32_t *__restrict__ bitmap, const double *__restrict__ urows,
                     const UnionTermsDev *__restrict__ ut)
{
    if constexpr (MM == 2) {
        if (!probe_use_bitmap(s.probe)) {
            portfolio_body<GU, BAL, 1, SH, SC>(s, map, bitmap, urows, ut);
            return;
        }
    }
    portfolio_body<GU, BAL, MM, SH, SC>(s, map, bitmap, urows, ut);
}

template <int GU, bool BAL, int MM, int SH, int SC>
cudaError_t launch_pum(const UnionStore &us, const uint32_t *d_map, const uint32_t *d_bitmap,
                       const ScanLaunch &s, int sm_count, cudaStream_t stream)
{
    const size_t smem = MM == 2 ? bitmap_bytes(kBitmapLog2Union) : 0;
    static std::atomic<int> occ_cache[kMaxDevices];  // resident blocks per SM, per device
    int occ = 0;
    cudaError_t oe = blocks_per_sm((const void *)portfolio_kernel<GU, BAL, MM, SH, SC>,
                                   kScanThreads, smem, occ_cache, occ);
    if (oe != cudaSuccess) return oe;
    const uint64_t per_block = kScanThreads / GU;
    const uint64_t max_blocks = (uint64_t)sm_count * occ;
    const uint64_t rounds = (s.n_trials + max_blocks * per_block - 1) / (max_blocks * per_block);
    const uint64_t slots = (s.n_trials + rounds - 1) / rounds;
    uint64_t blocks = (slots + per_block - 1) / per_block;
    if (blocks >= (uint64_t)sm_count) blocks = (blocks + sm_count - 1) / sm_count * sm_count;
    if (blocks > max_blocks) blocks = max_blocks;
    ScanLaunch sl = s;
    sl.zero_base = MM ? us.zero_base_direct : us.zero_base;
    sl.bitmap_log2 = kBitmapLog2Union;
    static const std::string name = kernel_name("portfolio_kernel", GU, BAL, MM, SH, SC);
    t_last_kernel = name.c_str();
    portfolio_kernel<GU, BAL, MM, SH, SC><<<(unsigned)blocks, kScanThreads, smem, stream>>>(
        sl, d_map, d_bitmap, MM ? us.d_rows_direct : us.d_rows, us.d_terms);
    return cudaGetLastError();
}

template <int GU, bool BAL, int SH, int SC>
cudaError_t launch_pus(const UnionStore &us, const uint32_t *d_map, int map_mode,
                       const uint32_t *d_bitmap, const ScanLaunch &s, int sm_count,
                       cudaStream_t stream)
{
    if (map_mode == 1) return launch_pum<GU, BAL, 1, SH, SC>(us, d_map, d_bitmap, s, sm_count, stream);
    if (map_mode == 2) return launch_pum<GU, BAL, 2, SH, SC>(us, d_map, d_bitmap, s, sm_count, stream);
    return launch_pum<GU, BAL, 0, SH, SC>(us, d_map, d_bitmap, s, sm_count, stream);
}

// Layer-sum variant (UnionStore::shfl); the shuffle variants are built for GU = 8 (up to 64
// union columns and 8 layers, configuration P), smaller unions use the shared-memory F row.
template <int GU, bool BAL>
cudaError_t launch_pu(const UnionStore &us, const uint32_t *d_map, int map_mode,
                      const uint32_t *d_bitmap, const ScanLaunch &s, int sm_count,
                      cudaStream_t stream)
{
    if constexpr (GU == 8) {
        if (us.shfl == 3) {  // block layout (configuration P), scaled clamps when allowed
            if constexpr (BAL)
                if (us.scaled)
                    return launch_pus<GU, BAL, 3, 1>(us, d_map, map_mode, d_bitmap, s, sm_count,
                                                     stream);
            return launch_pus<GU, BAL, 3, 0>(us, d_map, map_mode, d_bitmap, s, sm_count, stream);
        }
        if (us.shfl == 2) {  // configuration P: the scaled clamps when the inputs allow them
            if constexpr (BAL)
                if (us.scaled)
                    return launch_pus<GU, BAL, 2, 1>(us, d_map, map_mode, d_bitmap, s, sm_count,
                                                     stream);
            return launch_pus<GU, BAL, 2, 0>(us, d_map, map_mode, d_bitmap, s, sm_count, stream);
        }
        if (us.shfl == 1)
            return launch_pus<GU, BAL, 1, 0>(us, d_map, map_mode, d_bitmap, s, sm_count, stream);
    }
    return launch_pus<GU, BAL, 0, 0>(us, d_map, map_mode, d_bitmap, s, sm_count, stream);
}

}  // namespace

cudaError_t launch_portfolio(const UnionStore &us, const uint32_t *d_map, int map_mode,
                             const uint32_t *d_bitmap, const ScanLaunch &s, int sm_count,
                             cudaStream_t stream, uint64_t *launches)
{
    if (s.n_trials == 0) return cudaSuccess;
    ++*launches;
    const bool bal = s.perm != nullptr;
    switch (us.GU) {
        case 2: return bal ? launch_pu<2, true>(us, d_map, map_mode, d_bitmap, s, sm_count, stream)
                           : launch_pu<2, false>(us, d_map, map_mode, d_bitmap, s, sm_count, stream);
        case 4: return bal ? launch_pu<4, true>(us, d_map, map_mode, d_bitmap, s, sm_count, stream)
                           : launch_pu<4, false>(us, d_map, map_mode, d_bitmap, s, sm_count, stream);
        case 8: return bal ? launch_pu<8, true>(us, d_map, map_mode, d_bitmap, s, sm_count, stream)
                           : launch_pu<8, false>(us, d_map, map_mode, d_bitmap, s, sm_count, stream);
        default: --*launches; return cudaErrorInvalidValue;
    }
}

}  // namespace ara
