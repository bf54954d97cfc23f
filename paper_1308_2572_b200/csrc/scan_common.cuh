// scan_common.cuh -- device helpers shared by the scan kernels (scan.cu) and the union-row
// portfolio kernel (portfolio.cu).  Internal to libara.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "ara_internal.h"

namespace ara {
namespace scan_detail {

constexpr int kScanThreads = 128;  // 4 warps: fine occupancy steps for 80-170 registers
// F4 increment staging: one 8-double slot per group, padded to 9 doubles so that the writer
// lanes' per-event 8-byte stores of the 16 groups of a warp fall in distinct bank pairs (an
// 8-double stride put 8 groups on one bank pair: an 8-way conflict per event)
constexpr int kStageStride = 9;

// One 32-byte chunk of a row: 4 doubles (fp64 store) or 8 floats (fp32 store, F3).
template <typename R>
struct Chunk {
    static constexpr int N = 32 / (int)sizeof(R);
    R v[N];
};

__device__ __forceinline__ void load_row_chunk(const double *p, Chunk<double> &r)
{
    asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
        : "l"(p));
}

__device__ __forceinline__ void load_row_chunk(const float *p, Chunk<float> &r)
{
    asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
          "=f"(r.v[6]), "=f"(r.v[7])
        : "l"(p));
}

// F4 increment stores (8 GB at the headline): L2 evict-first, so the stream of writes does not
// displace the L2-resident rows every event gathers (with evict-normal stores 6 GB of row
// re-reads from DRAM appeared per launch: ncu lts__t_sectors_srcunit_tex_op_read_lookup_miss).
__device__ __forceinline__ uint64_t l2_evict_first_policy()
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void store_v2(double *p, double a, double b)
{
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p),
                 "d"(a), "d"(b), "l"(l2_evict_first_policy())
                 : "memory");
}
__device__ __forceinline__ void store_v4(double *p, double a, double b, double c, double d)
{
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p),
                 "d"(a), "d"(b), "d"(c), "d"(d), "l"(l2_evict_first_policy())
                 : "memory");
}

// Separately rounded arithmetic in the store's precision (no FMA contraction).
__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double rsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float rmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float rsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float radd(float a, float b) { return __fadd_rn(a, b); }

__device__ __forceinline__ void load_ids8(const uint32_t *p, uint32_t (&v)[8])
{
    asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7])
        : "l"(p));
}

__device__ __forceinline__ uint32_t load_id(const uint32_t *p)
{
    uint32_t v;
    asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ uint32_t load_map(const uint32_t *p)
{
    uint32_t v;
    asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// min(x, y) = (y < x ? y : x); max(x, 0) = (x < 0 ? 0 : x)   (the oracle's definitions)
template <typename R>
__device__ __forceinline__ R dmin(R x, R y) { return (y < x) ? y : x; }
template <typename R>
__device__ __forceinline__ R dmax0(R x) { return (x < R(0)) ? R(0) : x; }
// fp32 (F3): one FMNMX instead of FSETP + FSEL.  Equal to the compare-select for every non-NaN
// operand pair except a +0/-0 tie, where the sign of a zero may differ; a zero's sign never
// changes a sum on the scan path (reading R12), so the YLT is unchanged.  (sm_100a has
// no fp64 min/max instruction: the fp64 path keeps the compare-select.)
template <>
__device__ __forceinline__ float dmin<float>(float x, float y) { return fminf(x, y); }
template <>
__device__ __forceinline__ float dmax0<float>(float x) { return fmaxf(x, 0.0f); }

__device__ __forceinline__ uint32_t map_index(const uint32_t *__restrict__ map, uint32_t id,
                                              uint32_t C, bool &bad)
{
    const bool ok = (id - 1u) < C;  // id in [1, C]
    bad |= !ok;
    return load_map(map + (ok ? id : 0u));  // map[0] == 0: the zero row
}

// A3 for every map mode (ara_internal.h DeviceStore::map_mode): the row that holds catalogue id
// `id`'s losses.  0: dense row map[id] (one 4-byte L2 read per event); 1: row id of the direct
// store (no read: the L1 data pipe is the scan's binding resource and the map read was a third
// of its wavefronts); 2: as 1 behind the shared-memory presence bitmap `sbits`, so absent ids
// read an L2-resident zero row instead of a cold line of the direct store.  Absent and
// out-of-range ids read a zero row of the zero-row block (ara_internal.h kZeroRows); out-of-range
// ids also raise `bad`.
struct RowLookup {
    const uint32_t *__restrict__ map;  // mode 0: catalogue map
    const uint32_t *sbits;             // mode 2: presence bitmap in shared memory
    uint32_t C;                        // catalogue size
    uint32_t zero_base;                // first row of the zero-row block
    uint32_t bitmap_log2;              // mode 2: log2 of the bitmap's bit count
};

// Mode 2, per launch: consult the bitmap unless the hit probe (ScanLaunch::probe, written by
// hit_probe_kernel before the scan) says >= 99% of the YET's sampled ids are in the store; the
// kernels then run their mode-1 body (a separate instantiation chosen once at kernel entry --
// a per-event runtime test in the hot loop cost 20%).
__device__ __forceinline__ bool probe_use_bitmap(const unsigned long long *probe)
{
    if (probe == nullptr) return true;
    const unsigned long long hit = probe[0], cnt = probe[1];
    return !(cnt > 0 && 100ull * hit >= 99ull * cnt);
}

template <int MM>
__device__ __forceinline__ uint32_t row_index(const RowLookup &L, uint32_t id, bool &bad)
{
    const bool ok = (id - 1u) < L.C;  // id in [1, C]
    bad |= !ok;
    const uint32_t z = L.zero_base + (id & (kZeroRows - 1u));  // a zero row (absent, out of range)
    if (MM == 0) {
        const uint32_t r = load_map(L.map + (ok ? id : 0u));  // map[0] == 0
        return r ? r : z;
    }
    if (MM == 1) return ok ? id : z;
    const uint32_t h = bitmap_hash(id, L.bitmap_log2);
    const uint32_t w = L.sbits[h >> 5];
    return (ok && ((w >> (h & 31u)) & 1u)) ? id : z;
}

// Mode 2: copy the presence bitmap into this block's shared memory (16-byte loads).
template <int MM>
__device__ __forceinline__ void load_bitmap(uint32_t *sbits, const uint32_t *__restrict__ bitmap,
                                            uint32_t log2_bits)
{
    if (MM != 2) return;
    const uint4 *src = reinterpret_cast<const uint4 *>(bitmap);
    uint4 *dst = reinterpret_cast<uint4 *>(sbits);
    const uint32_t n16 = 1u << (log2_bits - 7);
    for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = src[i];
    __syncthreads();
}

// A row gather is issued only after the values it will overwrite have been consumed: `pin`
// gives the row index a true data dependency on such a value v (min with 2^32 - 1 - signbit(v),
// which leaves every row index unchanged because indices are < 2^32 - 1); without it ptxas
// hoists the gathers of an unrolled chunk above the arithmetic that frees their registers and
// runs out of registers.  v must be the EARLIEST value computed from the slot's data (the
// lane's own-column partial sum, or an F value), not the end of the event's serial chain (the
// running sum S): pinning on S serialised every event's gather behind the previous event's
// shuffle + occurrence/aggregate chain.
__device__ __forceinline__ uint32_t pin(uint32_t idx, double v)
{
    const uint32_t sbit = (uint32_t)__double2hiint(v) >> 31;
    return min(idx, 0xffffffffu - sbit);
}

__device__ __forceinline__ uint32_t pin(uint32_t idx, float v)
{
    const uint32_t sbit = __float_as_uint(v) >> 31;
    return min(idx, 0xffffffffu - sbit);
}

}  // namespace scan_detail
}  // namespace ara
