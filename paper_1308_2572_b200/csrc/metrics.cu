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
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ara_internal.h"

namespace cg = cooperative_groups;

namespace ara {
namespace {

constexpr int kThreads = 256;
constexpr int kBins = 256;
constexpr int kPasses = 8;

struct MetricsParams {
    const double *v;
    uint64_t n;
    uint32_t n_p;
    uint64_t rank[ARA_MAX_P];      // 0-based target ranks ceil(p n) - 1
    uint32_t *hist;                // [kPasses][ARA_MAX_P][kBins]
    double *part_sum;              // [grid][ARA_MAX_P]
    unsigned long long *part_cnt;  // [grid][ARA_MAX_P]
    double *out;                   // [2][n_p]: pml, tvar
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

__global__ void __launch_bounds__(kThreads) metrics_kernel(const __grid_constant__ MetricsParams P)
{
    cg::grid_group grid = cg::this_grid();
    __shared__ uint32_t sh[ARA_MAX_P][kBins];
    __shared__ uint64_t s_prefix[ARA_MAX_P];
    __shared__ uint64_t s_rank[ARA_MAX_P];
    __shared__ double s_red[kThreads / 32];
    __shared__ unsigned long long s_redc[kThreads / 32];

    const uint32_t n_p = P.n_p;
    const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;

    for (uint64_t i = gtid; i < (uint64_t)kPasses * ARA_MAX_P * kBins; i += gstride) P.hist[i] = 0;
    if (threadIdx.x < n_p) {
        s_prefix[threadIdx.x] = 0;
        s_rank[threadIdx.x] = P.rank[threadIdx.x];
    }
    grid.sync();

    for (int pass = 0; pass < kPasses; ++pass) {
        const int shift = 56 - 8 * pass;
        const uint64_t mask = pass == 0 ? 0ull : (~0ull << (shift + 8));
        for (uint32_t i = threadIdx.x; i < n_p * kBins; i += blockDim.x) (&sh[0][0])[i] = 0;
        __syncthreads();
        for (uint64_t e = gtid; e < P.n; e += gstride) {
            const uint64_t key = to_key(P.v[e]);
            for (uint32_t i = 0; i < n_p; ++i)
                if ((key & mask) == (s_prefix[i] & mask))
                    atomicAdd(&sh[i][(key >> shift) & 0xff], 1u);
        }
        __syncthreads();
        uint32_t *gh = P.hist + (size_t)pass * ARA_MAX_P * kBins;
        for (uint32_t i = threadIdx.x; i < n_p * kBins; i += blockDim.x) {
            const uint32_t c = (&sh[0][0])[i];
            if (c) atomicAdd(gh + i, c);
        }
        grid.sync();
        if (threadIdx.x < n_p) {  // every block walks the same global histogram
            const uint32_t i = threadIdx.x;
            uint64_t r = s_rank[i], cum = 0;
            for (int b = 0; b < kBins; ++b) {
                const uint64_t c = __ldcg(gh + (size_t)i * kBins + b);
                if (r < cum + c) {
                    s_prefix[i] |= (uint64_t)b << shift;
                    s_rank[i] = r - cum;
                    break;
                }
                cum += c;
            }
        }
        __syncthreads();
    }

    // Tail sums over this block's contiguous chunk, per probability, in a fixed order.  The sum
    // is of (v - PML) >= 0, so TVaR = PML + mean(v - PML) >= PML holds exactly and the
    // rounding error scales with the tail's spread, not its level.
    const uint64_t chunk = (P.n + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = (uint64_t)blockIdx.x * chunk;
    const uint64_t hi = lo + chunk < P.n ? lo + chunk : P.n;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t i = 0; i < n_p; ++i) {
        const uint64_t q = s_prefix[i];
        const double qv = from_key(q);
        double s = 0.0;
        unsigned long long c = 0;
        for (uint64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
            const double x = P.v[e];
            if (to_key(x) >= q) {
                s += x - qv;
                ++c;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            s += __shfl_down_sync(0xffffffffu, s, o);
            c += __shfl_down_sync(0xffffffffu, c, o);
        }
        if (lane == 0) {
            s_red[warp] = s;
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
            P.part_sum[(size_t)blockIdx.x * ARA_MAX_P + i] = bs;
            P.part_cnt[(size_t)blockIdx.x * ARA_MAX_P + i] = bc;
        }
        __syncthreads();
    }
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x < n_p) {
        const uint32_t i = threadIdx.x;
        double s = 0.0;
        unsigned long long c = 0;
        for (uint32_t b = 0; b < gridDim.x; ++b) {
            s += __ldcg(P.part_sum + (size_t)b * ARA_MAX_P + i);
            c += __ldcg(P.part_cnt + (size_t)b * ARA_MAX_P + i);
        }
        const double q = from_key(s_prefix[i]);
        P.out[i] = q;
        P.out[n_p + i] = q + s / (double)c;
    }
}

}  // namespace

cudaError_t launch_metrics(const double *d_row, uint64_t n, uint32_t n_p, const double *p,
                           double *pml_out, double *tvar_out, MetricsScratch &scratch,
                           int sm_count, int device, cudaStream_t stream, uint64_t *launches)
{
    cudaError_t e;
    if (scratch.d_buf == nullptr) {
        int occ = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, metrics_kernel, kThreads, 0);
        if (e != cudaSuccess) return e;
        int coop = 0;
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
        if (!coop || occ < 1) return cudaErrorNotSupported;
        scratch.grid = sm_count * (occ < 2 ? occ : 2);
        scratch.bytes = (size_t)kPasses * ARA_MAX_P * kBins * 4 +
                        (size_t)scratch.grid * ARA_MAX_P * 16 + 2 * ARA_MAX_P * 8;
        e = cudaMalloc(&scratch.d_buf, scratch.bytes);
        if (e != cudaSuccess) return e;
    }
    MetricsParams P{};
    P.v = d_row;
    P.n = n;
    P.n_p = n_p;
    for (uint32_t i = 0; i < n_p; ++i) {
        // nearest rank, computed in fp64 exactly as the reading states: ceil(p * n)
        uint64_t r = (uint64_t)ceil(p[i] * (double)n);
        if (r < 1) r = 1;
        if (r > n) r = n;
        P.rank[i] = r - 1;
    }
    char *b = (char *)scratch.d_buf;
    P.hist = (uint32_t *)b;
    b += (size_t)kPasses * ARA_MAX_P * kBins * 4;
    P.part_sum = (double *)b;
    b += (size_t)scratch.grid * ARA_MAX_P * 8;
    P.part_cnt = (unsigned long long *)b;
    b += (size_t)scratch.grid * ARA_MAX_P * 8;
    P.out = (double *)b;
    int grid = scratch.grid;
    const uint64_t want = (n + kThreads - 1) / kThreads;
    if ((uint64_t)grid > want) grid = (int)want;
    void *args[] = {&P};
    ++*launches;
    e = cudaLaunchCooperativeKernel((void *)metrics_kernel, grid, kThreads, args, 0, stream);
    if (e != cudaSuccess) return e;
    double host[2 * ARA_MAX_P];
    e = cudaMemcpyAsync(host, P.out, 2 * n_p * sizeof(double), cudaMemcpyDeviceToHost, stream);
    if (e != cudaSuccess) return e;
    e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return e;
    for (uint32_t i = 0; i < n_p; ++i) {
        pml_out[i] = host[i];
        tvar_out[i] = host[n_p + i];
    }
    return cudaSuccess;
}

}  // namespace ara
