// microbench_gather.cu -- B200 ceilings for the YET-scan memory pattern (not product code).
//
// Measures, for random event rows drawn from a pool of U rows of W doubles (event-major store,
// L2-resident) and a u32 catalogue map (C entries), the throughput of:
//   ids      : stream the per-trial id arrays only (HBM streaming floor)
//   map      : ids -> map lookup (one random 4 B read per event)
//   lane_row : ids -> map -> row; each lane gathers its own row with W/4 256-bit loads
//   coop_row : ids -> map -> row; 4 lanes gather one row together (coalesced 128 B), the
//              group's 4 trials' rows are loaded in 4 instructions (idx broadcast by shfl)
//   lane_row_nomap / coop_row_nomap : same, the id stream already holds row indices
// Trial-major layout as in the product: lane t owns trial t's k contiguous ids.
// Prints one JSON line per kernel.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

constexpr int W = 16;

__device__ __forceinline__ void ld8(const uint32_t* p, uint32_t (&v)[8]) {
  asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]) : "l"(p));
}
__device__ __forceinline__ void ldrow4(const double* p, double (&v)[4]) {
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]),"=d"(v[1]),"=d"(v[2]),"=d"(v[3]) : "l"(p));
}
__device__ __forceinline__ uint32_t ldmap(const uint32_t* p) {
  uint32_t v; asm("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p)); return v;
}

template <int MODE>  // 0 ids, 1 map, 2 lane_row, 3 lane_row_nomap
__global__ void __launch_bounds__(256) k_lane(const uint32_t* __restrict__ ids, const uint32_t* __restrict__ map,
                       const double* __restrict__ rows, double* out, int n, int k) {
  int stride = gridDim.x * blockDim.x;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += stride) {
    const uint32_t* ev = ids + (size_t)t * k;
    double acc = 0; uint32_t iacc = 0;
    for (int d = 0; d < k; d += 8) {
      uint32_t id[8]; ld8(ev + d, id);
      #pragma unroll 1
      for (int h = 0; h < 8; h += 2) {
        if (MODE == 0) { iacc += id[h] ^ id[h + 1]; continue; }
        uint32_t i0 = id[0], i1 = id[1];
        if (MODE == 1 || MODE == 2) { i0 = ldmap(map + i0); i1 = ldmap(map + i1); }
        if (MODE == 1) { iacc += i0 + i1; }
        else {
          double a[W / 4][4], b[W / 4][4];
          #pragma unroll
          for (int c = 0; c < W / 4; ++c) { ldrow4(rows + (size_t)i0 * W + 4 * c, a[c]); ldrow4(rows + (size_t)i1 * W + 4 * c, b[c]); }
          #pragma unroll
          for (int c = 0; c < W / 4; ++c)
            #pragma unroll
            for (int q = 0; q < 4; ++q) acc += a[c][q] + b[c][q];
        }
        #pragma unroll
        for (int i = 0; i < 6; ++i) id[i] = id[i + 2];
      }
    }
    out[t] = acc + iacc;
  }
}

template <int MODE>  // 4 coop_row, 5 coop_row_nomap
__global__ void __launch_bounds__(256) k_coop(const uint32_t* __restrict__ ids, const uint32_t* __restrict__ map,
                       const double* __restrict__ rows, double* out, int n, int k) {
  int lane = threadIdx.x & 31, c = lane & 3, g0 = lane & ~3;
  int stride = gridDim.x * blockDim.x;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += stride) {  // n multiple of 32
    const uint32_t* ev = ids + (size_t)t * k;
    double acc = 0;
    for (int d = 0; d < k; d += 8) {
      uint32_t id[8]; ld8(ev + d, id);
      #pragma unroll 1
      for (int h = 0; h < 8; ++h) {
        uint32_t my = id[0];
        if (MODE == 4) my = ldmap(map + my);
        double v[4][4];
        #pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t iq = __shfl_sync(0xffffffffu, my, g0 + q);
          ldrow4(rows + (size_t)iq * W + 4 * c, v[q]);
        }
        #pragma unroll
        for (int q = 0; q < 4; ++q)
          #pragma unroll
          for (int j = 0; j < 4; ++j) acc += v[q][j];
        #pragma unroll
        for (int i = 0; i < 7; ++i) id[i] = id[i + 1];
      }
    }
    out[t] = acc;
  }
}


// TMA variant: each group of 2 lanes keeps a ring of D row slots in shared memory; lane 0 issues a
// 128-byte cp.async.bulk per event D-1 events ahead (mbarrier completion), both lanes wait and read
// their 64 bytes with LDS.  Map lookups stay LDG.  (MODE 6: with map, 7: ids are row indices)
__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(m)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(m)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
               :: "r"((uint32_t)__cvta_generic_to_shared(m)), "r"(parity) : "memory");
}

template <int MODE, int D>   // D = ring slots per group (8): batches of 4 events issued one batch ahead
__global__ void __launch_bounds__(128) k_tma(const uint32_t* __restrict__ ids, const uint32_t* __restrict__ map,
                       const double* __restrict__ rows, double* out, int n, int k) {
  extern __shared__ __align__(128) unsigned char smem[];
  double (*ring)[D][W] = reinterpret_cast<double (*)[D][W]>(smem);                 // [64][D][W]
  uint64_t (*bar)[D] = reinterpret_cast<uint64_t (*)[D]>(smem + 64 * D * W * 8);  // [64][D]
  const int lane = threadIdx.x & 31, c = lane & 1, gb = threadIdx.x >> 1;
  const unsigned gmask = 3u << (lane - c);
  if (c == 0) for (int s = 0; s < D; ++s) mbar_init(&bar[gb][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  uint32_t phase = 0;   // bit s = parity of slot s
  int stride = gridDim.x * 64;
  for (int t = blockIdx.x * 64 + gb; t < n; t += stride) {
    const uint32_t* ev = ids + (size_t)t * k;
    double acc = 0;
    auto issue4 = [&](int d) {   // events d..d+3 (d multiple of 4)
      if (c == 0 && d < k) {
        uint4 q = *reinterpret_cast<const uint4*>(ev + d);
        uint32_t id4[4] = {q.x, q.y, q.z, q.w};
        #pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint32_t idx = MODE == 6 ? ldmap(map + id4[j]) : id4[j];
          const int s = (d + j) % D;
          mbar_expect_tx(&bar[gb][s], 128);
          bulk_g2s(&ring[gb][s][0], rows + (size_t)idx * W, 128, &bar[gb][s]);
        }
      }
    };
    issue4(0);
    for (int d = 0; d < k; d += 4) {
      issue4(d + 4);
      #pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int s = (d + j) % D;
        mbar_wait(&bar[gb][s], (phase >> s) & 1);
        phase ^= 1u << s;
        const double4* p = reinterpret_cast<const double4*>(&ring[gb][s][8 * c]);
        double4 a = p[0], b = p[1];
        acc += a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w;
      }
      __syncwarp(gmask);   // slots of this batch are reissued next iteration
    }
    out[(size_t)t * 2 + c] = acc;
  }
}

template <typename K>
void run(const char* name, K kern, int grid, const uint32_t* ids, const uint32_t* map, const double* rows,
         double* out, int n, int k, bool map_used, bool row_used, int threads = 256, int smem = 0) {
  if (smem) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  for (int w = 0; w < 2; ++w) kern<<<grid, threads, smem>>>(ids, map, rows, out, n, k);
  CK(cudaDeviceSynchronize());
  const int reps = 5;
  CK(cudaEventRecord(a));
  for (int r = 0; r < reps; ++r) kern<<<grid, threads, smem>>>(ids, map, rows, out, n, k);
  CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b)); ms /= reps;
  double ev = (double)n * k;
  double alg = ev * (4.0 + 8.0 * W);
  double l2 = ev * ((map_used ? 32.0 : 0) + (row_used ? 8.0 * W : 0));
  printf("{\"kernel\": \"%s\", \"grid\": %d, \"ms\": %.4f, \"events_per_s\": %.4e, \"alg_GBps\": %.1f, \"l2_gather_GBps\": %.1f}\n",
         name, grid, ms, ev / (ms * 1e-3), alg / (ms * 1e-3) / 1e9, l2 / (ms * 1e-3) / 1e9);
  fflush(stdout);
}

int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 262144;   // trials
  int k = argc > 2 ? atoi(argv[2]) : 1000;     // events per trial
  uint32_t C = 2000000, U = 20000;
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::mt19937_64 rng(1308);
  std::vector<uint32_t> pool(U), hmap(C + 1, 0);
  for (uint32_t u = 0; u < U; ++u) { uint32_t e; do { e = 1 + rng() % C; } while (hmap[e]); hmap[e] = u + 1; pool[u] = e; }
  std::vector<double> hrows((size_t)(U + 1) * W);
  for (auto& x : hrows) x = (double)(rng() % 1000);
  size_t ne = (size_t)n * k;
  std::vector<uint32_t> hids(ne), hidx(ne);
  for (size_t i = 0; i < ne; ++i) { uint32_t u = rng() % U; hids[i] = pool[u]; hidx[i] = u + 1; }
  uint32_t *dids, *didx, *dmap; double *drows, *dout;
  CK(cudaMalloc(&dids, ne * 4)); CK(cudaMalloc(&didx, ne * 4)); CK(cudaMalloc(&dmap, (C + 1) * 4));
  CK(cudaMalloc(&drows, hrows.size() * 8)); CK(cudaMalloc(&dout, (size_t)n * 8));
  CK(cudaMemcpy(dids, hids.data(), ne * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(didx, hidx.data(), ne * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dmap, hmap.data(), (C + 1) * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(drows, hrows.data(), hrows.size() * 8, cudaMemcpyHostToDevice));
  printf("{\"sms\": %d, \"n\": %d, \"k\": %d, \"W\": %d}\n", sms, n, k, W);
  CK(cudaMalloc(&dout, (size_t)n * 16));
  for (int occ : {2, 3}) {
    int grid = sms * occ;
    run("tma_D8", k_tma<6, 8>, grid, dids, dmap, drows, dout, n, k, true, true, 128, 64 * 8 * (W * 8 + 8));
    run("tma_D8_nomap", k_tma<7, 8>, grid, didx, dmap, drows, dout, n, k, false, true, 128, 64 * 8 * (W * 8 + 8));
  }
  for (int occ : {4, 8}) {
    int grid = sms * occ;
    run("ids", k_lane<0>, grid, dids, dmap, drows, dout, n, k, false, false);
    run("map", k_lane<1>, grid, dids, dmap, drows, dout, n, k, true, false);
    run("lane_row", k_lane<2>, grid, dids, dmap, drows, dout, n, k, true, true);
    run("lane_row_nomap", k_lane<3>, grid, didx, dmap, drows, dout, n, k, false, true);
    run("coop_row", k_coop<4>, grid, dids, dmap, drows, dout, n, k, true, true);
    run("coop_row_nomap", k_coop<5>, grid, didx, dmap, drows, dout, n, k, false, true);
  }
  return 0;
}
