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

template <typename K>
void run(const char* name, K kern, int grid, const uint32_t* ids, const uint32_t* map, const double* rows,
         double* out, int n, int k, bool map_used, bool row_used) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  for (int w = 0; w < 2; ++w) kern<<<grid, 256>>>(ids, map, rows, out, n, k);
  CK(cudaDeviceSynchronize());
  const int reps = 5;
  CK(cudaEventRecord(a));
  for (int r = 0; r < reps; ++r) kern<<<grid, 256>>>(ids, map, rows, out, n, k);
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
