// microbench_rowpattern.cu -- which intra-warp layout of the 128-byte row gathers does the L1
// data pipe serve fastest on B200?  (Tuning aid for csrc/scan.cu, not product code.)
//
// Trial-per-group like the scan: a group of G lanes owns one trial (k contiguous ids, read as
// 32-byte vectors); per event the group gathers the event's 128-byte row (rows indexed directly by
// the id, U rows, L2-resident) with 256-bit loads and each lane sums its doubles.
//   split  : G = 2, lane c loads bytes [64c, 64c+32) then [64c+32, 64c+64)   (scan.cu today)
//   adj    : G = 2, lane c loads bytes [32c, 32c+32) then [64+32c, 64+32c+32) (each instruction of
//            a group covers one contiguous 64-byte half line)
//   g4     : G = 4, lane c loads bytes [32c, 32c+32) (one instruction per row)
//   *_noalloc: the same with L1::no_allocate row loads
// Prints one JSON line per kernel.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void ld8(const uint32_t* p, uint32_t (&v)[8]) {
  asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]) : "l"(p));
}
__device__ __forceinline__ void ldrow4(const double* p, double (&v)[4]) {
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]),"=d"(v[1]),"=d"(v[2]),"=d"(v[3]) : "l"(p));
}

__device__ __forceinline__ void ldrow4_na(const double* p, double (&v)[4]) {
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]),"=d"(v[1]),"=d"(v[2]),"=d"(v[3]) : "l"(p));
}

// PAT 0 split, 1 adj (G = 2, two loads per lane); PAT 2 g4 (one load per lane);
// PAT 3 split and PAT 4 g4 with L1::no_allocate row loads
template <int G, int PAT>
__global__ void __launch_bounds__(128) k_rows(const uint32_t* __restrict__ ids,
                                              const double* __restrict__ rows, double* out, int n, int k) {
  const int lane = threadIdx.x & 31, c = lane % G;
  const int groups = gridDim.x * blockDim.x / G;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) / G; t < n; t += groups) {
    const uint32_t* ev = ids + (size_t)t * k;
    double acc = 0;
    uint32_t idn[8];
    ld8(ev, idn);
    for (int d = 0; d < k; d += 8) {
      uint32_t id[8];
      #pragma unroll
      for (int j = 0; j < 8; ++j) id[j] = idn[j];
      if (d + 8 < k) ld8(ev + d + 8, idn);
      #pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double* p = rows + (size_t)id[j] * 16;
        double a[4], b[4];
        if (PAT == 0) { ldrow4(p + 8 * c, a); ldrow4(p + 8 * c + 4, b); }
        else if (PAT == 1) { ldrow4(p + 4 * c, a); ldrow4(p + 8 + 4 * c, b); }
        else if (PAT == 2) { ldrow4(p + 4 * c, a); b[0] = b[1] = b[2] = b[3] = 0; }
        else if (PAT == 3) { ldrow4_na(p + 8 * c, a); ldrow4_na(p + 8 * c + 4, b); }
        else { ldrow4_na(p + 4 * c, a); b[0] = b[1] = b[2] = b[3] = 0; }
        acc += ((a[0] + a[1]) + (a[2] + a[3])) + ((b[0] + b[1]) + (b[2] + b[3]));
      }
    }
    out[(size_t)t * G + c] = acc;
  }
}

template <typename K>
void run(const char* name, K kern, int grid, int threads, const uint32_t* ids, const double* rows,
         double* out, int n, int k) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  for (int w = 0; w < 2; ++w) kern<<<grid, threads>>>(ids, rows, out, n, k);
  CK(cudaDeviceSynchronize());
  const int reps = 5;
  CK(cudaEventRecord(a));
  for (int r = 0; r < reps; ++r) kern<<<grid, threads>>>(ids, rows, out, n, k);
  CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b)); ms /= reps;
  double ev = (double)n * k;
  printf("{\"kernel\": \"%s\", \"grid\": %d, \"ms\": %.4f, \"events_per_s\": %.4e}\n", name, grid, ms,
         ev / (ms * 1e-3));
  fflush(stdout);
}

int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 262144;
  int k = argc > 2 ? atoi(argv[2]) : 1000;
  uint32_t U = 20000;
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::mt19937_64 rng(1308);
  std::vector<double> hrows((size_t)(U + 1) * 16);
  for (auto& x : hrows) x = (double)(rng() % 1000);
  size_t ne = (size_t)n * k;
  std::vector<uint32_t> hidx(ne);
  for (size_t i = 0; i < ne; ++i) hidx[i] = 1 + rng() % U;
  uint32_t* didx; double *drows, *dout;
  CK(cudaMalloc(&didx, ne * 4)); CK(cudaMalloc(&drows, hrows.size() * 8));
  CK(cudaMalloc(&dout, (size_t)n * 4 * 8));
  CK(cudaMemcpy(didx, hidx.data(), ne * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(drows, hrows.data(), hrows.size() * 8, cudaMemcpyHostToDevice));
  printf("{\"sms\": %d, \"n\": %d, \"k\": %d}\n", sms, n, k);
  for (int bps : {3, 4, 6, 8}) {
    int grid = sms * bps;
    run("split_g2", k_rows<2, 0>, grid, 128, didx, drows, dout, n, k);
    run("adj_g2", k_rows<2, 1>, grid, 128, didx, drows, dout, n, k);
    run("g4", k_rows<4, 2>, grid, 128, didx, drows, dout, n, k);
    run("split_g2_noalloc", k_rows<2, 3>, grid, 128, didx, drows, dout, n, k);
    run("g4_noalloc", k_rows<4, 4>, grid, 128, didx, drows, dout, n, k);
  }
  return 0;
}
