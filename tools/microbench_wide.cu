// microbench_wide.cu -- which load pattern serves 256-byte event rows (E = 32 fp64) fastest on
// B200?  (Tuning aid for csrc/scan_pair.cu's wide rows, not product code.)
//
// A group of 4 lanes owns a trial (k random rows of 256 B = 2 lines, L2-resident, indexed by the
// trial's ids); lane c owns chunks {2c, 2c+1} (32 B each) of a row, the kernel's layout.
//   same     : both load instructions of a step read ONE row (lanes 0,1 line 0, lanes 2,3 line 1)
//   skew     : lanes 0,1 read line 0 of event d, lanes 2,3 line 1 of event d-1 (the skewed chain)
//   split    : like skew, but each pair's loads are separate instructions predicated to that pair
//   line_g4  : reference: 128-byte rows, 4 lanes x 32 B (one instruction per row)
// Each lane sums what it loads (a dependency on every load).  Prints one JSON line per pattern.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_wide tools/microbench_wide.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <random>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void ld8(const uint32_t* p, uint32_t (&v)[8]) {
  asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]) : "l"(p));
}
__device__ __forceinline__ void ldc(const double* p, double (&v)[4]) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]),"=d"(v[1]),"=d"(v[2]),"=d"(v[3]) : "l"(p));
}

// PAT 0 same, 1 skew, 2 split; RB row bytes
template <int PAT, int RB>
__global__ void __launch_bounds__(128) k_wide(const uint32_t* __restrict__ ids, const double* __restrict__ rows,
                                              double* out, int n, int k) {
  const int lane = threadIdx.x & 31, c = lane % 4, p = c >> 1;
  const int groups = gridDim.x * blockDim.x / 4;
  constexpr int RD = RB / 8;  // doubles per row
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) / 4; t < n; t += groups) {
    const uint32_t* ev = ids + (size_t)t * k;
    double acc = 0;
    uint32_t prev = 0;
    uint32_t idn[8];
    ld8(ev, idn);
    for (int d = 0; d < k; d += 8) {
      uint32_t id[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) id[j] = idn[j];
      if (d + 8 < k) ld8(ev + d + 8, idn);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        double a[4], b[4];
        if (RB == 128) {  // line_g4
          ldc(rows + (size_t)id[j] * RD + 4 * c, a);
          acc += (a[0] + a[1]) + (a[2] + a[3]);
          continue;
        }
        const uint32_t mine = (PAT == 0 || p == 0) ? id[j] : prev;  // skew: pair 1 one event behind
        const double* r = rows + (size_t)mine * RD + 8 * c;
        if (PAT == 2) {
          if (p == 0) { ldc(r, a); ldc(r + 4, b); }
          __syncwarp();
          if (p == 1) { ldc(r, a); ldc(r + 4, b); }
        } else {
          ldc(r, a); ldc(r + 4, b);
        }
        acc += ((a[0] + a[1]) + (a[2] + a[3])) + ((b[0] + b[1]) + (b[2] + b[3]));
        prev = id[j];
      }
    }
    out[(size_t)t * 4 + c] = acc;
  }
}

template <typename K>
void run(const char* name, K kern, int grid, const uint32_t* ids, const double* rows, double* out,
         int n, int k, int lines_per_row) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  for (int w = 0; w < 2; ++w) kern<<<grid, 128>>>(ids, rows, out, n, k);
  CK(cudaDeviceSynchronize());
  const int reps = 5;
  CK(cudaEventRecord(a));
  for (int r = 0; r < reps; ++r) kern<<<grid, 128>>>(ids, rows, out, n, k);
  CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b)); ms /= reps;
  const double ev = (double)n * k;
  printf("{\"pattern\": \"%s\", \"grid\": %d, \"ms\": %.4f, \"events_per_s\": %.4e, \"lines_per_s\": %.4e}\n",
         name, grid, ms, ev / (ms * 1e-3), ev * lines_per_row / (ms * 1e-3));
  fflush(stdout);
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 131072, k = argc > 2 ? atoi(argv[2]) : 1000;
  const uint32_t U = 20000;
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::mt19937_64 rng(1308);
  std::vector<double> hrows((size_t)(U + 1) * 32);
  for (auto& x : hrows) x = (double)(rng() % 1000);
  const size_t ne = (size_t)n * k;
  std::vector<uint32_t> hidx(ne);
  for (size_t i = 0; i < ne; ++i) hidx[i] = 1 + rng() % U;
  uint32_t* didx; double *drows, *dout;
  CK(cudaMalloc(&didx, ne * 4)); CK(cudaMalloc(&drows, hrows.size() * 8));
  CK(cudaMalloc(&dout, (size_t)n * 4 * 8));
  CK(cudaMemcpy(didx, hidx.data(), ne * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(drows, hrows.data(), hrows.size() * 8, cudaMemcpyHostToDevice));
  printf("{\"sms\": %d, \"n\": %d, \"k\": %d}\n", sms, n, k);
  for (int bps : {3, 4, 8}) {
    const int grid = sms * bps;
    run("same", k_wide<0, 256>, grid, didx, drows, dout, n, k, 2);
    run("skew", k_wide<1, 256>, grid, didx, drows, dout, n, k, 2);
    run("split", k_wide<2, 256>, grid, didx, drows, dout, n, k, 2);
    run("line_g4", k_wide<0, 128>, grid, didx, drows, dout, n, k, 1);
  }
  return 0;
}
