// microbench_gather4.cu -- can Blackwell's TMA gather4 (cp.async.bulk.tensor.2d ... tile::gather4:
// four rows with arbitrary row coordinates per instruction, into shared memory) deliver the
// scan's 128-byte rows faster than coalesced 256-bit LDG gathers?  (Tuning aid, not product code.)
//
// Rows: [U+1][16] doubles (128 B, L2-resident, U = 20,000), random ids as in the headline YET.
// Each warp streams one "trial" of k events at a time: lane 0 issues one gather4 per 4 events
// into a ring of S slots (512 B each, one mbarrier per slot, expect_tx 512 B), every lane waits
// for the slot, reads the 4 rows with one 128-bit LDS each (1 wavefront per row) and accumulates.
// Prints one JSON line per (S, blocks per SM): rows/s, to compare with microbench_rowpattern.cu
// (LDG: 1.13e11 rows/s at 12 warps/SM with 2 lanes per row, 1.69e11 with 4 lanes per row).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather4 microbench_gather4.cu
// (cuTensorMapEncodeTiled through cudaGetDriverEntryPoint: no -lcuda)
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int S>
__global__ void __launch_bounds__(128) k_g4(const __grid_constant__ CUtensorMap tm, const uint32_t* __restrict__ ids,
                                            int n_trials, int k, double* out) {
  __shared__ __align__(128) double slots[4][S][64];  // per warp: S slots of 4 rows x 16 doubles
  __shared__ __align__(8) uint64_t bar[4][S];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
    for (int i = 0; i < S; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar[w][i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  uint32_t phase = 0;  // bit i: parity of slot i
  double acc = 0;
  const int warps = gridDim.x * 4;
  for (int t = blockIdx.x * 4 + w; t < n_trials; t += warps) {
    const uint32_t* ev = ids + (size_t)t * k;
    const int nq = k / 4;  // gathers of 4 rows
    auto issue = [&](int q) {
      if (lane == 0) {
        const int s = q % S;
        const uint32_t b = sa(&bar[w][s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 512;" :: "r"(b) : "memory");
        const uint4 r = *reinterpret_cast<const uint4*>(ev + 4 * q);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
            :: "r"(sa(&slots[w][s][0])), "l"(&tm), "r"(b), "r"(0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w)
            : "memory");
      }
    };
    for (int q = 0; q < S - 1 && q < nq; ++q) issue(q);
    for (int q = 0; q < nq; ++q) {
      if (q + S - 1 < nq) issue(q + S - 1);
      const int s = q % S;
      const uint32_t b = sa(&bar[w][s]);
      const uint32_t par = (phase >> s) & 1u;
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(b), "r"(par) : "memory");
      phase ^= 1u << s;
      const double2 v = reinterpret_cast<const double2*>(&slots[w][s][0])[lane];
      acc += v.x + v.y;
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int S>
void run(const CUtensorMap& tm, int bps, int sms, const uint32_t* ids, int n, int k, double* out) {
  const int grid = sms * bps;
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  for (int i = 0; i < 2; ++i) k_g4<S><<<grid, 128>>>(tm, ids, n, k, out);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  const int reps = 5;
  for (int i = 0; i < reps; ++i) k_g4<S><<<grid, 128>>>(tm, ids, n, k, out);
  CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b)); ms /= reps;
  printf("{\"kernel\": \"tma_gather4\", \"slots\": %d, \"blocks_per_sm\": %d, \"warps_per_sm\": %d, \"ms\": %.4f, \"rows_per_s\": %.4e}\n",
         S, bps, 4 * bps, ms, (double)n * k / (ms * 1e-3));
  fflush(stdout);
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 262144, k = argc > 2 ? atoi(argv[2]) : 1000;
  const uint32_t U = 20000;
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::mt19937_64 rng(1308);
  std::vector<double> hrows((size_t)(U + 1) * 16);
  for (auto& x : hrows) x = (double)(rng() % 1000);
  std::vector<uint32_t> hid((size_t)n * k);
  for (auto& x : hid) x = 1 + rng() % U;
  uint32_t* did; double *drows, *dout;
  CK(cudaMalloc(&did, hid.size() * 4)); CK(cudaMalloc(&drows, hrows.size() * 8));
  CK(cudaMalloc(&dout, (size_t)sms * 32 * 128 * 8));
  CK(cudaMemcpy(did, hid.data(), hid.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(drows, hrows.data(), hrows.size() * 8, cudaMemcpyHostToDevice));
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  CUtensorMap tm;
  const cuuint64_t dims[2] = {16, U + 1}, strides[1] = {128};
  const cuuint32_t box[2] = {16, 1}, es[2] = {1, 1};
  CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, drows, dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("{\"error\": \"cuTensorMapEncodeTiled %d\"}\n", (int)r); return 1; }
  printf("{\"sms\": %d, \"n\": %d, \"k\": %d}\n", sms, n, k);
  for (int bps : {3, 4, 8}) {
    run<4>(tm, bps, sms, did, n, k, dout);
    run<8>(tm, bps, sms, did, n, k, dout);
  }
  return 0;
}
