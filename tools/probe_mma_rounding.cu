// probe_mma_rounding.cu — how does tcgen05.mma kind::f16 (fp32 accumulate)
// round?  Decides how the fp32-accurate split-operand mode must accumulate.
//
// One M=128 x N=64 x K=64 MMA chain (4 x K16 steps); every A row m is an
// independent experiment read back from TMEM lane m:
//   col 0: within one K16 step      1 + c*2^-24          (c from the row table)
//   col 1: across K16 steps         acc=1 (step 0) then += c*2^-24 (step 1)
//   col 2: 16 tiny products in one step, each c*2^-26 (sum 16*c*2^-26)
//   col 3: same as col 1 with the big term negative (-1)
// Expected fp32 results are printed next to RN / RZ predictions.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 probe_mma_rounding.cu
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2006_10004_b200/csrc/sm100.cuh"

using namespace tvs;

#define CK(x)                                                                                    \
  do {                                                                                           \
    cudaError_t e = (x);                                                                         \
    if (e != cudaSuccess) {                                                                      \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);             \
      exit(1);                                                                                   \
    }                                                                                            \
  } while (0)

// no-swizzle K-major chunk-planar operands: chunk j (8 K values) of row r at j*(rows*16) + r*16
__global__ void __launch_bounds__(128, 1) k_probe(const __half* Ag, const __half* Bg, float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;               // 128 rows x 64 K
  uint8_t* sB = smem + 128 * 128;   // 64 rows x 64 K
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int idx = tid; idx < 128 * 8; idx += 128) {
    const int row = idx / 8, j = idx % 8;
    *reinterpret_cast<uint4*>(sA + j * (128 * 16) + row * 16) = reinterpret_cast<const uint4*>(Ag)[row * 8 + j];
  }
  for (int idx = tid; idx < 64 * 8; idx += 128) {
    const int row = idx / 8, j = idx % 8;
    *reinterpret_cast<uint4*>(sB + j * (64 * 16) + row * 16) = reinterpret_cast<const uint4*>(Bg)[row * 8 + j];
  }
  fence_async_smem();
  if (warp == 0) tmem_alloc<64>(&tbase);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t idesc = make_idesc(128, 64, kFmtF16, kFmtF16);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    for (int k = 0; k < 4; ++k) {
      const uint64_t ad = make_smem_desc(a0 + k * 2 * (128 * 16), 128 * 16, 128, kLayoutNone);
      const uint64_t bd = make_smem_desc(b0 + k * 2 * (64 * 16), 64 * 16, 128, kLayoutNone);
      mma_f16_ss(tmem, ad, bd, idesc, k > 0);
    }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < 64; c += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int i = 0; i < 16; ++i) out[tid * 64 + c + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<64>(tmem);
}

int main() {
  // Part 1: plain RN/RZ probes (see header).  Part 2: offset accumulator.
  const float cs[] = {0.25f, 0.5f, 0.75f, 1.0f, 1.25f, 1.5f, 1.75f, 2.0f, 2.5f, 3.0f, 3.5f};
  const int nc = sizeof(cs) / sizeof(cs[0]);
  std::vector<__half> A(128 * 64, __float2half(0.f)), B(64 * 64, __float2half(0.f));
  const float t12 = ldexpf(1.f, -12), t11 = ldexpf(1.f, -11);
  B[0 * 64 + 0] = __float2half(1.f);
  B[0 * 64 + 1] = __float2half(t12);
  B[1 * 64 + 0] = __float2half(1.f);
  B[1 * 64 + 16] = __float2half(t12);
  B[3 * 64 + 0] = __float2half(-1.f);
  B[3 * 64 + 16] = __float2half(t12);
  for (int m = 0; m < nc; ++m) {
    A[m * 64 + 0] = __float2half(1.f);
    A[m * 64 + 1] = __float2half(cs[m] * t12);
    A[m * 64 + 16] = __float2half(cs[m] * t12);
  }
  // Part 2 (rows 64..): acc = O = 1.5 from K step 0 (A=1 x B=1.5 at k=0), then K
  // step 1 adds products A[m][16+j] * B[n][16+j] = 2^-12 * c_j 2^-11 = c_j u,
  // u = ulp(1.5) = 2^-23.  Columns n = 8.. hold the c-lists below.
  const std::vector<std::vector<float>> lists = {
      {0.75f, 0.75f},                                      // sum 1.5u : once->1  each->0
      {1.5f, -0.75f},                                      // sum 0.75u: once->0  each->1
      {0.25f, 0.25f, 0.25f, 0.25f, 0.25f, 0.25f, 0.25f, 0.25f},  // 2u: once->2 each->0
      {1.75f},                                             // 1.75u: ->1
      {-0.25f},                                            // -0.25u: once -> -1 (floor) or 0 (RZ of |.|)
      {-1.25f},                                            // -1.25u
      {0.5f, 0.5f, 0.5f, -0.25f},                          // 1.25u: once->1 each->0
  };
  for (int m = 64; m < 128; ++m) {
    A[m * 64 + 0] = __float2half(1.f);
    for (int j = 0; j < 16; ++j) A[m * 64 + 16 + j] = __float2half(t12);
  }
  for (size_t l = 0; l < lists.size(); ++l) {
    const int n = 8 + (int)l;
    B[n * 64 + 0] = __float2half(1.5f);
    for (size_t j = 0; j < lists[l].size(); ++j) B[n * 64 + 16 + j] = __float2half(lists[l][j] * t11);
  }
  __half *dA, *dB;
  float* dO;
  CK(cudaMalloc(&dA, A.size() * 2));
  CK(cudaMalloc(&dB, B.size() * 2));
  CK(cudaMalloc(&dO, 128 * 64 * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
  const int smem = 128 * 128 + 64 * 128 + 1024;
  CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_probe<<<1, 128, smem>>>(dA, dB, dO);
  CK(cudaDeviceSynchronize());
  std::vector<float> O(128 * 64);
  CK(cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost));
  auto ulps = [](float v, float base) { return (double)(v - base) / ldexp(1.0, -24); };
  printf("c      col0 within-step  col1 across-steps  col3 across(neg)   [units of 2^-24]\n");
  for (int m = 0; m < nc; ++m)
    printf("%5.2f  %8.3f           %8.3f           %8.3f\n", cs[m], ulps(O[m * 64 + 0], 1.f), ulps(O[m * 64 + 1], 1.f),
           ulps(O[m * 64 + 3], -1.f));
  printf("offset accumulator O=1.5, u=2^-23: result (acc-O)/u per product list\n");
  for (size_t l = 0; l < lists.size(); ++l) {
    double ex = 0;
    printf("  list %zu [", l);
    for (float c : lists[l]) { printf(" %.2f", c); ex += c; }
    printf(" ]  exact %.2f  got %.3f\n", ex, (double)(O[64 * 64 + 8 + l] - 1.5f) / ldexp(1.0, -23));
  }
  printf("DONE\n");
  return 0;
}
