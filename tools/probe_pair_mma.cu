// probe_pair_mma.cu — groundwork for a CTA-pair (cta_group::2) hidden conv.
//
// (1) Semantics: one kind::f16 MMA with M = 256 over a 2-CTA cluster, N = 192,
//     K = 16.  A[m][k] = 1 if k == m % 16 (so D[m][n] = B[n][m % 16]) and
//     B[n][k] = 1000 * cta + n + k / 16 in each CTA's own shared memory at the
//     same offset.  Reading D back in both CTAs shows which CTA's A rows and B
//     rows fed which D lanes and columns.
// (2) Rate: back-to-back cta_group::2 M=256 N=192 MMAs issued by the leader
//     CTA (cycles per MMA; per SM the same MAC rate as a cta_group::1 M=128
//     N=192 MMA at 96 cycles would be full rate), with each CTA reading only
//     its half of B.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 probe_pair_mma.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2006_10004_b200/csrc/sm100.cuh"

using namespace tvs;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void cluster_arrive_wait() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma_pair(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
      ::"r"(smem_u32(bar)), "h"((uint16_t)0x3) : "memory");
}

constexpr int kN = 192;
// smem: A 16 KB (128 rows x 128 B, SW128), B half 12 KB (96 rows x 128 B)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
k_pair(int iters, float* dout, long long* cycles, int* err) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + 16384;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  const uint32_t cta = cluster_ctarank();
  // A: row m, fp16 k: 1 if k == m % 16 ; B: 96 rows of this CTA's half
  for (int idx = tid; idx < 128 * 64; idx += 128) {
    const int m = idx / 64, k = idx % 64;
    const __half v = __float2half((k == (m % 16)) ? 1.0f : 0.0f);
    *reinterpret_cast<__half*>(sA + m * 128 + (((k >> 3) ^ (m & 7)) << 4) + (k & 7) * 2) = v;
  }
  for (int idx = tid; idx < (kN / 2) * 64; idx += 128) {
    const int n = idx / 64, k = idx % 64;
    const __half v = __float2half((float)(1000 * (int)cta + n + (k < 16 ? k / 16 : 0)));
    *reinterpret_cast<__half*>(sB + n * 128 + (((k >> 3) ^ (n & 7)) << 4) + (k & 7) * 2) = v;
  }
  fence_async_smem();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tbase))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  cluster_arrive_wait();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t idesc = make_idesc(256, kN, kFmtF16, kFmtF16);
  const uint64_t ad0 = make_smem_desc(smem_u32(sA), 0, 1024, kLayoutSW128);
  const uint64_t bd0 = make_smem_desc(smem_u32(sB), 0, 1024, kLayoutSW128);
  long long t0 = clock64();
  if (cta == 0 && tid == 0) {
    if (iters == 0) {
      mma_pair(tmem, ad0, bd0, idesc, 0u);  // one K=16 step: the semantics probe
    } else {
      for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma_pair(tmem, ad0 + ((k * 32) >> 4), bd0 + ((k * 32) >> 4), idesc, (it | k) ? 1u : 0u);
    }
    commit_pair(&bar);
  }
  __syncwarp();
  const bool ok = mbar_wait_bounded(&bar, 0, 1ull << 26);
  long long t1 = clock64();
  if (!ok && tid == 0) atomicAdd(err, 1);
  tc_fence_after();
  if (tid == 0) cycles[blockIdx.x] = t1 - t0;
  if (iters == 0 && ok) {  // D: lane = tid (this CTA's 128 rows), kN columns
    for (int c = 0; c < kN; c += 16) {
      uint32_t r[16];
      tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
      tmem_ld_wait();
      for (int j = 0; j < 16; ++j)
        dout[((size_t)blockIdx.x * 128 + tid) * kN + c + j] = __uint_as_float(r[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_arrive_wait();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}

int main() {
  const int smem = 16384 + 12288 + 1024;
  CK(cudaFuncSetAttribute(k_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  float* dD; long long* dC; int* dErr;
  CK(cudaMalloc(&dD, 2 * 128 * kN * 4)); CK(cudaMalloc(&dC, 148 * 8)); CK(cudaMalloc(&dErr, 4));
  CK(cudaMemset(dErr, 0, 4));
  // (1) semantics
  k_pair<<<2, 128, smem>>>(0, dD, dC, dErr);
  CK(cudaDeviceSynchronize());
  int herr; CK(cudaMemcpy(&herr, dErr, 4, cudaMemcpyDeviceToHost));
  std::vector<float> D(2 * 128 * kN);
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  printf("SEMANTICS timeout=%d\n", herr);
  for (int cta = 0; cta < 2; ++cta)
    for (int m : {0, 5, 127})
      printf("  CTA%d lane %3d: D[n=0]=%6.0f D[n=95]=%6.0f D[n=96]=%6.0f D[n=191]=%6.0f\n", cta, m,
             D[(cta * 128 + m) * kN + 0], D[(cta * 128 + m) * kN + 95], D[(cta * 128 + m) * kN + 96],
             D[(cta * 128 + m) * kN + 191]);
  // (2) rate over all SMs
  const int iters = 4096;
  for (int ctas : {2, 148}) {
    CK(cudaMemset(dErr, 0, 4));
    k_pair<<<ctas, 128, smem>>>(64, dD, dC, dErr);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_pair<<<ctas, 128, smem>>>(iters, dD, dC, dErr);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> c(ctas);
    CK(cudaMemcpy(c.data(), dC, ctas * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&herr, dErr, 4, cudaMemcpyDeviceToHost));
    double avg = 0; for (int i = 0; i < ctas; i += 2) avg += c[i]; avg /= (ctas / 2);
    const double macs = 256.0 * kN * 64 * iters * (ctas / 2);
    printf("RATE pair M256 N%d: ctas=%3d cyc/mma=%7.2f (per-SM full rate = 96)  %.1f TFLOP/s  timeout=%d\n", kN, ctas,
           avg / (iters * 4.0), 2.0 * macs / (ms * 1e-3) / 1e12, herr);
  }
  return 0;
}
