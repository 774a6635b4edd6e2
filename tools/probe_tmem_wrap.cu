// probe_tmem_wrap.cu — does a tcgen05.mma whose N columns run past TMEM column
// 511 wrap around to column 0?  (If yes, the conv's dy-stacked N=192 windows
// never need splitting at the accumulator ring's end.)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 probe_tmem_wrap.cu
#include <cuda_fp16.h>
#include <cstdio>
#include "../paper_2006_10004_b200/csrc/sm100.cuh"
using namespace tvs;

__global__ void __launch_bounds__(128, 1) k_wrap(float* out, int col0, int n, int* err) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;              // 128 rows x 128 B
  uint8_t* sB = smem + 128 * 128;  // 256 rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 128 * 64; i += 128) reinterpret_cast<__half*>(sA)[i] = __float2half(1.0f);
  for (int i = tid; i < 256 * 64; i += 128) reinterpret_cast<__half*>(sB)[i] = __float2half((float)(i / 64 + 1));
  fence_async_smem();
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  // zero all 512 columns (each warp its 32 lanes)
  for (int c = 0; c < 512; c += 16) tmem_st16_zero(tmem + ((uint32_t)(warp * 32) << 16) + c);
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = make_idesc(128, n, kFmtF16, kFmtF16);
    const uint64_t ad = make_smem_desc(smem_u32(sA), 0, 1024, kLayoutSW128);
    const uint64_t bd = make_smem_desc(smem_u32(sB), 0, 1024, kLayoutSW128);
    mma_f16_ss(tmem + col0, ad, bd, idesc, 0u);  // K = 16: D[m][j] = 16 * (j + 1)
    mma_commit(&bar);
  }
  __syncwarp();
  if (!mbar_wait_bounded(&bar, 0, 1ull << 24)) { if (lane_id() == 0) atomicAdd(err, 1); }
  tc_fence_after();
  for (int c = 0; c < 512; c += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int i = 0; i < 16; ++i) out[tid * 512 + c + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  float* d; int* e;
  cudaMalloc(&d, 128 * 512 * 4);
  cudaMallocManaged(&e, 4);
  cudaFuncSetAttribute(k_wrap, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int cases[][2] = {{256, 192}, {448, 128}, {384, 192}, {480, 64}};
  for (auto& cs : cases) {
    *e = 0;
    k_wrap<<<1, 128, 100 * 1024>>>(d, cs[0], cs[1], e);
    cudaError_t r = cudaDeviceSynchronize();
    if (r != cudaSuccess) { printf("col0=%d N=%d: CUDA error %s\n", cs[0], cs[1], cudaGetErrorString(r)); return 1; }
    static float h[128 * 512];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    int wrote_hi = 0, wrote_lo = 0, first_lo = -1;
    for (int c = 0; c < 512; ++c) {
      if (h[5 * 512 + c] != 0.0f) { if (c >= cs[0]) ++wrote_hi; else { ++wrote_lo; if (first_lo < 0) first_lo = c; } }
    }
    printf("col0=%d N=%d: timeout=%d, nonzero cols >= col0: %d, below col0: %d (first %d, value %.0f; col0 value %.0f)\n",
           cs[0], cs[1], *e, wrote_hi, wrote_lo, first_lo, first_lo >= 0 ? h[5 * 512 + first_lo] : 0.f, h[5 * 512 + cs[0]]);
  }
  return 0;
}
