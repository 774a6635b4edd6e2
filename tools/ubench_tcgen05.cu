// ubench_tcgen05.cu — bring-up probes for the TVSpecNET conv kernels on B200.
//
//  (1) Descriptor/layout correctness of tcgen05.mma kind::f16 with the A
//      operand at an arbitrary pixel-row offset (the 3x3 tap shift):
//        a) SWIZZLE_128B K-major, start = base + s*128 B, base_offset 0 or s&7
//        b) no-swizzle K-major "chunk-planar" layout, start = base + s*16 B
//  (2) Issue-rate of back-to-back SS MMAs (cycles per MMA) for the shapes
//      the conv can use: M=128 x N in {64,128,192,256}, tf32, e4m3, and
//      collector::a reuse.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I.. ubench_tcgen05.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_2006_10004_b200/csrc/sm100.cuh"

using namespace tvs;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int kRowsA = 144;  // smem rows available for A (shift up to 16)

// ---------------------------------------------------------------- (1) ----
// layout 0: SW128, base_offset 0 ; layout 1: SW128, base_offset = s & 7 ;
// layout 2: no-swizzle chunk-planar.
__global__ void __launch_bounds__(128, 1)
k_layout(const __half* __restrict__ Ag, const __half* __restrict__ Bg, float* __restrict__ out,
         int layout, int s, int* err) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                       // kRowsA*128 B
  uint8_t* sB = smem + kRowsA * 128;        // 64*128 B  (kRowsA*128 = 18432 = 18*1024, aligned)
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;

  // fill A and B; each pixel row = 64 fp16 = 8 chunks of 16 B
  for (int idx = tid; idx < kRowsA * 8; idx += 128) {
    int row = idx / 8, j = idx % 8;
    uint4 v = reinterpret_cast<const uint4*>(Ag)[row * 8 + j];
    uint32_t off = (layout < 2) ? (row * 128 + ((j ^ (row & 7)) * 16)) : (j * (kRowsA * 16) + row * 16);
    *reinterpret_cast<uint4*>(sA + off) = v;
  }
  for (int idx = tid; idx < 64 * 8; idx += 128) {
    int row = idx / 8, j = idx % 8;
    uint4 v = reinterpret_cast<const uint4*>(Bg)[row * 8 + j];
    uint32_t off = (layout < 2) ? (row * 128 + ((j ^ (row & 7)) * 16)) : (j * (64 * 16) + row * 16);
    *reinterpret_cast<uint4*>(sB + off) = v;
  }
  fence_async_smem();
  if (warp == 0) tmem_alloc<64>(&tbase);
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;

  if (tid == 0) {
    const uint32_t idesc = make_idesc(128, 64, kFmtF16, kFmtF16);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    for (int k = 0; k < 4; ++k) {  // K = 64 in 4 steps of 16
      uint64_t ad, bd;
      if (layout < 2) {
        uint32_t bo = (layout == 1) ? (uint32_t)(s & 7) : 0u;
        ad = make_smem_desc(a0 + s * 128 + k * 32, 0, 1024, kLayoutSW128, bo);
        bd = make_smem_desc(b0 + k * 32, 0, 1024, kLayoutSW128, 0);
      } else {
        ad = make_smem_desc(a0 + s * 16 + k * 2 * (kRowsA * 16), kRowsA * 16, 128, kLayoutNone);
        bd = make_smem_desc(b0 + k * 2 * (64 * 16), 64 * 16, 128, kLayoutNone);
      }
      mma_f16_ss(tmem, ad, bd, idesc, k > 0);
    }
    mma_commit(&bar);
  }
  __syncwarp();
  if (!mbar_wait_bounded(&bar, 0, 1ull << 24)) { if (lane_id() == 0) atomicAdd(err, 1); }
  tc_fence_after();
  // thread t reads lane t (warp w -> lanes 32w..32w+31)
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

// ---------------------------------------------------------------- (2) ----
// variant: 0..3 f16 N=64/128/192/256 ; 4 tf32 N=64 ; 5 e4m3 N=64 ;
//          6 f16 N=64 with 3 taps sharing A via collector::a ;  7 f16 N=64
//          with A address shifted by +16 B per MMA (tap walk, no-swizzle).
// 16 / 17 / 18: the N=192 conv pattern (as 8) while warp 1 streams TMA bulk
// traffic through shared memory: 16 = global->smem loads, 17 = smem->global
// stores, 18 = both, plus warps 2-3 flooding st.shared (the epilogue staging)
__device__ __forceinline__ void bulk_store_g(void* gdst, uint32_t ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(ssrc), "r"(bytes)
               : "memory");
}
// 19: as 18 but the stores are TMA TENSOR stores (4D map, 32-px x 64-ch SW128
// boxes from an swizzled staging tile, as the conv epilogue issues them), and
// warps 2-3 also write the staging tiles with st.shared
template <int V>
__global__ void __launch_bounds__(128, 1)
k_rate(int iters, long long* cycles, int* err, uint8_t* gbuf, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < (112 * 1024) / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_async_smem();
  if (warp == 0) tmem_alloc<256>(&tbase);
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    constexpr int N = (V <= 3) ? 64 * (V + 1) : 64;
    const uint32_t fmt = (V == 4) ? kFmtTF32 : kFmtF16;
    const uint32_t idesc = make_idesc(128, N, fmt, fmt);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 32768);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint64_t ad = make_smem_desc(a0 + k * 32, 0, 1024, kLayoutSW128);
        uint64_t bd = make_smem_desc(b0 + k * 32, 0, 1024, kLayoutSW128);
        if constexpr (V <= 3) {
          mma_f16_ss(tmem, ad, bd, idesc, 1);
        } else if constexpr (V == 4) {
          mma_tf32_ss(tmem, ad, bd, idesc, 1);
        } else if constexpr (V == 5) {
          mma_f8_ss(tmem, ad, bd, make_idesc(128, 64, kFmtE4M3, kFmtE4M3), 1);
        } else if constexpr (V == 30) {  // the wide quarter kernels' shape: N=96 (32 co x 3 dy)
          mma_f16_ss(tmem, ad, bd, make_idesc(128, 96, kFmtF16, kFmtF16), 1);
        } else if constexpr (V == 31) {  // N=96 with e4m3 operands (the fp8 lo-product candidate)
          mma_f8_ss(tmem, ad, bd, make_idesc(128, 96, kFmtE4M3, kFmtE4M3), 1);
        } else if constexpr (V == 32) {
          mma_f8_ss(tmem, ad, bd, make_idesc(128, 192, kFmtE4M3, kFmtE4M3), 1);
        } else if constexpr (V == 6) {
          uint64_t bd1 = make_smem_desc(b0 + 8192 + k * 32, 0, 1024, kLayoutSW128);
          uint64_t bd2 = make_smem_desc(b0 + 16384 + k * 32, 0, 1024, kLayoutSW128);
          asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::fill [%0], %1, %2, %3, 1;"
                       ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc) : "memory");
          asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::use [%0], %1, %2, %3, 1;"
                       ::"r"(tmem + 64), "l"(ad), "l"(bd1), "r"(idesc) : "memory");
          asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::lastuse [%0], %1, %2, %3, 1;"
                       ::"r"(tmem + 128), "l"(ad), "l"(bd2), "r"(idesc) : "memory");
        } else if constexpr (V == 8 || V == 9 || V == 11 || V == 12 || (V >= 16 && V < 30)) {
          // conv row pattern: A shifted by dx*128 B (V=8) or aligned (V=9), B = N192 block of dx
          const int dx = it % 3;
          const uint32_t ash = (V == 9) ? 0u : (uint32_t)dx * 128u;
          uint64_t ad8 = make_smem_desc(a0 + ash + k * 32, 0, 1024, kLayoutSW128);
          uint64_t bd8 = make_smem_desc(b0 + dx * 24576 + k * 32, 0, 1024, kLayoutSW128);
          mma_f16_ss(tmem, ad8, bd8, make_idesc(128, 192, kFmtF16, kFmtF16), 1);
        } else if constexpr (V == 10) {
          // split step: N128 + N64 into different columns
          uint64_t bd1 = make_smem_desc(b0 + 16384 + k * 32, 0, 1024, kLayoutSW128);
          mma_f16_ss(tmem, ad, bd, make_idesc(128, 128, kFmtF16, kFmtF16), 1);
          mma_f16_ss(tmem + 128, ad, bd1, make_idesc(128, 64, kFmtF16, kFmtF16), 1);
        } else if constexpr (V == 13 || V == 14) {
          // split step with A reuse: N128 (collector::a::fill) + N64 (collector::a::lastuse)
          uint64_t bd1 = make_smem_desc(b0 + 16384 + k * 32, 0, 1024, kLayoutSW128);
          const uint32_t i128 = make_idesc(128, 128, kFmtF16, kFmtF16), i64 = make_idesc(128, 64, kFmtF16, kFmtF16);
          if constexpr (V == 13) {
            asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::fill [%0], %1, %2, %3, 1;"
                         ::"r"(tmem), "l"(ad), "l"(bd), "r"(i128) : "memory");
            asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::lastuse [%0], %1, %2, %3, 1;"
                         ::"r"(tmem + 128), "l"(ad), "l"(bd1), "r"(i64) : "memory");
          } else {  // N64 first then N128
            asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::fill [%0], %1, %2, %3, 1;"
                         ::"r"(tmem + 128), "l"(ad), "l"(bd1), "r"(i64) : "memory");
            asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::lastuse [%0], %1, %2, %3, 1;"
                         ::"r"(tmem), "l"(ad), "l"(bd), "r"(i128) : "memory");
          }
        } else if constexpr (V == 15) {
          // three N64 pieces sharing A (s=7 first step pattern)
          uint64_t bd1 = make_smem_desc(b0 + 8192 + k * 32, 0, 1024, kLayoutSW128);
          uint64_t bd2 = make_smem_desc(b0 + 16384 + k * 32, 0, 1024, kLayoutSW128);
          const uint32_t i64 = make_idesc(128, 64, kFmtF16, kFmtF16);
          asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::fill [%0], %1, %2, %3, 1;"
                       ::"r"(tmem), "l"(ad), "l"(bd), "r"(i64) : "memory");
          asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::use [%0], %1, %2, %3, 1;"
                       ::"r"(tmem + 64), "l"(ad), "l"(bd1), "r"(i64) : "memory");
          asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::lastuse [%0], %1, %2, %3, 1;"
                       ::"r"(tmem + 128), "l"(ad), "l"(bd2), "r"(i64) : "memory");
        } else if constexpr (V == 7) {
          uint64_t adn = make_smem_desc(a0 + (it & 15) * 16 + k * 2 * 2304, 2304, 128, kLayoutNone);
          uint64_t bdn = make_smem_desc(b0 + k * 2 * 1024, 1024, 128, kLayoutNone);
          mma_f16_ss(tmem, adn, bdn, idesc, 1);
        }
      }
    }
    mma_commit(&bar);
    bool ok = mbar_wait_bounded(&bar, 0, 1ull << 26);
    long long t1 = clock64();
    if (!ok) atomicAdd(err, 1);
    cycles[blockIdx.x] = t1 - t0;
    if constexpr (V == 11 || V == 12 || (V >= 16 && V < 30)) *reinterpret_cast<volatile uint32_t*>(smem + 110 * 1024) = 1;
  }
  if constexpr (V >= 16 && V < 30) {
    // warp 1, lanes 0-3: bulk traffic, each lane through its own 8 KB buffer
    // at 112 + 8*lane KB (4 copies in flight)
    volatile uint32_t* flag = reinterpret_cast<volatile uint32_t*>(smem + 110 * 1024);
    __shared__ uint64_t tb[4];
    __shared__ unsigned long long moved[4];
    const int ln = tid & 31;
    if (warp == 1 && ln < 4) { mbar_init(&tb[ln], 1); moved[ln] = 0; }
    if (tid == 32) fence_barrier_init();
    __syncwarp();
    if (warp == 1 && ln < 4) {
      uint32_t ph = 0;
      unsigned long long n = 0;
      uint8_t* buf = smem + (112 + 8 * ln) * 1024;
      for (uint32_t i = 0; *flag == 0; ++i) {
        uint8_t* g = gbuf + (size_t)(((blockIdx.x * 4 + ln) * 64 + (i % 64)) % 16384) * 8192;
        if constexpr (V == 16 || V == 18) {
          mbar_arrive_expect_tx(&tb[ln], 8192);
          bulk_load(buf, g, 8192, &tb[ln]);
          mbar_wait(&tb[ln], ph);
          ph ^= 1;
          n += 8192;
        }
        if constexpr (V == 17 || V == 18) {
          bulk_store_g(g + (size_t)8192 * 16384, smem_u32(buf), 8192);
          bulk_commit();
          bulk_wait_read<0>();
          n += 8192;
        }
        if constexpr (V == 19) {  // two 4 KB tensor-store boxes per 8 KB buffer
          const int row = (int)((blockIdx.x * 4 + ln) * 64 + (i % 64)) % 4096;
          tma_store_4d(&tmap, buf, 0, 0, row, 0);
          tma_store_4d(&tmap, buf + 4096, 0, 32, row, 0);
          bulk_commit();
          bulk_wait_read<0>();
          n += 8192;
        }
      }
      bulk_wait<0>();
      moved[ln] = n;
    }
    if constexpr (V == 18 || V == 19) {
      if (warp >= 2) {
        uint4* region = reinterpret_cast<uint4*>(smem + 104 * 1024) + (warp - 2) * 32 * 4;
        const uint4 v = make_uint4(tid, 1, 2, 3);
        while (*flag == 0) {
#pragma unroll
          for (int j = 0; j < 4; ++j) region[j * 32 + (tid & 31)] = v;
        }
      }
    }
    __syncwarp();
    if (tid == 32) cycles[gridDim.x + blockIdx.x] = (long long)(moved[0] + moved[1] + moved[2] + moved[3]);
  }
  if constexpr (V == 11 || V == 12) {
    if (warp != 0) {
      volatile uint32_t* flag = reinterpret_cast<volatile uint32_t*>(smem + 110 * 1024);
      uint4* region = reinterpret_cast<uint4*>(smem + 104 * 1024) + (warp - 1) * 32 * 4;
      const uint4 v = make_uint4(tid, 1, 2, 3);
      while (*flag == 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) region[j * 32 + (tid & 31)] = v;
        if constexpr (V == 12) __nanosleep(200);
      }
    }
  }
  __syncwarp();
  if (warp != 0) mbar_wait_bounded(&bar, 0, 1ull << 26);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tmem);
}

// issue-queue probe: clock after each of 24 back-to-back N=192 MMAs (96 cyc each)
__global__ void __launch_bounds__(128, 1) k_queue(long long* out, int gap) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < (64 * 1024) / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_async_smem();
  if (warp == 0) tmem_alloc<256>(&tbase);
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 32768);
    const uint32_t idesc = make_idesc(128, 192, kFmtF16, kFmtF16);
    long long t[25];
    t[0] = clock64();
    for (int i = 0; i < 24; ++i) {
      uint64_t ad = make_smem_desc(a0 + (i & 3) * 32, 0, 1024, kLayoutSW128);
      uint64_t bd = make_smem_desc(b0 + (i & 3) * 32, 0, 1024, kLayoutSW128);
      mma_f16_ss(tmem, ad, bd, idesc, 1);
      t[i + 1] = clock64();
      if (gap) { long long w = clock64(); while (clock64() - w < gap) {} }
    }
    mma_commit(&bar);
    mbar_wait_bounded(&bar, 0, 1ull << 26);
    long long tend = clock64();
    for (int i = 0; i <= 24; ++i) out[i] = t[i] - t[0];
    out[25] = tend - t[0];
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tmem);
}

static void run_queue_probe() {
  long long* d; CK(cudaMalloc(&d, 26 * 8));
  const int smem = 64 * 1024 + 1024;
  CK(cudaFuncSetAttribute(k_queue, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int gap : {0, 0, 200}) {
    k_queue<<<1, 128, smem>>>(d, gap);
    CK(cudaDeviceSynchronize());
    long long h[26]; CK(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
    printf("QUEUE gap=%d issue-clock after MMA i:", gap);
    for (int i = 1; i <= 24; ++i) printf(" %lld", h[i]);
    printf(" | all done %lld\n", h[25]);
  }
  cudaFree(d);
}

static void run_layout_tests() {
  std::vector<__half> A(kRowsA * 64), B(64 * 64);
  std::vector<float> Af(kRowsA * 64), Bf(64 * 64);
  srand(1);
  for (int i = 0; i < kRowsA * 64; ++i) { float v = (rand() % 17 - 8) / 8.0f; A[i] = __float2half(v); Af[i] = v; }
  for (int i = 0; i < 64 * 64; ++i) { float v = (rand() % 13 - 6) / 4.0f; B[i] = __float2half(v); Bf[i] = v; }
  __half *dA, *dB; float* dO; int* dErr;
  CK(cudaMalloc(&dA, A.size() * 2)); CK(cudaMalloc(&dB, B.size() * 2));
  CK(cudaMalloc(&dO, 128 * 64 * 4)); CK(cudaMalloc(&dErr, 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
  const int smem = kRowsA * 128 + 64 * 128 + 1024;
  CK(cudaFuncSetAttribute(k_layout, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  std::vector<float> O(128 * 64);
  const char* names[3] = {"SW128 bo=0", "SW128 bo=s&7", "NOSWZ planar"};
  for (int layout = 0; layout < 3; ++layout) {
    for (int s = 0; s <= 9; ++s) {
      CK(cudaMemset(dErr, 0, 4));
      CK(cudaMemset(dO, 0, 128 * 64 * 4));
      k_layout<<<1, 128, smem>>>(dA, dB, dO, layout, s, dErr);
      CK(cudaDeviceSynchronize());
      int herr; CK(cudaMemcpy(&herr, dErr, 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost));
      double maxerr = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
          double ref = 0;
          for (int k = 0; k < 64; ++k) ref += (double)Af[(m + s) * 64 + k] * Bf[n * 64 + k];
          maxerr = fmax(maxerr, fabs(ref - O[m * 64 + n]));
        }
      printf("LAYOUT %-14s shift=%d  max_abs_err=%.3e  timeout=%d  %s\n", names[layout], s, maxerr, herr,
             maxerr < 1e-3 && herr == 0 ? "OK" : "FAIL");
    }
  }
  cudaFree(dA); cudaFree(dB); cudaFree(dO); cudaFree(dErr);
}

template <int V>
static void run_rate(const char* name, int ctas, double macs_per_iter) {
  long long* dC; int* dErr;
  CK(cudaMalloc(&dC, 2 * ctas * sizeof(long long))); CK(cudaMalloc(&dErr, 4)); CK(cudaMemset(dErr, 0, 4));
  CK(cudaMemset(dC, 0, 2 * ctas * sizeof(long long)));
  static uint8_t* gbuf = nullptr;
  static CUtensorMap tmap;
  if (!gbuf) {
    CK(cudaMalloc(&gbuf, (size_t)2 * 16384 * 8192));
    void* fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q));
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
    // [1][4096 rows][64 px][64 ch] fp16, box {64 ch, 32 px, 1, 1}, SW128 (the conv epilogue's store)
    cuuint64_t dims[4] = {64, 64, 4096, 1};
    cuuint64_t strides[3] = {128, 64 * 128, (cuuint64_t)4096 * 64 * 128};
    cuuint32_t box[4] = {64, 32, 1, 1}, estr[4] = {1, 1, 1, 1};
    CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, gbuf + (size_t)16384 * 8192, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("tensor map encode failed %d\n", (int)r); exit(1); }
  }
  const int smem = ((V >= 16 && V < 30) ? 144 : 112) * 1024 + 1024;
  CK(cudaFuncSetAttribute(k_rate<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int iters = 4096;
  k_rate<V><<<ctas, 128, smem>>>(64, dC, dErr, gbuf, tmap);  // warm
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_rate<V><<<ctas, 128, smem>>>(iters, dC, dErr, gbuf, tmap);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<long long> c(ctas);
  CK(cudaMemcpy(c.data(), dC, ctas * sizeof(long long), cudaMemcpyDeviceToHost));
  int herr; CK(cudaMemcpy(&herr, dErr, 4, cudaMemcpyDeviceToHost));
  double avg = 0; for (auto v : c) avg += v; avg /= ctas;
  double n_mma = (double)iters * (V == 6 || V == 15 ? 12 : (V == 10 || V == 13 || V == 14 ? 8 : 4));
  double tflops = 2.0 * macs_per_iter * iters * ctas / (ms * 1e-3) / 1e12;
  std::vector<long long> mv(ctas);
  CK(cudaMemcpy(mv.data(), dC + ctas, ctas * sizeof(long long), cudaMemcpyDeviceToHost));
  double bytes = 0; for (auto v : mv) bytes += v; bytes /= ctas;
  printf("RATE %-26s ctas=%3d cyc/mma=%7.2f  cyc/iter=%8.2f  MAC/clk/SM=%7.1f  %.1f TFLOP/s  bulk B/clk/SM=%5.1f  timeout=%d\n",
         name, ctas, avg / n_mma, avg / iters, macs_per_iter * iters / avg, tflops, bytes / avg, herr);
  cudaFree(dC); cudaFree(dErr);
}

int main(int argc, char** argv) {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("device %s sm_%d%d SMs=%d smemOptin=%zu\n", p.name, p.major, p.minor, p.multiProcessorCount,
         p.sharedMemPerBlockOptin);
  if (argc < 2) run_layout_tests();
  run_queue_probe();
  if (argc > 1 && argv[1][0] == 'q') return 0;
  const int sms = p.multiProcessorCount;
  for (int ctas : {1, sms}) {
    run_rate<0>("f16 M128 N64 K64", ctas, 128.0 * 64 * 64);
    run_rate<1>("f16 M128 N128 K64", ctas, 128.0 * 128 * 64);
    run_rate<2>("f16 M128 N192 K64", ctas, 128.0 * 192 * 64);
    run_rate<3>("f16 M128 N256 K64", ctas, 128.0 * 256 * 64);
    run_rate<4>("tf32 M128 N64 K32", ctas, 128.0 * 64 * 32);
    run_rate<5>("e4m3 M128 N64 K128", ctas, 128.0 * 64 * 128);
    run_rate<30>("f16 M128 N96 K64", ctas, 128.0 * 96 * 64);
    run_rate<31>("e4m3 M128 N96 K128", ctas, 128.0 * 96 * 128);
    run_rate<32>("e4m3 M128 N192 K128", ctas, 128.0 * 192 * 128);
    run_rate<6>("f16 N64 x3 collector::a", ctas, 3 * 128.0 * 64 * 64);
    run_rate<7>("f16 N64 noswz shifted A", ctas, 128.0 * 64 * 64);
    run_rate<8>("f16 N192 conv dx-shifted A", ctas, 128.0 * 192 * 64);
    run_rate<9>("f16 N192 conv aligned A", ctas, 128.0 * 192 * 64);
    run_rate<10>("f16 N128+N64 split", ctas, 128.0 * 192 * 64);
    run_rate<13>("N128 fill + N64 lastuse", ctas, 128.0 * 192 * 64);
    run_rate<14>("N64 fill + N128 lastuse", ctas, 128.0 * 192 * 64);
    run_rate<15>("3x N64 fill/use/lastuse", ctas, 128.0 * 192 * 64);
    run_rate<11>("N192 conv + STS flood", ctas, 128.0 * 192 * 64);
    run_rate<12>("N192 conv + STS throttled", ctas, 128.0 * 192 * 64);
    run_rate<16>("N192 conv + bulk loads", ctas, 128.0 * 192 * 64);
    run_rate<17>("N192 conv + bulk stores", ctas, 128.0 * 192 * 64);
    run_rate<18>("N192 conv + loads+stores+STS", ctas, 128.0 * 192 * 64);
    run_rate<19>("N192 conv + TMA tensor st+STS", ctas, 128.0 * 192 * 64);
  }
  printf("DONE\n");
  return 0;
}
