// conv0_tc.cu — K1 (the first conv, Conv2d(1|4, 64, 3, p=1, bias) + ReLU,
// /root/reference/pkg/trainer/src/tvsurrogate/model.py:37-38) on tcgen05 for
// the fast path, which stores fp16 NHWC activations.
//
// The CUDA-core K1 spends ~750 issue slots per pixel on 576 FFMAs and the
// ReLU/convert/store around them (issue-bound at 89%, 170 us on config 2).
// Here each 128-pixel strip row is one M=128, N=64 GEMM with the 3x3 taps as
// K, kept fp32-accurate by splitting both operands into TF32 hi + lo parts:
//
//   A[px] = [x_hi(t) | x_lo(t) | x_hi(t) | 0]    B[co] = [W_hi | W_hi | W_lo | 0]
//
// so one K chain sums x_hi*W_hi + x_lo*W_hi + x_hi*W_lo (x_lo*W_lo ~ 2^-22 is
// dropped).  Weights: hi = RNA_tf32(w), lo = RNA_tf32(w - hi); inputs: hi =
// the tensor core's truncation of x, lo = x - trunc(x) (see the A build):
// 21-22 significant bits of each operand, fp32 range (an fp16 split would
// overflow past 65504).  The tf32 products are exact in the fp32 accumulator,
// so the pre-activation matches the fp32 FFMA sum to a few fp32 ulps before
// the fp16 rounding.
//
// kKB = 1: full-resolution conv0, 9 taps -> K = 27 of one 32-element SW128
//          block (128 B per pixel row).
// kKB = 4: the unshuffle = 2 variant's Conv2d(4, 64): input channel c = 2i + j
//          of half-res pixel (Y, X) is x[2Y+i][2X+j] (torch pixel_unshuffle
//          order), 36 taps -> K = 108 of four blocks.
//
// A CTA (4 warps, one pixel per thread) takes kTiles strip rows per round:
// builds their A rows, one thread issues the MMA chains into kTiles TMEM
// accumulators, and the next round's taps are loaded while they run.  The
// epilogue adds the bias, applies ReLU with the fp16 rounding
// (cvt.rn.relu.f16x2.f32), stages the rows in the freed A tile and copies each
// strip row's 16 KB out coalesced.  Several CTAs share an SM (4 for K = 9,
// register bound; 2 for K = 36, smem bound), so one CTA's tile build overlaps
// another's MMAs and stores.  Config 2: 149 us (CUDA-core K1: 170 us; the
// 537 MB write alone is 84 us at the copy bandwidth).
#include <algorithm>

#include "common.cuh"
#include "sm100.cuh"

namespace tvs {

template <int kKB>
struct Conv0TcCfg {
  static constexpr int kTaps = kKB == 1 ? 9 : 36;
  static constexpr int kTiles = kKB == 1 ? 2 : 1;     // strip rows per CTA iteration (one accumulator each)
  static constexpr int kPerSm = kKB == 1 ? 4 : 2;     // resident CTAs per SM (TMEM / smem bound)
  static constexpr int kTileA = kKB * 128 * 128;      // 128 pixel rows x 128 B per K block
  static constexpr int kABytes = kTiles * kTileA;
  static constexpr int kBBytes = kKB * 64 * 128;      // 64 output-channel rows x 128 B per K block
  static constexpr size_t kSmem = 1024 + kABytes + kBBytes;
  static constexpr int kTmemCols = kTiles * 64 <= 64 ? 64 : (kTiles * 64 <= 128 ? 128 : 256);
};

__device__ __forceinline__ float tf32_rna(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}

// element kk (0 .. 32*kKB-1) of SW128 K-major row `row` inside a tile of
// 8-row / 1024-byte swizzle atoms, one 128-row (or 64-row) tile per K block
__device__ __forceinline__ uint32_t sw128_off(int row, int kk, int rows_per_block) {
  const int kb = kk >> 5, c = (kk & 31) >> 2;
  return (uint32_t)(kb * rows_per_block * 128 + row * 128 + ((c ^ (row & 7)) << 4) + (kk & 3) * 4);
}

// (image, row, first pixel) of strip row `tile` (32-bit: tiles < 2^31)
struct TileXY {
  int b, y, x0;
};
__device__ __forceinline__ TileXY tile_xy(int tile, int strips, int H) {
  const int by = tile / strips;
  return {by / H, by - (by / H) * H, (tile - by * strips) * 128};
}

// taps of pixel x0 + t of strip row `c`; zero outside the image
template <int kKB>
__device__ __forceinline__ void conv0_taps(const float* __restrict__ x, TileXY c, int H, int W, int t,
                                           float (&tap)[Conv0TcCfg<kKB>::kTaps]) {
  const int px = c.x0 + t, y = c.y;
  if constexpr (kKB == 1) {
    const float* img = x + (long long)c.b * H * W;
#pragma unroll
    for (int ky = 0; ky < 3; ++ky)
#pragma unroll
      for (int kx = 0; kx < 3; ++kx) {
        const int yy = y + ky - 1, xx = px + kx - 1;
        tap[ky * 3 + kx] = (yy >= 0 && yy < H && xx >= 0 && xx < W) ? __ldg(img + (long long)yy * W + xx) : 0.0f;
      }
  } else {  // half-res grid (H, W); full-res plane (2H, 2W)
    const float* img = x + (long long)c.b * (2 * H) * (2 * W);
#pragma unroll
    for (int ky = 0; ky < 3; ++ky)
#pragma unroll
      for (int kx = 0; kx < 3; ++kx) {
        const int yy = y + ky - 1, xx = px + kx - 1;
        const bool ok = yy >= 0 && yy < H && xx >= 0 && xx < W;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const float2 v = ok ? __ldg(reinterpret_cast<const float2*>(img + (long long)(2 * yy + i) * (2 * W) + 2 * xx))
                              : make_float2(0.0f, 0.0f);
          tap[(2 * i) * 9 + ky * 3 + kx] = v.x;      // channel c = 2i + 0
          tap[(2 * i + 1) * 9 + ky * 3 + kx] = v.y;  // channel c = 2i + 1
        }
      }
  }
}

template <int kKB>
__global__ void __launch_bounds__(128) conv0_tc_kernel(const float* __restrict__ x,
                                                       const __grid_constant__ CUtensorMap out_map,
                                                       const uint8_t* __restrict__ bpack,
                                                       const float* __restrict__ bias,
                                                       const int* __restrict__ escale, int B, int H, int W) {
  using Cfg = Conv0TcCfg<kKB>;
  constexpr int n = Cfg::kTaps;
  constexpr int NT = Cfg::kTiles;
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t mma_done;
  __shared__ uint32_t tmem_base;
  __shared__ float sBias[64];
  uint8_t* sA = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = sA + Cfg::kABytes;
  const int t = threadIdx.x, warp = t >> 5;

  // PDL: the first hidden layer may start its prologue (it waits for this grid)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (warp == 0) tmem_alloc<Cfg::kTmemCols>(&tmem_base);
  {  // weights: packed SW128 tf32 rows, a plain copy into shared memory
    const uint4* src = reinterpret_cast<const uint4*>(bpack);
    uint4* dst = reinterpret_cast<uint4*>(sB);
    for (int i = t; i < Cfg::kBBytes / 16; i += 128) dst[i] = __ldg(src + i);
  }
  if (t < 64) sBias[t] = bias[t];
  if (t == 0) {
    mbar_init(&mma_done, 1);
    fence_barrier_init();
  }
  fence_async_smem();  // generic smem writes (B) -> the tensor core's async proxy
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = make_idesc(128, 64, kFmtTF32, kFmtTF32);
  const uint64_t adesc0 = make_smem_desc(smem_u32(sA), 0, 1024, kLayoutSW128);
  const uint64_t bdesc0 = make_smem_desc(smem_u32(sB), 0, 1024, kLayoutSW128);
  const uint32_t lane_addr = (uint32_t)(warp * 32) << 16;
  const int strips = (W + 127) / 128;
  const int tiles = B * H * strips;  // < 2^31 (launch_conv0_tc)
  const int step = gridDim.x * NT;
  uint32_t phase = 0;
  // tiles blockIdx.x*NT + i of each round; the next round's taps are loaded
  // while this round's MMAs and epilogue run (past the end: any valid row,
  // result unused)
  float tap[NT][n];
  int base = blockIdx.x * NT;
#pragma unroll
  for (int i = 0; i < NT; ++i) conv0_taps<kKB>(x, tile_xy(min(base + i, tiles - 1), strips, H), H, W, t, tap[i]);
  // programmatic launch after the input-scale kernel: the exponents (and the
  // right to overwrite the activation buffer) come after this wait; x was
  // complete before that kernel started.  A no-op for a plain launch.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (; base < tiles; base += step) {
    // ---- A rows of this thread's pixel in each tile: taps split hi / lo
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      const uint32_t arow = smem_u32(sA + i * Cfg::kTileA);
#pragma unroll
      for (int c4 = 0; c4 < 8 * kKB; ++c4) {  // 16-byte chunks of the row
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int kk = c4 * 4 + e;
          // the tensor core reads a tf32 operand as the top 19 bits of the fp32
          // container (the low 13 mantissa bits are ignored), so x itself is
          // x_hi = trunc(x) and x_lo = x - trunc(x) (exact) is the rest,
          // itself used to 10 bits: 2 instructions per tap instead of four
          // explicit RNA conversions (3 instructions each on sm_100)
          float r = 0.0f;
          if (kk < n) {
            r = tap[i][kk];
          } else if (kk < 2 * n) {
            const float xv = tap[i][kk - n];
            r = xv - __uint_as_float(__float_as_uint(xv) & 0xffffe000u);
          } else if (kk < 3 * n) {
            r = tap[i][kk - 2 * n];
          }
          v[e] = r;
        }
        st_shared_v4(arow + sw128_off(t, c4 * 4, 128), __float_as_uint(v[0]), __float_as_uint(v[1]),
                     __float_as_uint(v[2]), __float_as_uint(v[3]));
      }
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();  // A complete; every warp's TMEM reads of the previous round are done
    tc_fence_after();
    if (t == 0) {
#pragma unroll
      for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int k = 0; k < 4 * kKB; ++k) {  // K8 steps: 32 B along the row, blocks of 16 / 8 KB
          const uint32_t ka = (uint32_t)(i * Cfg::kTileA + (k >> 2) * 128 * 128 + (k & 3) * 32) >> 4;
          const uint32_t kb = (uint32_t)((k >> 2) * 64 * 128 + (k & 3) * 32) >> 4;
          mma_tf32_ss(tmem + i * 64, adesc0 + ka, bdesc0 + kb, idesc, k > 0 ? 1u : 0u);
        }
      mma_commit(&mma_done);
    }
    // next round's taps (global loads in flight during the MMAs and the epilogue)
#pragma unroll
    for (int i = 0; i < NT; ++i)
      conv0_taps<kKB>(x, tile_xy(min(base + step + i, tiles - 1), strips, H), H, W, t, tap[i]);
    mbar_wait(&mma_done, phase);
    phase ^= 1;
    tc_fence_after();
    // ---- epilogue: lane quarter `warp` = pixels 32*warp .. +31 of each tile,
    // staged through the (now free) A tile in the SW128 layout, then written
    // by one TMA tensor store per strip row (box 64 ch x 128 px; the tensor
    // map clips a partial last strip)
#pragma unroll 1
    for (int i = 0; i < NT; ++i) {
      // 2^-e of this tile's image (exact; 1 for in-range inputs)
      const int ti = min(base + i, tiles - 1);
      const float sc = escale ? pow2i(-__ldg(escale + tile_xy(ti, strips, H).b)) : 1.0f;
      uint32_t acc[4][16];
#pragma unroll
      for (int j = 0; j < 4; ++j) tmem_ld16(tmem + lane_addr + i * 64 + j * 16, acc[j]);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 4; ++j) reg_fence16(acc[j]);
      const uint32_t srow = smem_u32(sA + i * Cfg::kTileA) + t * 128;
      const float2 sc2 = make_float2(sc, sc);
#pragma unroll
      for (int c8 = 0; c8 < 8; ++c8) {
        uint32_t pk[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int c = c8 * 8 + e * 2;
          // (acc + bias) * 2^-e, packed fp32x2 (FADD2 / FMUL2)
          float2 f = __fadd2_rn(make_float2(__uint_as_float(acc[c >> 4][c & 15]),
                                            __uint_as_float(acc[c >> 4][(c & 15) + 1])),
                                make_float2(sBias[c], sBias[c + 1]));
          if (sc != 1.0f) f = __fmul2_rn(f, sc2);
          asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(pk[e]) : "f"(f.y), "f"(f.x));
        }
        st_shared_v4(srow + ((c8 ^ (t & 7)) << 4), pk[0], pk[1], pk[2], pk[3]);
      }
    }
    fence_async_smem();  // staging (generic proxy) -> the TMA store (async proxy)
    tc_fence_before();
    __syncthreads();
    if (t == 0) {
#pragma unroll 1
      for (int i = 0; i < NT; ++i) {
        if (base + i >= tiles) break;
        const TileXY c = tile_xy(base + i, strips, H);
        tma_store_4d(&out_map, sA + i * Cfg::kTileA, 0, c.x0, c.y, c.b);
      }
      bulk_commit();
      bulk_wait_read<0>();  // the staging tiles are the next round's A tiles
    }
    __syncthreads();
  }
  if (t == 0) bulk_wait<0>();  // stores complete before the grid ends (PDL dependents read them)
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem);
  }
}

// B pack: 64 rows (output channels) x 32*kKB tf32 [W_hi | W_hi | W_lo | 0],
// SW128 K-major, from fp32 weights w[co][tap] (n taps per channel).
__global__ void pack_conv0_tc_kernel(const float* __restrict__ w, int n, int kb_count, uint8_t* __restrict__ out) {
  const int co = blockIdx.x, kk = threadIdx.x;
  if (kk >= 32 * kb_count) return;
  float r = 0.0f;
  if (kk < n) {
    r = tf32_rna(w[co * n + kk]);
  } else if (kk < 2 * n) {
    r = tf32_rna(w[co * n + kk - n]);
  } else if (kk < 3 * n) {
    const float v = w[co * n + kk - 2 * n];
    r = tf32_rna(v - tf32_rna(v));
  }
  *reinterpret_cast<float*>(out + sw128_off(co, kk, 64)) = r;
}

size_t conv0_tc_pack_bytes(int in_ch) { return in_ch == 1 ? Conv0TcCfg<1>::kBBytes : Conv0TcCfg<4>::kBBytes; }

cudaError_t launch_pack_conv0_tc(const float* w, int in_ch, uint8_t* out, cudaStream_t st) {
  const int kb = in_ch == 1 ? 1 : 4;
  pack_conv0_tc_kernel<<<64, 32 * kb, 0, st>>>(w, 9 * in_ch, kb, out);
  return cudaGetLastError();
}

cudaError_t launch_conv0_tc(int in_ch, const float* x, const CUtensorMap& out_map, const uint8_t* bpack,
                            const float* bias, const int* escale, int B, int H, int W, int num_sms, bool pdl,
                            cudaStream_t st) {
  static std::mutex mu;
  static uint64_t done = 0;
  cudaError_t e = once_per_device(mu, done, [] {
    cudaError_t r = cudaFuncSetAttribute(conv0_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)Conv0TcCfg<1>::kSmem);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(conv0_tc_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)Conv0TcCfg<4>::kSmem);
    return r;
  });
  if (e != cudaSuccess) return e;
  const long long tiles = (long long)B * H * ((W + 127) / 128);
  if (tiles >= (1LL << 31) - 1024) return cudaErrorInvalidValue;  // 32-bit tile indices
  const int nt = in_ch == 1 ? Conv0TcCfg<1>::kTiles : Conv0TcCfg<4>::kTiles;
  const int per_sm = in_ch == 1 ? Conv0TcCfg<1>::kPerSm : Conv0TcCfg<4>::kPerSm;
  const int grid = (int)std::max(1LL, std::min<long long>((tiles + nt - 1) / nt, (long long)num_sms * per_sm));
  // PDL only behind the input-scale kernel (which reads x and nothing else);
  // as a forward's first kernel K1 is a plain launch, so it cannot overlap
  // the previous forward's head or whatever produced x
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  if (in_ch == 1) {
    cfg.dynamicSmemBytes = Conv0TcCfg<1>::kSmem;
    return cudaLaunchKernelEx(&cfg, conv0_tc_kernel<1>, x, out_map, bpack, bias, escale, B, H, W);
  }
  cfg.dynamicSmemBytes = Conv0TcCfg<4>::kSmem;
  return cudaLaunchKernelEx(&cfg, conv0_tc_kernel<4>, x, out_map, bpack, bias, escale, B, H, W);
}

}  // namespace tvs
