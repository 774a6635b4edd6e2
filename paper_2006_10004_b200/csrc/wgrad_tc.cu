// wgrad_tc.cu — the training step's weight gradient of one 3x3 conv layer on
// tcgen05 (the backward of model.py:40 / :44 as driven by
// training.py:45-61):
//
//   dW[co][ci][ky][kx] = alpha * sum_p G[p][co] * A[p + (ky-1)(W+2) + (kx-1)][ci]
//
// over ALL pixels p of the zero-bordered buffers (train.cu "Layout": border
// pixels carry a zero gradient and the shifted pixel of an interior p stays in
// its own image, so one sum over the padded pixel list is the exact tap sum).
// It replaces 9 cuBLAS split-K GEMMs + 9 split-K reductions per layer (190 us
// per layer at 8 x 128 x 128: 2.6 of the step's 7.7 ms).
//
// GEMM shape.  The pixel list is the K dimension, and both operands are stored
// pixel-major ([pixel][channel], channel contiguous): MN-major operands.  A TMA
// box of R pixel rows x 64 fp16 channels (128 B per row, SWIZZLE_128B) is
// exactly the canonical MN-major SW128 layout (64 MN elements x 8 K rows per
// 1024-byte atom; the descriptor's leading byte offset is the stride between
// 64-element MN blocks, its stride byte offset the 1024 B between 8-row K
// groups), so the tiles feed tcgen05.mma as they land, with the instruction
// descriptor's A-major / B-major bits set.
//   * D[M = 128][N = 64]: M = two taps x 64 input channels, N = 64 output
//     channels.  The A operand's two 64-channel MN blocks are the SAME
//     activation tile at two pixel shifts: the block stride (LBO) is the byte
//     distance between the taps' shifted views (128 B for kx -> kx + 1), the
//     trick the forward conv uses for its dx taps, here along K.
//   * 9 taps = pairs (0,1) (2,3) (4,5) (6,7) (7,8): five accumulators of 64
//     TMEM columns (tap 7 is computed twice; the reduction reads it once).
//   * per chunk of R = 128 pixels a stage holds G[R] and, for each ky, the
//     activation rows p0 + (ky-1)(W+2) - 1 .. + R (R + 2 rows): 68 KB, 3 stages.
// Split-K: CTA i sums chunks i, i + grid, ...; its five accumulators go to a
// partial buffer [cta][5][128][64] fp32 and `wgrad_reduce_kernel` adds the
// partials in a fixed order (deterministic, like cuBLAS split-K), applies
// alpha = 2^-s (the gradient operand's power-of-two scale) and writes the
// Conv2d weight layout.
#include <algorithm>

#include "common.cuh"
#include "host_util.h"
#include "sm100.cuh"

namespace tvs {

namespace wg {
constexpr int kR = 128;                    // pixels per chunk (K per stage)
constexpr int kGBytes = kR * 128;          // 16 KB
constexpr int kARows = kR + 2;             // one tile per ky, all three kx shifts inside
constexpr int kABytes = kARows * 128;      // 16640
constexpr int kAStride = 17408;            // 1024-aligned tile stride
constexpr int kStage = kGBytes + 3 * kAStride;  // 68608
constexpr int kStages = 3;
constexpr int kPairs = 5;
constexpr size_t kSmem = 1024 + (size_t)kStages * kStage;
constexpr int kThreads = 192;              // w0 TMA, w1 MMA, w2-5 epilogue
constexpr uint32_t kTxBytes = kGBytes + 3 * kABytes;
}  // namespace wg

// first tap of accumulator `pair` and the byte distance to its second tap
__host__ __device__ constexpr int wg_tap0(int pair) { return pair < 4 ? 2 * pair : 7; }

__global__ void __launch_bounds__(wg::kThreads, 1)
wgrad_tc_kernel(const __grid_constant__ CUtensorMap gmap, const __grid_constant__ CUtensorMap amap, long long PP,
                int guard, int Wp /* W + 2 */, float* __restrict__ part) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t full[wg::kStages], empty[wg::kStages], acc_full;
  __shared__ uint32_t tmem_base_smem;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < wg::kStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(&acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&tmem_base_smem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_smem;
  const long long nchunks = (PP + wg::kR - 1) / wg::kR;

  if (warp == 0) {
    if (elect_one()) {
      prefetch_tmap(&gmap);
      prefetch_tmap(&amap);
      int stage = 0;
      uint32_t phase = 0;
      for (long long c = blockIdx.x; c < nchunks; c += gridDim.x) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* s = smem + stage * wg::kStage;
        const long long row = guard + c * wg::kR;  // buffer row of the chunk's first pixel
        mbar_arrive_expect_tx(&full[stage], wg::kTxBytes);
        tma_load_2d(s, &gmap, &full[stage], 0, (int)row);
#pragma unroll
        for (int ky = 0; ky < 3; ++ky)
          tma_load_2d(s + wg::kGBytes + ky * wg::kAStride, &amap, &full[stage], 0,
                      (int)(row + (long long)(ky - 1) * Wp - 1));
        if (++stage == wg::kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      // M = 128 (two 64-channel MN blocks of A), N = 64, both operands MN-major
      const uint32_t idesc = make_idesc(128, 64, kFmtF16, kFmtF16) | (1u << 15) | (1u << 16);
      int stage = 0;
      uint32_t phase = 0;
      bool first = true;
      for (long long c = blockIdx.x; c < nchunks; c += gridDim.x) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t sg = smem_u32(smem + stage * wg::kStage);
        const uint32_t sa = sg + wg::kGBytes;
#pragma unroll
        for (int ks = 0; ks < wg::kR / 16; ++ks) {
          const uint64_t bdesc = make_smem_desc(sg + ks * 2048, 1024, 1024, kLayoutSW128);
#pragma unroll
          for (int pr = 0; pr < wg::kPairs; ++pr) {
            const int t0 = wg_tap0(pr), t1 = t0 + 1;
            const uint32_t a0 = sa + (t0 / 3) * wg::kAStride + (t0 % 3) * 128;
            const uint32_t a1 = sa + (t1 / 3) * wg::kAStride + (t1 % 3) * 128;
            const uint64_t adesc = make_smem_desc(a0 + ks * 2048, a1 - a0, 1024, kLayoutSW128);
            mma_f16_ss(tmem + pr * 64, adesc, bdesc, idesc, (first && ks == 0) ? 0u : 1u);
          }
        }
        mma_commit(&empty[stage]);
        first = false;
        if (++stage == wg::kStages) { stage = 0; phase ^= 1; }
      }
      mma_commit(&acc_full);
    }
  } else {
    // epilogue: lane quarter (warp % 4) of the five accumulators -> this CTA's partial
    const int quarter = warp & 3;
    const int m = quarter * 32 + lane;
    const bool any = (long long)blockIdx.x < nchunks;
    if (any) {
      mbar_wait(&acc_full, 0);
      tc_fence_after();
    }
    float* dst = part + ((size_t)blockIdx.x * wg::kPairs * 128 + m) * 64;
#pragma unroll 1
    for (int pr = 0; pr < wg::kPairs; ++pr) {
      uint32_t v[4][16];
      if (any) {
#pragma unroll
        for (int j = 0; j < 4; ++j) tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + pr * 64 + j * 16, v[j]);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int i = 0; i < 16; ++i) v[j][i] = 0u;
      }
      float4* d4 = reinterpret_cast<float4*>(dst + (size_t)pr * 128 * 64);
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i)
          d4[j * 4 + i] = make_float4(__uint_as_float(v[j][4 * i]), __uint_as_float(v[j][4 * i + 1]),
                                      __uint_as_float(v[j][4 * i + 2]), __uint_as_float(v[j][4 * i + 3]));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// dW[co][ci][tap] = alpha * sum_cta part[cta][pair][half*64 + ci][co] for co < rows
// (tap -> (pair, half): 0-7 -> (tap / 2, tap % 2), 8 -> (4, 1)).  A block of
// 256 threads = 64 output channels (co fastest: the partial reads coalesce) x 4
// slices of the CTA list; the slices are summed in a fixed order (deterministic).
__global__ void __launch_bounds__(256)
wgrad_reduce_kernel(const float* __restrict__ part, int nctas, int rows, const float* __restrict__ alpha,
                    float* __restrict__ dw) {
  const int co = threadIdx.x & 63, slice = threadIdx.x >> 6;
  const int ci = blockIdx.x & 63, tap = blockIdx.x >> 6;
  const int pair = tap < 8 ? tap >> 1 : 4, half = tap < 8 ? (tap & 1) : 1;
  const float* p = part + ((size_t)pair * 128 + half * 64 + ci) * 64 + co;
  const size_t stride = (size_t)wg::kPairs * 128 * 64;
  const int per = (nctas + 3) / 4, c0 = slice * per, c1 = min(nctas, c0 + per);
  float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f, s3 = 0.0f;
  int c = c0;
  for (; c + 4 <= c1; c += 4) {
    s0 += p[(size_t)c * stride];
    s1 += p[(size_t)(c + 1) * stride];
    s2 += p[(size_t)(c + 2) * stride];
    s3 += p[(size_t)(c + 3) * stride];
  }
  for (; c < c1; ++c) s0 += p[(size_t)c * stride];
  __shared__ float sh[4][64];
  sh[slice][co] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (slice == 0 && co < rows)
    dw[((size_t)co * 64 + ci) * 9 + tap] = ((sh[0][co] + sh[1][co]) + (sh[2][co] + sh[3][co])) * __ldg(alpha);
}

size_t wgrad_part_bytes(int num_sms) { return (size_t)num_sms * wg::kPairs * 128 * 64 * sizeof(float); }

// [rows][row_halves] fp16 pixel-major buffer as a 2-D tensor map over its first 64 channels
// (L2 promotion 128 B: the activation rows are 256 B (hi | lo) of which only the hi
// half is read; 256 B promotion fetched the lo halves too, 415 instead of 276 MB
// per layer at 64 x 128^2 in a kernel that runs at HBM speed)
CUtensorMap make_wgrad_map(const void* base, long long rows, int row_halves, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {64, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)row_halves * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = tvs_host::get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides,
                                      box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw tvs_host::TvsError(TVS_E_CUDA, "cuTensorMapEncodeTiled (wgrad) failed: " + std::to_string((int)r));
  return m;
}
CUtensorMap make_wgrad_gmap(const void* base, long long rows) { return make_wgrad_map(base, rows, 64, wg::kR); }
CUtensorMap make_wgrad_amap(const void* base, long long rows) { return make_wgrad_map(base, rows, 128, wg::kARows); }

cudaError_t launch_wgrad_tc(const CUtensorMap& gmap, const CUtensorMap& amap, long long PP, int guard, int W,
                            int rows, const float* alpha, float* part, float* dw, int num_sms, cudaStream_t st) {
  static std::mutex mu;
  static uint64_t done = 0;
  cudaError_t e = once_per_device(mu, done, [] {
    return cudaFuncSetAttribute(wgrad_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wg::kSmem);
  });
  if (e != cudaSuccess) return e;
  const long long nchunks = (PP + wg::kR - 1) / wg::kR;
  const int grid = (int)std::max(1LL, std::min<long long>(num_sms, nchunks));
  wgrad_tc_kernel<<<grid, wg::kThreads, wg::kSmem, st>>>(gmap, amap, PP, guard, W + 2, part);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  wgrad_reduce_kernel<<<9 * 64, 256, 0, st>>>(part, grid, rows, alpha, dw);
  return cudaGetLastError();
}

}  // namespace tvs
