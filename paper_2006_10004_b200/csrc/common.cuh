// common.cuh — shared constants and small helpers for the TVSpecNET kernels.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace tvs {

constexpr int kC = 64;            // hidden feature maps (ARCH_SPEC["channels"], model.py:19-26)
constexpr int kStripPx = 128;     // output pixels per strip = tcgen05 M
constexpr int kHaloPx = kStripPx + 2;
constexpr int kInRowBytes = kHaloPx * kC * 2;          // 16640: one halo'd input row, fp16 NHWC
constexpr int kInRowStride = 17408;                    // 1024-aligned ring stride (17 KB)
constexpr int kWdxBytes = 3 * kC * kC * 2;             // 24576: [W(dy=+1)|W(0)|W(-1)] for one dx
constexpr int kWBytes = 3 * kWdxBytes;                 // 73728 per hidden layer
constexpr int kOutRowBytes = kStripPx * kC * 2;        // 16384 staging for one output row
constexpr int kSlots = 8;                              // TMEM accumulator slots (64 cols each)

// Hidden-layer weight pack offset (fp16, SW128 K-major rows of 64 ci):
//   n = dyslot*64 + co with dyslot = 2 - ky  (dy=+1 -> 0, dy=0 -> 1, dy=-1 -> 2)
//   byte = kx*kWdxBytes + n*128 + ((ci/8) ^ (n&7))*16 + (ci%8)*2
__host__ __device__ __forceinline__ uint32_t wpack_offset(int co, int ci, int ky, int kx) {
  const int n = (2 - ky) * kC + co;
  return (uint32_t)kx * kWdxBytes + (uint32_t)n * 128u + (uint32_t)(((ci >> 3) ^ (n & 7)) << 4) +
         (uint32_t)((ci & 7) << 1);
}

// hidden-layer kernel launch geometry (conv_hidden_tc.cu)
constexpr int kStages = 6;              // input-row ring depth
constexpr int kHiddenThreads = 192;     // w0 TMA, w1 MMA, w2..w5 epilogue
constexpr size_t kHiddenSmem = 1024 /*align slack*/ + kWBytes + kStages * kInRowStride + 2 * kOutRowBytes + 1024;

struct HiddenArgs {
  int B, H, W;
  int strips;            // ceil(W / 128)
  int band_rows;         // output rows per work unit
  int bands;             // ceil(H / band_rows)
  int units;             // B * bands * strips
  const uint8_t* wpack;  // kWBytes, SW128-packed fp16
  const float* bias;     // 64 folded biases
};

// fp32 hidden layer (conv_edge.cu)
constexpr int kF32TileRows = 4, kF32TilePx = 32, kF32CiChunk = 16;
constexpr int kF32InRows = kF32TileRows + 2, kF32InPx = kF32TilePx + 2;
constexpr size_t kF32Smem = (size_t)(kF32InRows * kF32InPx * kF32CiChunk + kF32CiChunk * 9 * kC) * 4;
constexpr int kMaxBands = 8;

// host-side launchers (defined next to their kernels)
cudaError_t launch_hidden_f16(const CUtensorMap& tm_in, const CUtensorMap& tm_out, const HiddenArgs& a, int grid,
                              cudaStream_t st);
cudaError_t launch_pack_hidden_f16(const float* w, const float* scale, uint8_t* out, cudaStream_t st);
cudaError_t launch_fill(float* dst, float v, int n, cudaStream_t st);
cudaError_t launch_conv0(bool fp16_act, const float* x, void* act, const float* w0, const float* b0, int B, int H,
                         int W, cudaStream_t st);
cudaError_t launch_head(bool fp16_act, const void* act, const float* x, const float* wh, const float* bh,
                        float* bands, float* closure, int B, int H, int W, int K, int row0, int rows,
                        cudaStream_t st);
cudaError_t launch_hidden_f32(const float* in, float* out, const float* w, const float* scale, const float* shift,
                              int B, int H, int W, cudaStream_t st);
cudaError_t configure_kernels();  // one-time smem opt-ins

}  // namespace tvs
