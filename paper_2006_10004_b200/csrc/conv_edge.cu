// conv_edge.cu — the two thin ends of the TVSpecNET stack and the fp32
// hidden layer used by the fp32-accurate mode.
//
//   K1 conv0_kernel : Conv2d(1,64,3,p=1,bias) + ReLU  (model.py:37-38)
//       fp32 NCHW plane -> activation NHWC (fp16 or fp32).  K = 9, so it runs
//       on CUDA cores (0.10% of the FLOPs).
//   head_kernel<float> : Conv2d(64,K,3,p=1,bias) (model.py:44) + closure
//       plane (inference.py:34-42) for the fp32-accurate mode (fp32 NHWC
//       activations, fp64 accumulation).  The fast mode's head runs on
//       tcgen05 (conv_tc.cu).
//   hidden_f32_kernel : Conv2d(C,C)+BN+ReLU on fp32 NHWC (fp32-accurate
//       mode).  fp32 FFMA partial sums per 16-input-channel chunk, combined in
//       fp64, BatchNorm scale/shift applied after the sum in fp64.  A plain
//       sequential fp32 sum over all 576 terms lands at 1.0e-5 from the
//       reference - too close to the 1e-5 gate; chunked
//       partials are as good as full fp64 (5.1e-6).
#include <algorithm>
#include <type_traits>

#include <cuda_fp8.h>

#include "common.cuh"

namespace tvs {

// ------------------------------------------------------------------ K1 ----
template <typename T>
__device__ __forceinline__ void store_act8(T* dst, const float* v);
template <>
__device__ __forceinline__ void store_act8<__half>(__half* dst, const float* v) {
  uint4 o;
  __half2 h0 = __floats2half2_rn(v[0], v[1]), h1 = __floats2half2_rn(v[2], v[3]);
  __half2 h2 = __floats2half2_rn(v[4], v[5]), h3 = __floats2half2_rn(v[6], v[7]);
  o.x = *reinterpret_cast<uint32_t*>(&h0); o.y = *reinterpret_cast<uint32_t*>(&h1);
  o.z = *reinterpret_cast<uint32_t*>(&h2); o.w = *reinterpret_cast<uint32_t*>(&h3);
  *reinterpret_cast<uint4*>(dst) = o;
}
template <>
__device__ __forceinline__ void store_act8<float>(float* dst, const float* v) {
  reinterpret_cast<float4*>(dst)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(dst)[1] = make_float4(v[4], v[5], v[6], v[7]);
}

// One thread per pixel; the conv0 weights/bias arrive BY VALUE in the kernel
// parameter block (constant bank), so every FFMA takes its weight operand
// straight from the constant cache (no shared-memory loads).  128 pixels per
// block are contiguous in NHWC, so the block's output is staged through shared
// memory and written coalesced.
template <typename T, int C, bool kSplit = false>
__global__ void __launch_bounds__(128)
conv0_kernel(const float* __restrict__ x, T* __restrict__ act, const Conv0Params p, const int* __restrict__ escale,
             int B, int H, int W) {
  constexpr int P = (C == 64) ? 128 : 64;  // pixels per block (static smem <= 32 KB)
  // bytes per pixel: split 64-ch = [hi 64 | lo 64] fp16 (fp32 mode); split
  // 128-ch = the wide pair format [hi 128 fp16 | lo 128 e4m3 x 2^11]
  constexpr bool kLo8 = kSplit && C == 128;
  constexpr int kPxB = kLo8 ? 3 * C : (kSplit ? 2 : 1) * C * (int)sizeof(T);
  __shared__ __align__(16) uint8_t stage_b[P * kPxB];
  // PDL: the first hidden layer may start its prologue (it waits for this grid's completion)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const long long npx = (long long)B * H * W;
  const long long p0 = (long long)blockIdx.x * P;
  const long long pix = p0 + threadIdx.x;
  if (pix < npx) {
    const int xw = (int)(pix % W);
    const long long t = pix / W;
    const int y = (int)(t % H);
    const long long b = t / H;
    const float* img = x + b * (long long)H * W;
    const float sc = image_scale(escale, (int)b);  // exact 2^-e_b (1 for in-range inputs)
    float in[9];
#pragma unroll
    for (int ky = 0; ky < 3; ++ky)
#pragma unroll
      for (int kx = 0; kx < 3; ++kx) {
        const int yy = y + ky - 1, xx = xw + kx - 1;
        in[ky * 3 + kx] = (yy >= 0 && yy < H && xx >= 0 && xx < W) ? __ldg(img + (long long)yy * W + xx) : 0.0f;
      }
    T* dst = reinterpret_cast<T*>(stage_b + threadIdx.x * kPxB);
#pragma unroll
    for (int c8 = 0; c8 < C / 8; ++c8) {
      float v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int co = c8 * 8 + e;
        // fp32 accumulation of the 9 taps (a few ulps, the reference's own
        // fp32 conv class) for the split formats: fp64 cost the fp32 mode
        // 700 us per config-2 forward; the CUDA-core fp32 path keeps fp64
        using Acc = std::conditional_t<std::is_same_v<T, float>, double, float>;
        Acc acc = 0;
#pragma unroll
        for (int t9 = 0; t9 < 9; ++t9) acc = fma((Acc)p.w[co * 9 + t9], (Acc)in[t9], acc);
        v[e] = fmaxf((float)(acc + (Acc)p.b[co]), 0.0f) * sc;
      }
      if constexpr (kLo8) {
        uint32_t lo8[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float l0 = (v[2 * e] - __half2float(__float2half_rn(v[2 * e]))) * (float)(1 << 11);
          const float l1 = (v[2 * e + 1] - __half2float(__float2half_rn(v[2 * e + 1]))) * (float)(1 << 11);
          lo8[e] = __nv_cvt_float2_to_fp8x2(make_float2(l0, l1), __NV_SATFINITE, __NV_E4M3);
        }
        store_act8<T>(dst + c8 * 8, v);
        *reinterpret_cast<uint2*>(stage_b + threadIdx.x * kPxB + 2 * C + c8 * 8) =
            make_uint2(lo8[0] | (lo8[1] << 16), lo8[2] | (lo8[3] << 16));
      } else if constexpr (kSplit) {
        float lo[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) lo[e] = v[e] - __half2float(__float2half_rn(v[e]));
        store_act8<T>(dst + c8 * 8, v);
        store_act8<T>(dst + C + c8 * 8, lo);
      } else {
        store_act8<T>(dst + c8 * 8, v);
      }
    }
  }
  __syncthreads();
  // coalesced copy of the staged block (valid pixels only)
  const long long nvalid = min((long long)P, npx - p0);
  const int n16 = (int)(nvalid * kPxB / 16);
  const uint4* src = reinterpret_cast<const uint4*>(stage_b);
  uint4* out = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(act) + p0 * kPxB);
  for (int i = threadIdx.x; i < n16; i += blockDim.x) out[i] = src[i];
}

// ------------------------------------------------------------------ K3 ----
template <typename T>
__device__ __forceinline__ void load_act8(const T* src, float* v);
template <>
__device__ __forceinline__ void load_act8<__half>(const __half* src, float* v) {
  const uint4 u = __ldg(reinterpret_cast<const uint4*>(src));
  const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) { float2 f = __half22float2(h[i]); v[2 * i] = f.x; v[2 * i + 1] = f.y; }
}
template <>
__device__ __forceinline__ void load_act8<float>(const float* src, float* v) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(src));
  const float4 b = __ldg(reinterpret_cast<const float4*>(src) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// wh: [K][64][3][3] fp32 ; output rows [row0, row0+rows) of each image go to
// bands[b][k][r-row0][x] and closure[b][0][r-row0][x].
template <typename T, int C>
__global__ void __launch_bounds__(128)
head_kernel(const T* __restrict__ act, const float* __restrict__ x, const float* __restrict__ wh,
            const float* __restrict__ bh, float* __restrict__ bands, float* __restrict__ closure,
            double* __restrict__ recon, int B, int H, int W, int K, int row0, int rows, int* __restrict__ status) {
  extern __shared__ float swh[];  // [9][64][K]
  for (int i = threadIdx.x; i < 9 * C * K; i += blockDim.x) {
    const int k = i % K, ci = (i / K) % C, t = i / (K * C);
    swh[i] = wh[(k * C + ci) * 9 + t];
  }
  __syncthreads();
  const long long nout = (long long)B * rows * W;
  const long long p0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = p0 < nout;
  if (!live && !recon) return;
  const long long p = live ? p0 : nout - 1;  // dead lanes of the last warp only feed zeros to recon
  const int xw = (int)(p % W);
  const long long t = p / W;
  const int rr = (int)(t % rows);
  const long long b = t / rows;
  const int y = row0 + rr;
  using Acc = std::conditional_t<std::is_same_v<T, float>, double, float>;  // fp64 in fp32 mode
  Acc acc[kMaxBands];
#pragma unroll
  for (int k = 0; k < kMaxBands; ++k) acc[k] = 0;
  const T* base = act + b * (long long)H * W * C;
  for (int ky = 0; ky < 3; ++ky) {
    const int yy = y + ky - 1;
    if (yy < 0 || yy >= H) continue;
    for (int kx = 0; kx < 3; ++kx) {
      const int xx = xw + kx - 1;
      if (xx < 0 || xx >= W) continue;
      const T* src = base + ((long long)yy * W + xx) * C;
      const float* wt = swh + (ky * 3 + kx) * C * K;
#pragma unroll 2
      for (int c8 = 0; c8 < C / 8; ++c8) {
        float v[8];
        load_act8<T>(src + c8 * 8, v);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float* wr = wt + (c8 * 8 + e) * K;
#pragma unroll
          for (int k = 0; k < kMaxBands; ++k)
            if (k < K) acc[k] = fma((Acc)wr[k], (Acc)v[e], acc[k]);
        }
      }
    }
  }
  float sum = 0.0f;
  const long long plane = (long long)rows * W;
  float* ob = bands + b * K * plane + (long long)rr * W + xw;
  bool bad = false;
#pragma unroll
  for (int k = 0; k < kMaxBands; ++k)
    if (k < K) {
      const float o = (float)(acc[k] + (Acc)bh[k]);
      if (live) ob[k * plane] = o;
      sum += o;
      bad |= !isfinite(o);
    }
  if (bad && status) flag_set(status + kStatNonFiniteOut);
  const float xv = x[(b * H + y) * (long long)W + xw];
  const float c = xv - sum;
  if (closure != nullptr && live) closure[b * plane + (long long)rr * W + xw] = c;
  if (recon) {
    // warps of this kernel straddle images when rows*W % 32 != 0: one atomic
    // pair per lane-image run would need segmented reduction, so use per-lane
    // atomics there (the CUDA-core fp32 path is the slow reference path)
    const float r = live ? xv - (sum + c) : 0.0f, xx = live ? xv : 0.0f;
    const long long b0 = __shfl_sync(0xffffffffu, b, 0);
    if (__all_sync(0xffffffffu, b == b0)) {
      recon_accumulate(recon, (int)b0, r, xx);
    } else if (live) {
      atomicAdd(recon + 2 * b, (double)r * r);
      atomicAdd(recon + 2 * b + 1, (double)xx * xx);
    }
  }
}

// --------------------------------------------------- fp32 hidden layer ----
// Output tile 4 rows x 32 px x 64 co per 256-thread block; thread = (co
// group of 8, px column); input channels streamed in chunks of 16.
template <int C>
__global__ void __launch_bounds__(32 * (C / 8))
hidden_f32_kernel(const float* __restrict__ in, float* __restrict__ out, const float* __restrict__ w /*[co][ci][9]*/,
                  const float* __restrict__ scale, const float* __restrict__ shift, int B, int H, int W) {
  extern __shared__ float sm[];
  float* sIn = sm;                                        // [rows][px][ci]
  float* sWt = sm + kF32InRows * kF32InPx * kF32CiChunk;  // [ci][tap][co]
  const int tx = threadIdx.x & 31;  // px column
  const int g = threadIdx.x >> 5;   // co group (8 channels)
  const int tiles_x = (W + kF32TilePx - 1) / kF32TilePx;
  const int tiles_y = (H + kF32TileRows - 1) / kF32TileRows;
  const int tile = blockIdx.x;
  const int b = tile / (tiles_x * tiles_y);
  const int ty0 = ((tile / tiles_x) % tiles_y) * kF32TileRows;
  const int tx0 = (tile % tiles_x) * kF32TilePx;
  // fp32 FFMA partial sums over one 16-input-channel chunk (144 terms), added
  // into fp64 accumulators per chunk: each output is then within the fp32
  // reference's own rounding of the exact value (tools/emulate_fp32_accum.py:
  // 5.1e-6 vs 4.9e-6 for full fp64 on config 1), at FFMA speed.
  double acc[kF32TileRows][8];
#pragma unroll
  for (int r = 0; r < kF32TileRows; ++r)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[r][e] = 0.0;
  const float* ib = in + (long long)b * H * W * C;
  for (int c0 = 0; c0 < C; c0 += kF32CiChunk) {
    __syncthreads();
    for (int i = threadIdx.x; i < kF32InRows * kF32InPx * kF32CiChunk; i += blockDim.x) {
      const int ci = i % kF32CiChunk, px = (i / kF32CiChunk) % kF32InPx, r = i / (kF32CiChunk * kF32InPx);
      const int yy = ty0 + r - 1, xx = tx0 + px - 1;
      sIn[i] = (yy >= 0 && yy < H && xx >= 0 && xx < W) ? ib[((long long)yy * W + xx) * C + c0 + ci] : 0.0f;
    }
    for (int i = threadIdx.x; i < kF32CiChunk * 9 * C; i += blockDim.x) {
      const int co = i % C, t = (i / C) % 9, ci = i / (C * 9);
      sWt[i] = w[((long long)co * C + c0 + ci) * 9 + t];
    }
    __syncthreads();
    float part[kF32TileRows][8];
#pragma unroll
    for (int r = 0; r < kF32TileRows; ++r)
#pragma unroll
      for (int e = 0; e < 8; ++e) part[r][e] = 0.0f;
#pragma unroll 2
    for (int ci = 0; ci < kF32CiChunk; ++ci) {
#pragma unroll
      for (int ky = 0; ky < 3; ++ky)
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
          const float4 w0 = *reinterpret_cast<const float4*>(sWt + (ci * 9 + ky * 3 + kx) * C + g * 8);
          const float4 w1 = *reinterpret_cast<const float4*>(sWt + (ci * 9 + ky * 3 + kx) * C + g * 8 + 4);
          const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
          for (int r = 0; r < kF32TileRows; ++r) {
            const float av = sIn[((r + ky) * kF32InPx + tx + kx) * kF32CiChunk + ci];
#pragma unroll
            for (int e = 0; e < 8; ++e) part[r][e] = fmaf(wv[e], av, part[r][e]);
          }
        }
    }
#pragma unroll
    for (int r = 0; r < kF32TileRows; ++r)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[r][e] += (double)part[r][e];
  }
  const int xw = tx0 + tx;
  if (xw >= W) return;
#pragma unroll
  for (int r = 0; r < kF32TileRows; ++r) {
    const int y = ty0 + r;
    if (y >= H) break;
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e)
      v[e] = fmaxf((float)fma(acc[r][e], (double)scale[g * 8 + e], (double)shift[g * 8 + e]), 0.0f);
    float* dst = out + (((long long)b * H + y) * W + xw) * C + g * 8;
    reinterpret_cast<float4*>(dst)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(dst)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
}

cudaError_t launch_conv0(int act_fmt, int C, const float* x, void* act, const Conv0Params& p, const int* escale,
                         int B, int H, int W, cudaStream_t st) {
  const long long npx = (long long)B * H * W;
  if (C == 64) {
    const unsigned grid = (unsigned)((npx + 127) / 128);
    if (act_fmt == kActF16)
      conv0_kernel<__half, 64><<<grid, 128, 0, st>>>(x, static_cast<__half*>(act), p, escale, B, H, W);
    else if (act_fmt == kActSplit)
      conv0_kernel<__half, 64, true><<<grid, 128, 0, st>>>(x, static_cast<__half*>(act), p, escale, B, H, W);
    else
      conv0_kernel<float, 64><<<grid, 128, 0, st>>>(x, static_cast<float*>(act), p, escale, B, H, W);
  } else if (C == 128 && act_fmt == kActF32) {
    const unsigned grid = (unsigned)((npx + 63) / 64);
    conv0_kernel<float, 128><<<grid, 64, 0, st>>>(x, static_cast<float*>(act), p, escale, B, H, W);
  } else if (C == 128 && act_fmt == kActF16) {
    const unsigned grid = (unsigned)((npx + 63) / 64);
    conv0_kernel<__half, 128><<<grid, 64, 0, st>>>(x, static_cast<__half*>(act), p, escale, B, H, W);
  } else if (C == 128 && act_fmt == kActSplit) {
    const unsigned grid = (unsigned)((npx + 63) / 64);
    conv0_kernel<__half, 128, true><<<grid, 64, 0, st>>>(x, static_cast<__half*>(act), p, escale, B, H, W);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}


// ------------------------------------------------- K1, unshuffle = 2 ----
// Conv2d(4, 64, 3, p=1) + ReLU over pixel_unshuffle(x, 2), computed straight
// from the full-resolution plane: input channel c = 2i + j of half-res pixel
// (Y, X) is x[2Y + i][2X + j] (torch pixel_unshuffle order), zero outside the
// half-res grid.  One thread per half-res pixel, weights (64 x 36) staged in
// shared memory, output staged and written coalesced as fp16 NHWC.
__global__ void __launch_bounds__(128)
conv0_unshuffle_kernel(const float* __restrict__ x, __half* __restrict__ act, const float* __restrict__ w,
                       const float* __restrict__ bias, const int* __restrict__ escale, int B, int H, int W) {
  constexpr int P = 128, C = 64;
  __shared__ float sw[C * 36];
  __shared__ float sb[C];
  __shared__ __align__(16) __half stage[P * C];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int i = threadIdx.x; i < C * 36; i += blockDim.x) sw[i] = w[i];
  if (threadIdx.x < C) sb[threadIdx.x] = bias[threadIdx.x];
  __syncthreads();
  const long long npx = (long long)B * H * W;
  const long long p0 = (long long)blockIdx.x * P;
  const long long pix = p0 + threadIdx.x;
  if (pix < npx) {
    const int X = (int)(pix % W);
    const long long t = pix / W;
    const int Y = (int)(t % H);
    const long long b = t / H;
    const int Wf = 2 * W;
    const float* img = x + b * (long long)(2 * H) * Wf;
    const float sc = image_scale(escale, (int)b);
    float in[36];  // [c = 2i + j][ky][kx]
#pragma unroll
    for (int ky = 0; ky < 3; ++ky)
#pragma unroll
      for (int kx = 0; kx < 3; ++kx) {
        const int yy = Y + ky - 1, xx = X + kx - 1;
        const bool ok = yy >= 0 && yy < H && xx >= 0 && xx < W;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          in[c * 9 + ky * 3 + kx] = ok ? __ldg(img + (long long)(2 * yy + (c >> 1)) * Wf + 2 * xx + (c & 1)) : 0.0f;
      }
    __half* dst = stage + threadIdx.x * C;
#pragma unroll
    for (int c8 = 0; c8 < C / 8; ++c8) {
      float v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int co = c8 * 8 + e;
        float acc = 0.0f;
#pragma unroll
        for (int t36 = 0; t36 < 36; ++t36) acc = fmaf(sw[co * 36 + t36], in[t36], acc);
        v[e] = fmaxf(acc + sb[co], 0.0f) * sc;
      }
      store_act8<__half>(dst + c8 * 8, v);
    }
  }
  __syncthreads();
  const long long nvalid = min((long long)P, npx - p0);
  const int n16 = (int)(nvalid * C * 2 / 16);
  const uint4* src = reinterpret_cast<const uint4*>(stage);
  uint4* out = reinterpret_cast<uint4*>(act + p0 * C);
  for (int i = threadIdx.x; i < n16; i += blockDim.x) out[i] = src[i];
}

cudaError_t launch_conv0_unshuffle(const float* x, void* act, const float* w, const float* b, const int* escale, int B,
                                   int H, int W, cudaStream_t st) {
  const long long npx = (long long)B * H * W;
  conv0_unshuffle_kernel<<<(unsigned)((npx + 127) / 128), 128, 0, st>>>(x, static_cast<__half*>(act), w, b, escale,
                                                                        B, H, W);
  return cudaGetLastError();
}

cudaError_t launch_head_f32(int C, const float* act, const float* x, const float* wh, const float* bh, float* bands,
                            double* recon,
                            float* closure, int B, int H, int W, int K, int row0, int rows, int* status,
                            cudaStream_t st) {
  const long long nout = (long long)B * rows * W;
  const unsigned grid = (unsigned)((nout + 127) / 128);
  const size_t smem = (size_t)9 * C * K * sizeof(float);
  if (C == 64)
    head_kernel<float, 64><<<grid, 128, smem, st>>>(act, x, wh, bh, bands, closure, recon, B, H, W, K, row0, rows, status);
  else if (C == 128)
    head_kernel<float, 128><<<grid, 128, smem, st>>>(act, x, wh, bh, bands, closure, recon, B, H, W, K, row0, rows, status);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_hidden_f32(int C, const float* in, float* out, const float* w, const float* scale,
                              const float* shift, int B, int H, int W, cudaStream_t st) {
  const long long tiles = (long long)B * ((H + kF32TileRows - 1) / kF32TileRows) * ((W + kF32TilePx - 1) / kF32TilePx);
  if (C == 64)
    hidden_f32_kernel<64><<<(unsigned)tiles, 256, f32_smem(64), st>>>(in, out, w, scale, shift, B, H, W);
  else if (C == 128)
    hidden_f32_kernel<128><<<(unsigned)tiles, 512, f32_smem(128), st>>>(in, out, w, scale, shift, B, H, W);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

// ------------------------------------------------ per-image input scale ----
// Grid (chunks, B): each block reduces one chunk of image b to amax and a
// non-finite flag, merges them with atomics (amax as order-preserving bits of
// a non-negative float), and the image's last block turns them into e_b.  The
// exponent keeps the conv0 output bound M = amax * w0_l1 + b0_max (and with it
// every fp16 activation of a well-conditioned network) near 1: inputs whose M
// lies in [2^-6, 2^6] (every BASELINE workload) keep e = 0, so their
// arithmetic is unchanged and bitwise identical across batch/row-band shards.
// scratch: 2 * B zeroed ints per forward ([0, B) amax bits, [B, 2B) block count).
__global__ void __launch_bounds__(256)
input_scale_kernel(const float* __restrict__ x, long long n, float w0_l1, float b0_max, int* __restrict__ escale,
                   int* __restrict__ scratch, int* __restrict__ status, int vec4) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // conv0 may start its prologue
  const int b = blockIdx.y, B = gridDim.y;
  const float* img = x + (long long)b * n;
  const long long per = ((n + gridDim.x - 1) / gridDim.x + 3) & ~3LL;  // a multiple of 4 px
  const long long lo = min(n, per * blockIdx.x), hi = min(n, lo + per);
  float amax = 0.0f;
  int bad = 0;
  // max and the non-finite flag are order-independent, so the vector path
  // (block ranges are multiples of 4 px; taken when the image is 16 B aligned)
  // gives the same bits: independent 16 B loads instead of a chain of 4 B ones
  if (vec4) {
    const float4* img4 = reinterpret_cast<const float4*>(img);
    for (long long i = lo / 4 + threadIdx.x; i < hi / 4; i += blockDim.x) {
      const float4 e = __ldg(img4 + i);
      const float m4 = fmaxf(fmaxf(fabsf(e.x), fabsf(e.y)), fmaxf(fabsf(e.z), fabsf(e.w)));
      if (isfinite(e.x) && isfinite(e.y) && isfinite(e.z) && isfinite(e.w)) {
        amax = fmaxf(amax, m4);
      } else {
        bad = 1;
        if (isfinite(e.x)) amax = fmaxf(amax, fabsf(e.x));
        if (isfinite(e.y)) amax = fmaxf(amax, fabsf(e.y));
        if (isfinite(e.z)) amax = fmaxf(amax, fabsf(e.z));
        if (isfinite(e.w)) amax = fmaxf(amax, fabsf(e.w));
      }
    }
  } else {
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      const float e = __ldg(img + i);
      if (isfinite(e)) amax = fmaxf(amax, fabsf(e));
      else bad = 1;
    }
  }
  __shared__ float s_max[8];
  __shared__ int s_bad[8];
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) { s_max[threadIdx.x >> 5] = amax; s_bad[threadIdx.x >> 5] = bad; }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int w = 1; w < 8; ++w) { amax = fmaxf(amax, s_max[w]); bad |= s_bad[w]; }
  if (bad && status) flag_set(status + kStatNonFiniteIn);
  atomicMax(scratch + b, __float_as_int(amax));
  __threadfence();
  if (atomicAdd(scratch + B + b, 1) != (int)gridDim.x - 1) return;
  __threadfence();
  const float m = fmaf(__int_as_float(atomicExch(scratch + b, 0)), w0_l1, b0_max);
  scratch[B + b] = 0;  // re-armed for the next forward (stream order)
  int e = 0;
  if (m > 0.0f && (m < 0.015625f || m > 64.0f)) e = min(60, max(-60, ilogbf(m) - 1));
  escale[b] = e;
}

cudaError_t launch_input_scale(const float* x, int B, long long px_per_image, float w0_l1, float b0_max, int* escale,
                               int* scratch, int* status, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  // ~4 blocks per SM in total, >= 1024 px per block (one 16 B load per thread:
  // a batch-1 256 x 256 image took 8 us with 16 dependent 4 B loads per thread)
  const long long want = std::max(1LL, std::min((592LL + B - 1) / B, (px_per_image + 1023) / 1024));
  const int vec4 = (px_per_image % 4 == 0) && (reinterpret_cast<uintptr_t>(x) % 16 == 0);
  input_scale_kernel<<<dim3((unsigned)want, (unsigned)B), 256, 0, st>>>(x, px_per_image, w0_l1, b0_max, escale,
                                                                          scratch, status, vec4);
  return cudaGetLastError();
}

cudaError_t configure_edge_kernels() {
  cudaError_t e = cudaFuncSetAttribute(hidden_f32_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)f32_smem(64));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(hidden_f32_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f32_smem(128));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(head_kernel<float, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              9 * 128 * kMaxBands * 4);
}

}  // namespace tvs
