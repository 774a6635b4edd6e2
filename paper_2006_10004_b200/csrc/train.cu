// train.cu — one TVSpecNET training step on B200:
// the train-mode forward (batch-statistics BatchNorm) and the backward of
// /root/reference/pkg/trainer/src/tvsurrogate/model.py:29-52 as called by
// training.py:45-61 (_epoch_pass: model(img) -> compute_loss -> backward).
//
// Numerics.  The gradients of a 17-layer BN network at its
// Kaiming init are ill-conditioned: the reference's own fp32 gradients sit
// 3e-3 from fp64, and an fp16 forward (activations or weights rounded to
// fp16) moves them by ~20% (tools/emulate_train.py).  Rounding the BACKWARD
// operands to fp16 does not.  So:
//   * forward convs are fp32-accurate: the split hi/lo fp16 tcgen05 kernel of
//     the fp32 inference mode (conv_tc.cu mode 3, raw fp32 output), batch
//     statistics in fp64;
//   * dgrad convs run the fp16 tcgen05 hidden kernel (mode 0, raw fp32
//     output) on per-layer power-of-two-scaled fp16 gradients and the
//     transposed, flipped fp16 filters;
//   * wgrad is a GEMM over pixels on zero-bordered fp16 buffers (see Layout):
//     one tcgen05 launch per layer with MN-major operands (wgrad_tc.cu); the
//     first version, one cuBLAS split-K GEMM per tap, stays behind the train
//     option wgrad_tc = 0 as the A/B reference;
//   * the head's input gradient runs on the same tcgen05 dgrad kernel (bands
//     as channels 0..K-1 of the 64-channel gradient operand);
//   * conv0 backward and BatchNorm backward: CUDA cores, fp32/fp64.
//
// Layout.  Activations a_j (j = 0..depth-2) are stored as fp16 hi/lo pairs
// [B][H+2][W+2][128] with a zero border and `guard` zero pixels before and
// after: the split conv reads them through a tensor map on the interior, and
// the wgrad GEMM reads the hi half shifted by a tap offset
// (ky-1)*(W+2) + (kx-1) pixels: for every interior pixel q the shifted pixel
// stays inside q's own image (border -> the zero padding), and border pixels
// q carry a zero gradient, so one GEMM over all B*(H+2)*(W+2) pixels is the
// exact tap sum.  Pre-BN conv outputs y_j are fp32 [B][H][W][64].
#include <cublas_v2.h>
#include <cuda.h>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "host_util.h"

namespace tvs {

constexpr int kTB = 256;  // threads per elementwise block

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// conv0 + ReLU (model.py:37-38) in fp32 -> pair a_0
// (padded).  One thread per pixel, weights from global (uniform loads).
__global__ void __launch_bounds__(kTB)
train_conv0_kernel(const float* __restrict__ x, const float* __restrict__ w, const float* __restrict__ b, int B, int H,
                   int W, __half* __restrict__ apad) {
  const long long P = (long long)B * H * W;
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const int xw = (int)(p % W);
  const long long t = p / W;
  const int y = (int)(t % H), bi = (int)(t / H);
  const float* img = x + (long long)bi * H * W;
  float in[9];
#pragma unroll
  for (int ky = 0; ky < 3; ++ky)
#pragma unroll
    for (int kx = 0; kx < 3; ++kx) {
      const int yy = y + ky - 1, xx = xw + kx - 1;
      in[ky * 3 + kx] = (yy >= 0 && yy < H && xx >= 0 && xx < W) ? __ldg(img + (long long)yy * W + xx) : 0.0f;
    }
  __half* dst = apad + (((long long)bi * (H + 2) + y + 1) * (W + 2) + xw + 1) * 128;
#pragma unroll
  for (int c8 = 0; c8 < 8; ++c8) {
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float f[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int co = c8 * 8 + e * 2 + u;
        // fp32 accumulation over the 9 taps (the reference's own precision class, as the
        // fp32 inference mode's conv0; fp64 FMAs made this kernel 238 us at 64 x 128^2)
        float acc = 0.0f;
#pragma unroll
        for (int k = 0; k < 9; ++k) acc = fmaf(__ldg(w + co * 9 + k), in[k], acc);
        f[u] = fmaxf(acc + __ldg(b + co), 0.0f);
      }
      const __half2 hh = __floats2half2_rn(f[0], f[1]);
      const float2 hf = __half22float2(hh);
      const __half2 ll = __floats2half2_rn(f[0] - hf.x, f[1] - hf.y);
      hi[e] = *reinterpret_cast<const uint32_t*>(&hh);
      lo[e] = *reinterpret_cast<const uint32_t*>(&ll);
    }
    *reinterpret_cast<uint4*>(dst + c8 * 8) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4*>(dst + 64 + c8 * 8) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  }
}

// Batch statistics of y [P][64] fp32: sums[c] += y, sums[64 + c] += y^2 (fp64).
// Thread t of a block owns channels 4*(t % 16) .. +3 (one 16 B load per pixel)
// and pixel lane t / 16; four pixels are in flight per thread (independent
// loads: the first version walked one pixel at a time and was latency-bound,
// 19.5 us for 8 x 128 x 128 against 5 us of HBM time).
constexpr int kRedPx = kTB / 16;  // pixels per block per step
__global__ void __launch_bounds__(kTB) bn_stats_kernel(const float* __restrict__ y, long long P, double* sums) {
  const int c4 = threadIdx.x & 15, lane = threadIdx.x >> 4;
  double s1[4] = {0, 0, 0, 0}, s2[4] = {0, 0, 0, 0};
  const long long step = (long long)gridDim.x * kRedPx;
  auto add = [&](const float4& q) {
    const float e[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double d = e[k];
      s1[k] += d;
      s2[k] += d * d;
    }
  };
  long long p0 = (long long)blockIdx.x * kRedPx + lane;
  for (; p0 + 7 * step < P; p0 += 8 * step) {  // eight unpredicated loads in flight
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(y + (p0 + u * step) * 64) + c4);
#pragma unroll
    for (int u = 0; u < 8; ++u) add(v[u]);
  }
  for (; p0 < P; p0 += step) add(__ldg(reinterpret_cast<const float4*>(y + p0 * 64) + c4));
  __shared__ double sh[2][kRedPx][64];
#pragma unroll
  for (int k = 0; k < 4; ++k) { sh[0][lane][c4 * 4 + k] = s1[k]; sh[1][lane][c4 * 4 + k] = s2[k]; }
  __syncthreads();
  if (threadIdx.x < 128) {
    const int which = threadIdx.x >> 6, c = threadIdx.x & 63;
    double t = 0.0;
    for (int l = 0; l < kRedPx; ++l) t += sh[which][l][c];
    atomicAdd(sums + which * 64 + c, t);
  }
}

// per-channel mean / 1/sqrt(var + eps) from the sums (biased variance, the
// normalisation BatchNorm2d uses in train mode)
__device__ __forceinline__ void bn_moments(const double* sums, int c, double n, float eps, float& mean, float& rstd) {
  const double m = sums[c] / n;
  const double v = fmax(sums[64 + c] / n - m * m, 0.0);
  mean = (float)m;
  rstd = (float)(1.0 / sqrt(v + (double)eps));
}

// a = ReLU(gamma * (y - mean) * rstd + beta) -> pair a_j (padded); block 0
// also exports the batch mean and the unbiased variance (running-stat update,
// done by the caller with BatchNorm2d's momentum).
__global__ void __launch_bounds__(kTB)
bn_apply_kernel(const float* __restrict__ y, int B, int H, int W, const double* __restrict__ sums,
                const float* __restrict__ gamma, const float* __restrict__ beta, float eps, __half* __restrict__ apad,
                float* __restrict__ mean_out, float* __restrict__ var_out) {
  __shared__ float s_a[64], s_b[64];
  const double n = (double)B * H * W;
  if (threadIdx.x < 64) {
    const int c = threadIdx.x;
    float mean, rstd;
    bn_moments(sums, c, n, eps, mean, rstd);
    const float g = __ldg(gamma + c);
    s_a[c] = g * rstd;
    s_b[c] = __ldg(beta + c) - mean * g * rstd;
    if (blockIdx.x == 0) {
      mean_out[c] = mean;
      const double m = sums[c] / n;
      const double v = fmax(sums[64 + c] / n - m * m, 0.0);
      var_out[c] = (float)(n > 1.0 ? v * n / (n - 1.0) : v);
    }
  }
  __syncthreads();
  const long long P = (long long)B * H * W;
  // thread = (pixel, 8-channel chunk)
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < P * 8; i += (long long)gridDim.x * blockDim.x) {
    const long long p = i >> 3;
    const int c8 = (int)(i & 7);
    const float4 v0 = __ldg(reinterpret_cast<const float4*>(y + p * 64 + c8 * 8));
    const float4 v1 = __ldg(reinterpret_cast<const float4*>(y + p * 64 + c8 * 8 + 4));
    const float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float f[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int c = c8 * 8 + e * 2 + u;
        f[u] = fmaxf(fmaf(s_a[c], v[e * 2 + u], s_b[c]), 0.0f);
      }
      const __half2 hh = __floats2half2_rn(f[0], f[1]);
      const float2 hf = __half22float2(hh);
      const __half2 ll = __floats2half2_rn(f[0] - hf.x, f[1] - hf.y);
      hi[e] = *reinterpret_cast<const uint32_t*>(&hh);
      lo[e] = *reinterpret_cast<const uint32_t*>(&ll);
    }
    const int xw = (int)(p % W);
    const long long t = p / W;
    const int yy = (int)(t % H), bi = (int)(t / H);
    __half* dst = apad + (((long long)bi * (H + 2) + yy + 1) * (W + 2) + xw + 1) * 128;
    *reinterpret_cast<uint4*>(dst + c8 * 8) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4*>(dst + 64 + c8 * 8) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  }
}

// BatchNorm backward, pass 1 (torch's batch_norm backward, train mode):
// g_z = g_a * [z > 0] with z = gamma*yhat + beta recomputed exactly as the
// forward did; S1[c] = sum g_z, S2[c] = sum g_z * yhat (fp64), and the
// amax of |g_z| and |yhat| (as float bits) for the fp16 scale of pass 2.
__device__ __forceinline__ void
bn_bwd_reduce_body(const float* __restrict__ ga, const float* __restrict__ y, long long P, const double* sums,
                   const float* __restrict__ gamma, const float* __restrict__ beta, float eps, double* red,
                   int* amax_bits) {
  // thread = (4 channels, pixel lane), four pixels in flight (see bn_stats_kernel)
  const int c4 = threadIdx.x & 15, lane = threadIdx.x >> 4;
  float mean[4], rstd[4], sa[4], sb[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int c = c4 * 4 + k;
    bn_moments(sums, c, (double)P, eps, mean[k], rstd[k]);
    const float g = __ldg(gamma + c), bb = __ldg(beta + c);
    sa[k] = g * rstd[k];
    sb[k] = bb - mean[k] * g * rstd[k];
  }
  double s1[4] = {0, 0, 0, 0}, s2[4] = {0, 0, 0, 0};
  float mz = 0.0f, mh = 0.0f;
  const long long step = (long long)gridDim.x * kRedPx;
  for (long long p0 = (long long)blockIdx.x * kRedPx + lane; p0 < P; p0 += 4 * step) {
    float4 vy[4], vg[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long p = p0 + u * step;
      const bool ok = p < P;
      vy[u] = ok ? __ldg(reinterpret_cast<const float4*>(y + p * 64) + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
      vg[u] = ok ? __ldg(reinterpret_cast<const float4*>(ga + p * 64) + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (p0 + u * step >= P) continue;
      const float ev[4] = {vy[u].x, vy[u].y, vy[u].z, vy[u].w};
      const float eg[4] = {vg[u].x, vg[u].y, vg[u].z, vg[u].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float z = fmaf(sa[k], ev[k], sb[k]);
        const float gz = z > 0.0f ? eg[k] : 0.0f;
        const float yh = (ev[k] - mean[k]) * rstd[k];
        s1[k] += gz;
        s2[k] += (double)gz * yh;
        mz = fmaxf(mz, fabsf(gz));
        mh = fmaxf(mh, fabsf(yh));
      }
    }
  }
  __shared__ double sh[2][kRedPx][64];
#pragma unroll
  for (int k = 0; k < 4; ++k) { sh[0][lane][c4 * 4 + k] = s1[k]; sh[1][lane][c4 * 4 + k] = s2[k]; }
  mz = warp_max(mz);
  mh = warp_max(mh);
  __syncthreads();
  if (threadIdx.x < 128) {
    const int which = threadIdx.x >> 6, c = threadIdx.x & 63;
    double t = 0.0;
    for (int l = 0; l < kRedPx; ++l) t += sh[which][l][c];
    atomicAdd(red + which * 64 + c, t);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(amax_bits, __float_as_int(mz));
    atomicMax(amax_bits + 1, __float_as_int(mh));
  }
}

// Pass 2: g_y = gamma*rstd*(g_z - S1/N - yhat*S2/N), stored as fp16 times 2^s
// into the zero-bordered gradient buffer [B][H+2][W+2][64]; s puts a bound of
// |g_y| near 2^10 (no overflow in the dgrad conv's fp16 operand, full fp16
// precision).  Block 0 exports dgamma = S2, dbeta = S1, s and 2^-s.
__device__ __forceinline__ void
bn_bwd_apply_body(const float* __restrict__ ga, const float* __restrict__ y, int B, int H, int W,
                  const double* sums, const float* __restrict__ gamma, const float* __restrict__ beta, float eps,
                  const double* red, const int* amax_bits, __half* __restrict__ gpad, int* gexp, float* ginv,
                  float* dgamma, float* dbeta) {
  __shared__ __align__(16) float s_sa[64], s_sb[64], s_k[64], s_m1[64], s_m2[64], s_mean[64], s_rstd[64];
  __shared__ float s_scale;
  const double n = (double)B * H * W;
  if (threadIdx.x < 64) {
    const int c = threadIdx.x;
    float mean, rstd;
    bn_moments(sums, c, n, eps, mean, rstd);
    const float g = __ldg(gamma + c);
    s_sa[c] = g * rstd;
    s_sb[c] = __ldg(beta + c) - mean * g * rstd;
    s_k[c] = g * rstd;
    s_mean[c] = mean;
    s_rstd[c] = rstd;
    s_m1[c] = (float)(red[c] / n);
    s_m2[c] = (float)(red[64 + c] / n);
    if (blockIdx.x == 0) {
      dgamma[c] = (float)red[64 + c];
      dbeta[c] = (float)red[c];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const float mz = __int_as_float(amax_bits[0]), mh = __int_as_float(amax_bits[1]);
    float bound = 0.0f;
    for (int c = 0; c < 64; ++c)
      bound = fmaxf(bound, fabsf(s_k[c]) * (mz + fabsf(s_m1[c]) + mh * fabsf(s_m2[c])));
    const int e = bound > 0.0f ? min(100, max(-100, 10 - (ilogbf(bound) + 1))) : 0;
    s_scale = pow2i(e);
    if (blockIdx.x == 0) {
      *gexp = e;
      *ginv = pow2i(-e);
    }
  }
  __syncthreads();
  const float sc = s_scale;
  const long long P = (long long)B * H * W;
  // thread = (pixel, 4 channels), as bn_apply_kernel; the channel constants stay in registers
  const int c4 = threadIdx.x & 15;
  float csa[4], csb[4], ck[4], cm1[4], cm2[4], cmean[4], crstd[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int c = c4 * 4 + k;
    csa[k] = s_sa[c]; csb[k] = s_sb[c]; ck[k] = s_k[c]; cm1[k] = s_m1[c];
    cm2[k] = s_m2[c]; cmean[k] = s_mean[c]; crstd[k] = s_rstd[c];
  }
  for (long long p = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 4; p < P;
       p += ((long long)gridDim.x * blockDim.x) >> 4) {
    const float4 y4 = __ldg(reinterpret_cast<const float4*>(y + p * 64) + c4);
    const float4 g4 = __ldg(reinterpret_cast<const float4*>(ga + p * 64) + c4);
    const float yv[4] = {y4.x, y4.y, y4.z, y4.w};
    const float gv[4] = {g4.x, g4.y, g4.z, g4.w};
    float f[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float v = yv[k];
      const float z = fmaf(csa[k], v, csb[k]);
      const float gz = z > 0.0f ? gv[k] : 0.0f;
      const float yh = (v - cmean[k]) * crstd[k];
      f[k] = ck[k] * (gz - cm1[k] - yh * cm2[k]) * sc;
    }
    const __half2 h01 = __floats2half2_rn(f[0], f[1]), h23 = __floats2half2_rn(f[2], f[3]);
    const int xw = (int)(p % W);
    const long long t = p / W;
    const int yy = (int)(t % H), bi = (int)(t / H);
    __half* dst = gpad + (((long long)bi * (H + 2) + yy + 1) * (W + 2) + xw + 1) * 64 + c4 * 4;
    *reinterpret_cast<uint2*>(dst) =
        make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
  }
}

__global__ void __launch_bounds__(kTB)
bn_bwd_reduce_kernel(const float* __restrict__ ga, const float* __restrict__ y, long long P, const double* sums,
                     const float* __restrict__ gamma, const float* __restrict__ beta, float eps, double* red,
                     int* amax_bits) {
  bn_bwd_reduce_body(ga, y, P, sums, gamma, beta, eps, red, amax_bits);
}
__global__ void __launch_bounds__(kTB)
bn_bwd_apply_kernel(const float* __restrict__ ga, const float* __restrict__ y, int B, int H, int W,
                    const double* sums, const float* __restrict__ gamma, const float* __restrict__ beta, float eps,
                    const double* red, const int* amax_bits, __half* __restrict__ gpad, int* gexp, float* ginv,
                    float* dgamma, float* dbeta) {
  bn_bwd_apply_body(ga, y, B, H, W, sums, gamma, beta, eps, red, amax_bits, gpad, gexp, ginv, dgamma, dbeta);
}
// Both passes in one cooperative launch: the grid-wide barrier replaces the
// kernel boundary, and the second read of ga and y comes from L2 when the
// layer fits (33 MB each at 8 x 128^2).  Launched with
// cudaLaunchCooperativeKernel on a co-resident grid (tvs_train_backward).
__global__ void __launch_bounds__(kTB)
bn_bwd_fused_kernel(const float* __restrict__ ga, const float* __restrict__ y, int B, int H, int W,
                    const double* sums, const float* __restrict__ gamma, const float* __restrict__ beta, float eps,
                    double* red, int* amax_bits, __half* __restrict__ gpad, int* gexp, float* ginv, float* dgamma,
                    float* dbeta) {
  bn_bwd_reduce_body(ga, y, (long long)B * H * W, sums, gamma, beta, eps, red, amax_bits);
  __threadfence();
  cooperative_groups::this_grid().sync();
  bn_bwd_apply_body(ga, y, B, H, W, sums, gamma, beta, eps, red, amax_bits, gpad, gexp, ginv, dgamma, dbeta);
}

// Head backward, pass 1: dbias[k] = sum g_out[k] (fp64) and amax |g_out|.
__global__ void __launch_bounds__(kTB)
head_bwd_reduce_kernel(const float* __restrict__ gout, int B, int K, long long HW, double* dbias, int* amax_bits) {
  const int k = blockIdx.y;
  double s = 0.0;
  float m = 0.0f;
  for (int b = 0; b < B; ++b) {
    const float* g = gout + ((long long)b * K + k) * HW;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < HW; i += (long long)gridDim.x * blockDim.x) {
      const float v = __ldg(g + i);
      s += v;
      m = fmaxf(m, fabsf(v));
    }
  }
  __shared__ double sh[kTB];
  sh[threadIdx.x] = s;
  m = warp_max(m);
  __syncthreads();
  for (int o = kTB / 2; o; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicAdd(dbias + k, sh[0]);
  if ((threadIdx.x & 31) == 0) atomicMax(amax_bits, __float_as_int(m));
}

// Head backward, pass 2: g_out as fp16 * 2^s into [B][H+2][W+2][cs] (bands
// padded with zero channels to cs = 8 for the cuBLAS wgrad, or to cs = 64 in
// the hidden layers' gradient buffer for the tcgen05 wgrad), the wgrad
// operand; exports s and 2^-s.
__global__ void __launch_bounds__(kTB)
head_bwd_pack_kernel(const float* __restrict__ gout, int B, int K, int H, int W, const int* amax_bits,
                     __half* __restrict__ gpadc, int cs, int* gexp, float* ginv) {
  const float m = __int_as_float(amax_bits[0]);
  const int e = m > 0.0f ? min(100, max(-100, 10 - (ilogbf(m) + 1))) : 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *gexp = e;
    *ginv = pow2i(-e);
  }
  const float sc = pow2i(e);
  const long long P = (long long)B * H * W;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (long long)gridDim.x * blockDim.x) {
    const int xw = (int)(p % W);
    const long long t = p / W;
    const int yy = (int)(t % H), bi = (int)(t / H);
    __half v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      v[k] = __float2half_rn(k < K ? __ldg(gout + (((long long)bi * K + k) * H + yy) * W + xw) * sc : 0.0f);
    uint4* dst = reinterpret_cast<uint4*>(gpadc + (((long long)bi * (H + 2) + yy + 1) * (W + 2) + xw + 1) * cs);
    dst[0] = *reinterpret_cast<const uint4*>(v);
    for (int c8 = 1; c8 < cs / 8; ++c8) dst[c8] = make_uint4(0u, 0u, 0u, 0u);
  }
}

// Head dgrad (K <= 8 input channels, CUDA cores, fp32): g_a[p][ci] =
// sum_{k,ky,kx} Wh[k][ci][ky][kx] * g_out[k][y+1-ky][x+1-kx].  Thread =
// (pixel, 8-channel chunk); the head weights are staged in shared memory.
__global__ void __launch_bounds__(kTB)
head_dgrad_kernel(const float* __restrict__ gout, const float* __restrict__ wh, int B, int K, int H, int W,
                  float* __restrict__ ga) {
  // [k][tap][ci]: a thread's 8 channels are two 16 B shared loads per (k, tap)
  // (the [k][ci][tap] global order read 8 scalars at stride 9 with 2-way bank
  // conflicts: 104 us for 8 x 128 x 128, shared-memory bound)
  __shared__ __align__(16) float sw[kMaxBands * 9 * 64];
  for (int i = threadIdx.x; i < K * 64 * 9; i += blockDim.x) {
    const int tap = i % 9, ci = (i / 9) % 64, k = i / (9 * 64);
    sw[(k * 9 + tap) * 64 + ci] = wh[i];
  }
  __syncthreads();
  const long long P = (long long)B * H * W;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < P * 8; i += (long long)gridDim.x * blockDim.x) {
    const long long p = i >> 3;
    const int c8 = (int)(i & 7);
    const int xw = (int)(p % W);
    const long long t = p / W;
    const int yy = (int)(t % H), bi = (int)(t / H);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int k = 0; k < K; ++k) {
      const float* g = gout + ((long long)bi * K + k) * H * W;
#pragma unroll
      for (int ky = 0; ky < 3; ++ky) {
        const int sy = yy + 1 - ky;
        if (sy < 0 || sy >= H) continue;
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
          const int sx = xw + 1 - kx;
          if (sx < 0 || sx >= W) continue;
          const float gv = __ldg(g + (long long)sy * W + sx);
          const float4 w0 = *reinterpret_cast<const float4*>(&sw[(k * 9 + ky * 3 + kx) * 64 + c8 * 8]);
          const float4 w1 = *reinterpret_cast<const float4*>(&sw[(k * 9 + ky * 3 + kx) * 64 + c8 * 8 + 4]);
          acc[0] = fmaf(w0.x, gv, acc[0]); acc[1] = fmaf(w0.y, gv, acc[1]);
          acc[2] = fmaf(w0.z, gv, acc[2]); acc[3] = fmaf(w0.w, gv, acc[3]);
          acc[4] = fmaf(w1.x, gv, acc[4]); acc[5] = fmaf(w1.y, gv, acc[5]);
          acc[6] = fmaf(w1.z, gv, acc[6]); acc[7] = fmaf(w1.w, gv, acc[7]);
        }
      }
    }
    float* dst = ga + p * 64 + c8 * 8;
    *reinterpret_cast<float4*>(dst) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    *reinterpret_cast<float4*>(dst + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
}

// conv0 backward: g_z0 = g_a0 * [a_0 > 0]; dW0[co][tap] = sum g_z0 * x(tap),
// db0[co] = sum g_z0 (fp64).  Thread t owns channel t % 64, pixel lane t / 64.
__global__ void __launch_bounds__(kTB)
conv0_bwd_kernel(const float* __restrict__ ga, const __half* __restrict__ apad, const float* __restrict__ x, int B,
                 int H, int W, double* acc /*[64][10]*/) {
  // thread = (4 channels, pixel lane): one 16 B gradient load and one 8 B
  // activation load per pixel, the 9 image taps shared by the pixel's 16
  // threads (the one-channel-per-thread walk was latency-bound: 125 us)
  const int c4 = threadIdx.x & 15, lane = threadIdx.x >> 4;
  const long long P = (long long)B * H * W;
  float s[4][10];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int j = 0; j < 10; ++j) s[k][j] = 0.0f;
  for (long long p = (long long)blockIdx.x * kRedPx + lane; p < P; p += (long long)gridDim.x * kRedPx) {
    const int xw = (int)(p % W);
    const long long t = p / W;
    const int yy = (int)(t % H), bi = (int)(t / H);
    const uint2 a0 = __ldg(reinterpret_cast<const uint2*>(
        apad + (((long long)bi * (H + 2) + yy + 1) * (W + 2) + xw + 1) * 128 + c4 * 4));
    const float4 g4 = __ldg(reinterpret_cast<const float4*>(ga + p * 64) + c4);
    const __half2 h01 = *reinterpret_cast<const __half2*>(&a0.x), h23 = *reinterpret_cast<const __half2*>(&a0.y);
    const float av[4] = {__low2float(h01), __high2float(h01), __low2float(h23), __high2float(h23)};
    const float gv[4] = {g4.x, g4.y, g4.z, g4.w};
    const float* img = x + (long long)bi * H * W;
    float tap[9];
#pragma unroll
    for (int ky = 0; ky < 3; ++ky)
#pragma unroll
      for (int kx = 0; kx < 3; ++kx) {
        const int sy = yy + ky - 1, sx = xw + kx - 1;
        tap[ky * 3 + kx] = (sy >= 0 && sy < H && sx >= 0 && sx < W) ? __ldg(img + (long long)sy * W + sx) : 0.0f;
      }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float gz = av[k] > 0.0f ? gv[k] : 0.0f;
#pragma unroll
      for (int j = 0; j < 9; ++j) s[k][j] = fmaf(gz, tap[j], s[k][j]);
      s[k][9] += gz;
    }
  }
  __shared__ float sh[kRedPx][64][10];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int j = 0; j < 10; ++j) sh[lane][c4 * 4 + k][j] = s[k][j];
  __syncthreads();
  for (int i = threadIdx.x; i < 640; i += blockDim.x) {
    double v = 0.0;
    for (int l = 0; l < kRedPx; ++l) v += (&sh[l][0][0])[i];
    atomicAdd(acc + i, v);
  }
}

// wgrad GEMM outputs C_tap (col-major M x 64: element (m, ci) at m + M*ci) ->
// dW[m][ci][ky][kx] (the Conv2d weight layout) for the first `rows` channels
__global__ void wgrad_scatter_kernel(const float* __restrict__ c9, int M, int rows, float* __restrict__ dw) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // (m, ci, tap)
  if (i >= rows * 64 * 9) return;
  const int tap = i % 9, ci = (i / 9) % 64, m = i / (9 * 64);
  dw[i] = c9[(long long)tap * M * 64 + m + (long long)M * ci];
}

__global__ void conv0_grad_finish_kernel(const double* acc, float* dw0, float* db0) {
  const int c = threadIdx.x;
  if (c >= 64) return;
  for (int k = 0; k < 9; ++k) dw0[c * 9 + k] = (float)acc[c * 10 + k];
  db0[c] = (float)acc[c * 10 + 9];
}

__global__ void head_bias_finish_kernel(const double* acc, int K, float* dbh) {
  if (threadIdx.x < K) dbh[threadIdx.x] = (float)acc[threadIdx.x];
}

__global__ void fill_ones_kernel(float* p, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = 1.0f;
}

}  // namespace tvs

// ---------------------------------------------------------------- host ----
using tvs_host::DeviceGuard;
using tvs_host::TvsError;
using tvs_host::guarded;
using tvs_host::make_act_map;

struct tvs_train {
  int device = 0, depth = 17, out_bands = 5, num_sms = 148;
  cublasHandle_t blas = nullptr;
  // weights of the current step: split packs (forward), transposed fp16 packs
  // (dgrad), head hi/lo pack, unit BN scales
  uint8_t* wsplit = nullptr;
  uint8_t* wt = nullptr;
  uint8_t* hpack = nullptr;
  uint8_t* wt_head = nullptr;  // head filter as a transposed 64 x 64 dgrad pack (zero rows above out_bands)
  float* ones = nullptr;
  float* zero_shift = nullptr;
  // per-shape workspace
  int B = 0, H = 0, W = 0;
  long long guard = 0;       // zero pixels before/after every padded buffer
  std::vector<void*> apad;   // depth-1 pair buffers (interior origin = base + guard + (W+2) + 1 pixels)
  std::vector<float*> y;     // depth-2 pre-BN outputs
  void* gpad = nullptr;      // fp16 gradient operand [B][H+2][W+2][64] (+ guards)
  void* gpad8 = nullptr;     // head gradient operand [B][H+2][W+2][8] (+ guards)
  float* ga[2] = {nullptr, nullptr};
  double* sums = nullptr;    // (depth-2) x 128 batch sums
  // backward reductions, zeroed by ONE memset per step (they share an allocation):
  // red = [8 head bias | 640 conv0 | 128 BN-backward sums per hidden layer] doubles,
  // amax = [2 head | 2 per hidden layer] ints (float bits)
  double* red = nullptr;
  int* amax = nullptr;
  size_t red_bytes = 0;
  int* gexp = nullptr;
  float* ginv = nullptr;     // 2^-s per layer (device scalars for cuBLAS alpha)
  float* fzero = nullptr;
  float* c9 = nullptr;       // 9 x 64 x 64 wgrad GEMM outputs
  // wgrad on tcgen05 (wgrad_tc.cu; option "wgrad_tc", default on): split-K
  // partials and the 2-D tensor maps of the gradient / activation buffers
  int wgrad_tc = 1;
  int bn_bwd_fused = 1;   // BatchNorm backward's two passes in one cooperative launch (0: two kernels)
  int bn_bwd_coop_blocks = 0;  // co-resident blocks of bn_bwd_fused_kernel on this device (0: unknown yet)
  int bn_fused = 1;       // batch statistics summed in the forward conv's epilogue (0: bn_stats_kernel pass)
  int head_dgrad_tc = 1;  // head input gradient on the tcgen05 dgrad kernel (needs wgrad_tc's 64-channel operand)
  float* wpart = nullptr;
  CUtensorMap gmap;
  std::vector<CUtensorMap> amaps;
  float eps = 1e-5f;
  bool have_forward = false;
  std::vector<const float*> wv, biasv, gammav, betav;
  const float* x = nullptr;
};

namespace {

void train_free_ws(tvs_train* t) {
  for (void* p : t->apad) cudaFree(p);
  for (float* p : t->y) cudaFree(p);
  t->apad.clear();
  t->y.clear();
  void* ptrs[] = {t->gpad, t->gpad8, t->ga[0], t->ga[1]};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  t->gpad = t->gpad8 = nullptr;
  t->ga[0] = t->ga[1] = nullptr;
  t->B = t->H = t->W = 0;
}

size_t pad_px(const tvs_train* t) { return (size_t)t->B * (t->H + 2) * (t->W + 2) + 2 * (size_t)t->guard; }
template <typename T>
T* interior(void* base, const tvs_train* t, int ch) {  // pixel (b=0, y=0, x=0) of a padded buffer
  return reinterpret_cast<T*>(base) + ((size_t)t->guard + (size_t)(t->W + 2) + 1) * ch;
}
template <typename T>
T* padded0(void* base, const tvs_train* t, int ch) {  // pixel (b=0, y=-1, x=-1)
  return reinterpret_cast<T*>(base) + (size_t)t->guard * ch;
}

void train_ensure_ws(tvs_train* t, int B, int H, int W) {
  if (t->B == B && t->H == H && t->W == W) return;
  train_free_ws(t);
  t->B = B; t->H = H; t->W = W;
  t->guard = W + 3;
  const size_t P = (size_t)B * H * W, PP = pad_px(t);
  const int nh = t->depth - 2;
  for (int j = 0; j <= nh; ++j) {  // a_0 .. a_{nh}
    void* p = nullptr;
    TVS_CUDA(cudaMalloc(&p, PP * 256));
    TVS_CUDA(cudaMemset(p, 0, PP * 256));  // borders and guards stay zero
    t->apad.push_back(p);
  }
  for (int j = 0; j < nh; ++j) {
    float* p = nullptr;
    TVS_CUDA(cudaMalloc(&p, P * 256));
    t->y.push_back(p);
  }
  TVS_CUDA(cudaMalloc(&t->gpad, PP * 128));
  TVS_CUDA(cudaMemset(t->gpad, 0, PP * 128));
  TVS_CUDA(cudaMalloc(&t->gpad8, PP * 16));
  TVS_CUDA(cudaMemset(t->gpad8, 0, PP * 16));
  for (int i = 0; i < 2; ++i) TVS_CUDA(cudaMalloc(&t->ga[i], P * 256));
  t->gmap = tvs::make_wgrad_gmap(t->gpad, (long long)PP);
  t->amaps.clear();
  for (int j = 0; j <= nh; ++j) t->amaps.push_back(tvs::make_wgrad_amap(t->apad[j], (long long)PP));
}

// dW of one conv (rows = its output channels) from the gradient operand in
// t->gpad and the pair activations a_j (hi halves)
void wgrad_tc(tvs_train* t, int j, int rows, const float* alpha, float* dw, cudaStream_t st) {
  const long long PP = (long long)t->B * (t->H + 2) * (t->W + 2);
  TVS_CUDA(tvs::launch_wgrad_tc(t->gmap, t->amaps[j], PP, (int)t->guard, t->W, rows, alpha, t->wpart, dw, t->num_sms,
                                st));
}

// reductions ending in fp64 atomics on one address per channel: 2 blocks per SM
// (1184 blocks' atomics serialised in L2 and were slower than 512)
int grid_red(long long work, int per_block, int num_sms) {
  return (int)std::max(1LL, std::min<long long>((work + per_block - 1) / per_block, (long long)num_sms * 2));
}

int grid_for(long long work, int per_block, int num_sms) {
  return (int)std::max(1LL, std::min<long long>((work + per_block - 1) / per_block, (long long)num_sms * 8));
}

// C_tap = G (M x PP, ld ldg) * A_shift(tap)^T (PP x 64, ld 128 halves), alpha = 2^-s on the device
void wgrad_gemms(tvs_train* t, const __half* g, int M, int ldg, void* a_base, const float* alpha, cudaStream_t st) {
  const long long PP = (long long)t->B * (t->H + 2) * (t->W + 2);
  const __half* a0 = padded0<__half>(a_base, t, 128);
  TVS_CUDA(cudaMemsetAsync(t->c9, 0, 9 * 64 * 64 * sizeof(float), st));
  if (cublasSetStream(t->blas, st) != CUBLAS_STATUS_SUCCESS) throw TvsError(TVS_E_CUDA, "cublasSetStream failed");
  for (int tap = 0; tap < 9; ++tap) {
    const long long off = (long long)(tap / 3 - 1) * (t->W + 2) + (tap % 3 - 1);
    const cublasStatus_t r = cublasGemmEx(t->blas, CUBLAS_OP_N, CUBLAS_OP_T, M, 64, (int)PP, alpha, g, CUDA_R_16F,
                                          ldg, a0 + off * 128, CUDA_R_16F, 128, t->fzero, t->c9 + (size_t)tap * M * 64,
                                          CUDA_R_32F, M, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
    if (r != CUBLAS_STATUS_SUCCESS) throw TvsError(TVS_E_CUDA, "cublasGemmEx (wgrad) failed: " + std::to_string((int)r));
  }
}

}  // namespace

extern "C" {

int tvs_train_create(int device, int depth, int out_bands, tvs_train** out) {
  return guarded([&] {
    if (!out) throw TvsError(TVS_E_INVALID, "out is null");
    *out = nullptr;
    if (depth < 3) throw TvsError(TVS_E_INVALID, "depth must be at least 3 (first, hidden, last)");
    if (out_bands < 1 || out_bands > 8) throw TvsError(TVS_E_UNSUPPORTED, "out_bands must be in [1, 8]");
    int ndev = 0;
    TVS_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw TvsError(TVS_E_INVALID, "bad device ordinal");
    DeviceGuard dg(device);
    cudaDeviceProp prop;
    TVS_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0) throw TvsError(TVS_E_UNSUPPORTED, "libtvsb200 is built for sm_100a only");
    auto* t = new tvs_train();
    t->device = device; t->depth = depth; t->out_bands = out_bands; t->num_sms = prop.multiProcessorCount;
    try {
      TVS_CUDA(tvs::configure_kernels());
      if (cublasCreate(&t->blas) != CUBLAS_STATUS_SUCCESS) throw TvsError(TVS_E_CUDA, "cublasCreate failed");
      cublasSetPointerMode(t->blas, CUBLAS_POINTER_MODE_DEVICE);
      const int nh = depth - 2;
      TVS_CUDA(cudaMalloc(&t->wsplit, (size_t)nh * tvs::conv_wpack_split_bytes()));
      TVS_CUDA(cudaMalloc(&t->wt, (size_t)nh * tvs::conv_wpack_bytes(false)));
      TVS_CUDA(cudaMalloc(&t->hpack, tvs::conv_wpack_bytes(true)));
      TVS_CUDA(cudaMalloc(&t->wt_head, tvs::conv_wpack_bytes(false)));
      TVS_CUDA(cudaMalloc(&t->ones, 64 * sizeof(float)));
      TVS_CUDA(cudaMalloc(&t->zero_shift, 64 * sizeof(float)));
      TVS_CUDA(cudaMemset(t->zero_shift, 0, 64 * sizeof(float)));
      tvs::fill_ones_kernel<<<1, 64>>>(t->ones, 64);
      TVS_CUDA(cudaGetLastError());
      TVS_CUDA(cudaMalloc(&t->sums, (size_t)nh * 128 * sizeof(double)));
      t->red_bytes = (size_t)(8 + 640 + 128 * nh) * sizeof(double) + (size_t)(2 + 2 * nh) * sizeof(int);
      TVS_CUDA(cudaMalloc(&t->red, t->red_bytes));
      t->amax = reinterpret_cast<int*>(t->red + 8 + 640 + 128 * nh);
      TVS_CUDA(cudaMalloc(&t->gexp, (depth + 1) * sizeof(int)));
      TVS_CUDA(cudaMalloc(&t->ginv, (depth + 1) * sizeof(float)));
      TVS_CUDA(cudaMalloc(&t->fzero, sizeof(float)));
      TVS_CUDA(cudaMemset(t->fzero, 0, sizeof(float)));
      TVS_CUDA(cudaMalloc(&t->c9, 9 * 64 * 64 * sizeof(float)));
      TVS_CUDA(cudaMalloc(&t->wpart, tvs::wgrad_part_bytes(t->num_sms)));
      TVS_CUDA(cudaDeviceSynchronize());
    } catch (...) {
      if (t->blas) cublasDestroy(t->blas);
      delete t;
      throw;
    }
    *out = t;
  });
}

int tvs_train_forward(tvs_train* t, const float* const* w_dev, const float* const* bias_dev,
                      const float* const* gamma_dev, const float* const* beta_dev, float eps, const float* x,
                      float* out, float* mean_out, float* var_out, int B, int H, int W, void* stream) {
  return guarded([&] {
    if (!t || !w_dev || !bias_dev || !gamma_dev || !beta_dev || !x || !out || !mean_out || !var_out)
      throw TvsError(TVS_E_INVALID, "null argument");
    if (B < 1 || H < 1 || W < 1) throw TvsError(TVS_E_INVALID, "bad shape B/H/W");
    const int nh = t->depth - 2;
    for (int i = 0; i < t->depth; ++i)
      if (!w_dev[i]) throw TvsError(TVS_E_INVALID, "null weight pointer");
    if (!bias_dev[0] || !bias_dev[t->depth - 1]) throw TvsError(TVS_E_INVALID, "conv0/head bias required");
    for (int j = 0; j < nh; ++j)
      if (!gamma_dev[j] || !beta_dev[j]) throw TvsError(TVS_E_INVALID, "null BatchNorm parameter");
    DeviceGuard dg(t->device);
    cudaStream_t st = (cudaStream_t)stream;
    train_ensure_ws(t, B, H, W);
    t->eps = eps;
    t->wv.assign(w_dev, w_dev + t->depth);
    t->biasv.assign(bias_dev, bias_dev + t->depth);
    t->gammav.assign(gamma_dev, gamma_dev + nh);
    t->betav.assign(beta_dev, beta_dev + nh);
    t->x = x;
    // this step's weight packs
    TVS_CUDA(tvs::launch_train_pack_hidden(w_dev + 1, nh, t->wsplit, t->wt, st));
    TVS_CUDA(tvs::launch_pack_head_f16(w_dev[t->depth - 1], t->out_bands, t->hpack, st));
    TVS_CUDA(tvs::launch_pack_head_f16_t(w_dev[t->depth - 1], t->out_bands, t->wt_head, st));
    const long long P = (long long)B * H * W;
    tvs::train_conv0_kernel<<<(unsigned)((P + tvs::kTB - 1) / tvs::kTB), tvs::kTB, 0, st>>>(
        x, w_dev[0], bias_dev[0], B, H, W, padded0<__half>(t->apad[0], t, 128));
    TVS_CUDA(cudaGetLastError());
    TVS_CUDA(cudaMemsetAsync(t->sums, 0, (size_t)nh * 128 * sizeof(double), st));
    const int strips = (W + tvs::kStripPx - 1) / tvs::kStripPx;
    for (int j = 0; j < nh; ++j) {
      const CUtensorMap m = make_act_map(interior<__half>(t->apad[j], t, 128), B, H, W, tvs::kHaloPx, 128, 1);
      tvs::ConvArgs a{};
      a.B = B; a.H = H; a.W = W; a.strips = strips; a.row0 = 0; a.rows = H;
      a.wpack = t->wsplit + (size_t)j * tvs::conv_wpack_split_bytes();
      a.shift = t->zero_shift;
      a.nshift = 64;
      a.act_out = reinterpret_cast<uint8_t*>(t->y[j]);
      a.raw_f32 = 1;
      // CTA pairs (conv_tc.cu mode 12 / 13: one output-channel half per CTA of a
      // cluster, input rows multicast): the fp32 inference mode's faster layout
      const long long total = (long long)B * strips * H;
      const int grid = 2 * (int)std::max(1LL, std::min<long long>(t->num_sms / 2, (total + 2) / 3));
      if (t->bn_fused) a.bn_sums = t->sums + j * 128;
      TVS_CUDA(tvs::launch_conv_tc(12, m, m, a, grid, st));
      if (!t->bn_fused) {
        tvs::bn_stats_kernel<<<grid_red(P, 8 * tvs::kRedPx, t->num_sms), tvs::kTB, 0, st>>>(t->y[j], P,
                                                                                            t->sums + j * 128);
        TVS_CUDA(cudaGetLastError());
      }
      tvs::bn_apply_kernel<<<grid_for(P * 8, tvs::kTB * 4, t->num_sms), tvs::kTB, 0, st>>>(
          t->y[j], B, H, W, t->sums + j * 128, gamma_dev[j], beta_dev[j], eps, padded0<__half>(t->apad[j + 1], t, 128),
          mean_out + j * 64, var_out + j * 64);
      TVS_CUDA(cudaGetLastError());
    }
    // head (model.py:44): fp32-accurate hi/lo head on the last pair
    {
      const CUtensorMap m = make_act_map(interior<__half>(t->apad[nh], t, 128), B, H, W, tvs::kHaloPx, 128, 1);
      tvs::ConvArgs a{};
      a.B = B; a.H = H; a.W = W; a.strips = strips; a.row0 = 0; a.rows = H;
      a.wpack = t->hpack;
      a.shift = bias_dev[t->depth - 1];
      a.nshift = t->out_bands;
      a.x = x; a.bands = out; a.closure = nullptr; a.K = t->out_bands;
      const long long total = (long long)B * strips * H;
      const int grid = (int)std::max(1LL, std::min<long long>(t->num_sms, (total + 2) / 3));
      TVS_CUDA(tvs::launch_conv_tc(4, m, m, a, grid, st));
    }
    t->have_forward = true;
  });
}

int tvs_train_backward(tvs_train* t, const float* g_out, float* const* dw, float* const* dbias, float* const* dgamma,
                       float* const* dbeta, void* stream) {
  return guarded([&] {
    if (!t || !g_out || !dw || !dbias || !dgamma || !dbeta) throw TvsError(TVS_E_INVALID, "null argument");
    if (!t->have_forward) throw TvsError(TVS_E_STATE, "tvs_train_backward before tvs_train_forward");
    const int nh = t->depth - 2, K = t->out_bands;
    for (int i = 0; i < t->depth; ++i)
      if (!dw[i]) throw TvsError(TVS_E_INVALID, "null weight-gradient pointer");
    if (!dbias[0] || !dbias[t->depth - 1]) throw TvsError(TVS_E_INVALID, "conv0/head bias gradient required");
    DeviceGuard dg(t->device);
    cudaStream_t st = (cudaStream_t)stream;
    const int B = t->B, H = t->H, W = t->W;
    const long long P = (long long)B * H * W;
    const int strips = (W + tvs::kStripPx - 1) / tvs::kStripPx;
    // ---- head: bias grad, fp16 gradient operand, wgrad GEMM, dgrad (CUDA cores)
    TVS_CUDA(cudaMemsetAsync(t->red, 0, t->red_bytes, st));  // every reduction slot of this backward
    double* red_head = t->red;                // 8 head-bias sums
    double* acc0 = t->red + 8;                // 640 conv0 sums
    double* red_bn = t->red + 8 + 640;        // 128 per hidden layer
    int* amax_bn = t->amax + 2;               // 2 per hidden layer
    tvs::head_bwd_reduce_kernel<<<dim3(grid_for((long long)H * W, tvs::kTB * 4, t->num_sms / K + 1), K), tvs::kTB, 0,
                                  st>>>(g_out, B, K, (long long)H * W, red_head, t->amax);
    TVS_CUDA(cudaGetLastError());
    if (t->wgrad_tc) {
      // bands as channels 0..K-1 of the 64-channel gradient buffer (zero above;
      // the hidden layers overwrite its whole interior afterwards)
      tvs::head_bwd_pack_kernel<<<grid_for(P, tvs::kTB * 4, t->num_sms), tvs::kTB, 0, st>>>(
          g_out, B, K, H, W, t->amax, padded0<__half>(t->gpad, t, 64), 64, t->gexp + nh, t->ginv + nh);
      TVS_CUDA(cudaGetLastError());
      wgrad_tc(t, nh, K, t->ginv + nh, dw[t->depth - 1], st);
    } else {
      tvs::head_bwd_pack_kernel<<<grid_for(P, tvs::kTB * 4, t->num_sms), tvs::kTB, 0, st>>>(
          g_out, B, K, H, W, t->amax, padded0<__half>(t->gpad8, t, 8), 8, t->gexp + nh, t->ginv + nh);
      TVS_CUDA(cudaGetLastError());
      wgrad_gemms(t, padded0<__half>(t->gpad8, t, 8), 8, 8, t->apad[nh], t->ginv + nh, st);
      // the GEMM's M = 8 rows hold bands 0..K-1 (the rest are zero channels)
      tvs::wgrad_scatter_kernel<<<(K * 64 * 9 + 255) / 256, 256, 0, st>>>(t->c9, 8, K, dw[t->depth - 1]);
      TVS_CUDA(cudaGetLastError());
    }
    tvs::head_bias_finish_kernel<<<1, 32, 0, st>>>(red_head, K, dbias[t->depth - 1]);
    if (t->wgrad_tc && t->head_dgrad_tc) {
      // head dgrad on the hidden layers' tcgen05 dgrad kernel: the gradient buffer
      // holds the scaled fp16 bands in channels 0..K-1 (zero above), the filter
      // pack has zero rows above K (the CUDA-core kernel below took 109 us, this 22)
      const CUtensorMap m = make_act_map(interior<__half>(t->gpad, t, 64), B, H, W, tvs::kHaloPx, 64, 1);
      tvs::ConvArgs a{};
      a.B = B; a.H = H; a.W = W; a.strips = strips; a.row0 = 0; a.rows = H;
      a.wpack = t->wt_head;
      a.shift = t->zero_shift;
      a.nshift = 64;
      a.act_out = reinterpret_cast<uint8_t*>(t->ga[0]);
      a.raw_f32 = 1;
      a.out_exp = t->gexp + nh;
      const long long total = (long long)B * strips * H;
      const int grid = (int)std::max(1LL, std::min<long long>(t->num_sms, (total + 2) / 3));
      TVS_CUDA(tvs::launch_conv_tc(0, m, m, a, grid, st));
    } else {
      tvs::head_dgrad_kernel<<<grid_for(P * 8, tvs::kTB * 4, t->num_sms), tvs::kTB, 0, st>>>(
          g_out, t->wv[t->depth - 1], B, K, H, W, t->ga[0]);
      TVS_CUDA(cudaGetLastError());
    }
    int cur = 0;
    // ---- hidden layers, top down
    for (int j = nh - 1; j >= 0; --j) {
      const int red_grid = grid_red(P, 4 * tvs::kRedPx, t->num_sms);
      if (t->bn_bwd_fused && t->bn_bwd_coop_blocks == 0) {
        int per_sm = 0;
        TVS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tvs::bn_bwd_fused_kernel, tvs::kTB, 0));
        t->bn_bwd_coop_blocks = std::max(1, per_sm * t->num_sms);
      }
      // one cooperative launch while ga and y (512 B per pixel) stay in L2 between
      // the passes; beyond that the apply pass wants its own, larger grid (64 x 128^2:
      // 13.3 ms fused against 12.4 ms as two kernels)
      const bool fits_l2 = P * 512 <= (96LL << 20);
      if (t->bn_bwd_fused && fits_l2 && red_grid <= t->bn_bwd_coop_blocks) {
        const float* ga_p = t->ga[cur];
        const float* y_p = t->y[j];
        int Bv = B, Hv = H, Wv = W;
        const double* sums_p = t->sums + j * 128;
        const float* gam = t->gammav[j];
        const float* bet = t->betav[j];
        float epsv = t->eps;
        double* red_p = red_bn + j * 128;
        int* amax_p = amax_bn + j * 2;
        __half* gp = padded0<__half>(t->gpad, t, 64);
        int* gexp_p = t->gexp + j;
        float* ginv_p = t->ginv + j;
        float* dg = dgamma[j];
        float* db = dbeta[j];
        void* args[] = {&ga_p, &y_p, &Bv, &Hv, &Wv, &sums_p, &gam, &bet, &epsv, &red_p, &amax_p, &gp, &gexp_p,
                        &ginv_p, &dg, &db};
        const cudaError_t ce = cudaLaunchCooperativeKernel(
            reinterpret_cast<const void*>(tvs::bn_bwd_fused_kernel), dim3(red_grid), dim3(tvs::kTB), args, 0, st);
        if (ce == cudaErrorCooperativeLaunchTooLarge) {
          // the driver cannot make the grid co-resident here (MPS SM limits, green
          // contexts): nothing ran; use the two kernels from now on
          cudaGetLastError();
          t->bn_bwd_fused = 0;
        } else {
          TVS_CUDA(ce);
        }
      }
      if (!(t->bn_bwd_fused && fits_l2 && red_grid <= t->bn_bwd_coop_blocks)) {
        tvs::bn_bwd_reduce_kernel<<<red_grid, tvs::kTB, 0, st>>>(
            t->ga[cur], t->y[j], P, t->sums + j * 128, t->gammav[j], t->betav[j], t->eps, red_bn + j * 128,
            amax_bn + j * 2);
        TVS_CUDA(cudaGetLastError());
        tvs::bn_bwd_apply_kernel<<<grid_for(P * 16, tvs::kTB * 4, t->num_sms), tvs::kTB, 0, st>>>(
            t->ga[cur], t->y[j], B, H, W, t->sums + j * 128, t->gammav[j], t->betav[j], t->eps, red_bn + j * 128,
            amax_bn + j * 2, padded0<__half>(t->gpad, t, 64), t->gexp + j, t->ginv + j, dgamma[j], dbeta[j]);
        TVS_CUDA(cudaGetLastError());
      }
      // wgrad: dW_j = sum g_y (x) a_j-1 (hi halves), unscaled by alpha = 2^-s
      if (t->wgrad_tc) {
        wgrad_tc(t, j, 64, t->ginv + j, dw[j + 1], st);
      } else {
        wgrad_gemms(t, padded0<__half>(t->gpad, t, 64), 64, 64, t->apad[j], t->ginv + j, st);
        tvs::wgrad_scatter_kernel<<<(64 * 64 * 9 + 255) / 256, 256, 0, st>>>(t->c9, 64, 64, dw[j + 1]);
        TVS_CUDA(cudaGetLastError());
      }
      // dgrad: g_a_{j-1} = conv(g_y, W^T flipped) on tcgen05, raw fp32 out * 2^-s
      const CUtensorMap m = make_act_map(interior<__half>(t->gpad, t, 64), B, H, W, tvs::kHaloPx, 64, 1);
      tvs::ConvArgs a{};
      a.B = B; a.H = H; a.W = W; a.strips = strips; a.row0 = 0; a.rows = H;
      a.wpack = t->wt + (size_t)j * tvs::conv_wpack_bytes(false);
      a.shift = t->zero_shift;
      a.nshift = 64;
      a.act_out = reinterpret_cast<uint8_t*>(t->ga[cur ^ 1]);
      a.raw_f32 = 1;
      a.out_exp = t->gexp + j;
      const long long total = (long long)B * strips * H;
      const int grid = (int)std::max(1LL, std::min<long long>(t->num_sms, (total + 2) / 3));
      TVS_CUDA(tvs::launch_conv_tc(0, m, m, a, grid, st));
      cur ^= 1;
    }
    // ---- conv0
    tvs::conv0_bwd_kernel<<<grid_red(P, 8 * tvs::kRedPx, t->num_sms), tvs::kTB, 0, st>>>(
        t->ga[cur], padded0<__half>(t->apad[0], t, 128), t->x, B, H, W, acc0);
    TVS_CUDA(cudaGetLastError());
    tvs::conv0_grad_finish_kernel<<<1, 64, 0, st>>>(acc0, dw[0], dbias[0]);
    TVS_CUDA(cudaGetLastError());
  });
}

int tvs_train_set_option(tvs_train* t, const char* name, int value) {
  return guarded([&] {
    if (!t || !name) throw TvsError(TVS_E_INVALID, "null argument");
    const std::string k(name);
    if (k == "wgrad_tc") t->wgrad_tc = value != 0;  // 0: the cuBLAS split-K GEMMs (one per tap)
    else if (k == "head_dgrad_tc") t->head_dgrad_tc = value != 0;  // 0: the fp32 CUDA-core head dgrad
    else if (k == "bn_bwd_fused") t->bn_bwd_fused = value != 0;  // 0: BatchNorm backward as two kernels
    else if (k == "bn_fused") t->bn_fused = value != 0;  // 0: batch statistics by a separate pass over y
    else throw TvsError(TVS_E_INVALID, "unknown training option: " + k);
  });
}

int tvs_train_destroy(tvs_train* t) {
  return guarded([&] {
    if (!t) return;
    DeviceGuard dg(t->device);
    cudaDeviceSynchronize();
    train_free_ws(t);
    if (t->blas) cublasDestroy(t->blas);
    void* ptrs[] = {t->wsplit, t->wt, t->hpack, t->wt_head, t->ones, t->zero_shift, t->sums, t->red,
                    t->gexp, t->ginv, t->fzero, t->c9, t->wpart};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    delete t;
  });
}

}  // extern "C"
