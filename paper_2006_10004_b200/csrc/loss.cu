// loss.cu — the training losses of /root/reference/pkg/trainer/src/tvsurrogate/
// losses.py:54-129 (compute_loss: per-band normalised squared error, optional
// sum constraint and gradient-Huber terms) as two passes on the GPU, for the
// training step of SURVEY §8(f) row 4 (training.py:45-61 calls
// compute_loss(model(img), gt, img, res, selector) and backpropagates .total).
//
// The reference evaluates the loss with ~100 small torch ops and their autograd
// graph; on B200 that is ~1.2 ms of host time in a 3.7 ms step.  Here:
//   tvs_loss_sums : one pass over pred / gt / image / residual -> fp64 sums
//                   per (b, k): [gt energy, residual energy, Huber num, Huber den]
//                   per b     : [reconstruction error, image energy]
//   tvs_loss_value: the six scalars of LossValue from the sums (one block)
//   tvs_loss_grad : d total / d pred from the same sums (closed form), scaled
//                   by the upstream gradient
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "host_util.h"

namespace tvs {

constexpr int kLossTB = 256;

// huber(d) with torch's convention (F.huber_loss, reduction none)
__device__ __forceinline__ double huber(float d, float delta) {
  const float a = fabsf(d);
  return a <= delta ? 0.5 * (double)d * d : (double)delta * ((double)a - 0.5 * delta);
}
__device__ __forceinline__ float huber_d(float d, float delta) { return fminf(fmaxf(d, -delta), delta); }

__device__ __forceinline__ void block_add(double v, double* dst) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __shared__ double sh[kLossTB / 32];  // reused by the next call after the trailing barrier
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < kLossTB / 32; ++i) t += sh[i];
    atomicAdd(dst, t);
  }
  __syncthreads();
}

// grid (x blocks, B*K): plane (b, k); the k == 0 planes also sum the
// reconstruction error and the image energy of image b (terms bit 0)
__global__ void __launch_bounds__(kLossTB)
loss_sums_kernel(const float* __restrict__ pred, const float* __restrict__ gt, const float* __restrict__ image,
                 const float* __restrict__ residual, int B, int K, int H, int W, int terms, float delta,
                 double* __restrict__ sums) {
  const int bk = blockIdx.y, b = bk / K, k = bk % K;
  const long long HW = (long long)H * W;
  const float* p = pred + (long long)bk * HW;
  const float* g = gt + (long long)bk * HW;
  double e_gt = 0.0, e_res = 0.0, h_num = 0.0, h_den = 0.0, e_rec = 0.0, e_img = 0.0;
  const bool do_sum = (terms & 1) && k == 0, do_hub = terms & 2;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < HW; i += (long long)gridDim.x * blockDim.x) {
    const float pv = __ldg(p + i), gv = __ldg(g + i);
    e_gt += (double)gv * gv;
    const float d = pv - gv;
    e_res += (double)d * d;
    if (do_hub) {
      const int x = (int)(i % W), y = (int)(i / W);
      if (x + 1 < W) {
        const float dp = __ldg(p + i + 1) - pv, dg = __ldg(g + i + 1) - gv;
        h_num += huber(dp - dg, delta);
        h_den += huber(dg, delta);
      }
      if (y + 1 < H) {
        const float dp = __ldg(p + i + W) - pv, dg = __ldg(g + i + W) - gv;
        h_num += huber(dp - dg, delta);
        h_den += huber(dg, delta);
      }
    }
    if (do_sum) {
      float rec = __ldg(residual + (long long)b * HW + i);
      for (int kk = 0; kk < K; ++kk) rec += __ldg(pred + ((long long)b * K + kk) * HW + i);
      const float im = __ldg(image + (long long)b * HW + i);
      const float r = rec - im;
      e_rec += (double)r * r;
      e_img += (double)im * im;
    }
  }
  double* s = sums + (long long)bk * 4;
  block_add(e_gt, s + 0);
  block_add(e_res, s + 1);
  if (do_hub) {
    block_add(h_num, s + 2);
    block_add(h_den, s + 3);
  }
  if (do_sum) {
    block_add(e_rec, sums + (long long)B * K * 4 + b * 2);
    block_add(e_img, sums + (long long)B * K * 4 + b * 2 + 1);
  }
}

// out[0] total, [1] mse, [2] sum term, [3] gradient term, [4] skipped mse bands,
// [5] skipped gradient bands, [6] valid mse bands (losses.py:83-127)
__global__ void loss_value_kernel(const double* __restrict__ sums, int B, int K, int terms, float* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double mse = 0.0, grad = 0.0, sum = 0.0;
  int skip = 0, gskip = 0, valid = 0;
  for (int i = 0; i < B * K; ++i) {
    const double* s = sums + (long long)i * 4;
    if (s[0] > 0.0) { mse += s[1] / s[0]; ++valid; } else ++skip;
    if (terms & 2) {
      if (s[3] > 0.0) grad += s[2] / s[3]; else ++gskip;
    }
  }
  mse /= (double)(B * K);
  grad /= (double)(B * K);
  if (terms & 1) {
    for (int b = 0; b < B; ++b) {
      const double* s = sums + (long long)B * K * 4 + b * 2;
      sum += s[0] / fmax(s[1], 1e-30);
    }
    sum /= (double)B;
  }
  out[1] = (float)mse;
  out[2] = (float)sum;
  out[3] = (float)grad;
  out[0] = (float)(mse + ((terms & 1) ? sum : 0.0) + ((terms & 2) ? grad : 0.0));
  out[4] = (float)skip;
  out[5] = (float)gskip;
  out[6] = (float)valid;
}

// grad[b][k][y][x] = g_total * d total / d pred
__global__ void __launch_bounds__(kLossTB)
loss_grad_kernel(const float* __restrict__ pred, const float* __restrict__ gt, const float* __restrict__ image,
                 const float* __restrict__ residual, int B, int K, int H, int W, int terms, float delta,
                 const double* __restrict__ sums, const float* __restrict__ g_total, float* __restrict__ grad) {
  const int bk = blockIdx.y, b = bk / K;
  const long long HW = (long long)H * W;
  const float* p = pred + (long long)bk * HW;
  const float* g = gt + (long long)bk * HW;
  const double* s = sums + (long long)bk * 4;
  const float up = __ldg(g_total);
  const float c_mse = s[0] > 0.0 ? (float)(2.0 / (s[0] * B * K)) : 0.0f;
  const float c_hub = ((terms & 2) && s[3] > 0.0) ? (float)(1.0 / (s[3] * B * K)) : 0.0f;
  const float c_sum =
      (terms & 1) ? (float)(2.0 / (fmax(sums[(long long)B * K * 4 + b * 2 + 1], 1e-30) * B)) : 0.0f;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < HW; i += (long long)gridDim.x * blockDim.x) {
    const float pv = __ldg(p + i), gv = __ldg(g + i);
    float acc = c_mse * (pv - gv);
    if (c_hub != 0.0f) {
      const int x = (int)(i % W), y = (int)(i / W);
      float h = 0.0f;
      // d(x) = (p[x+1] - p[x]) - (g[x+1] - g[x]), associated as in the forward pass
      if (x + 1 < W) h -= huber_d((__ldg(p + i + 1) - pv) - (__ldg(g + i + 1) - gv), delta);
      if (x > 0) h += huber_d((pv - __ldg(p + i - 1)) - (gv - __ldg(g + i - 1)), delta);
      if (y + 1 < H) h -= huber_d((__ldg(p + i + W) - pv) - (__ldg(g + i + W) - gv), delta);
      if (y > 0) h += huber_d((pv - __ldg(p + i - W)) - (gv - __ldg(g + i - W)), delta);
      acc = fmaf(c_hub, h, acc);
    }
    if (terms & 1) {
      float rec = __ldg(residual + (long long)b * HW + i);
      for (int kk = 0; kk < K; ++kk) rec += __ldg(pred + ((long long)b * K + kk) * HW + i);
      acc = fmaf(c_sum, rec - __ldg(image + (long long)b * HW + i), acc);
    }
    grad[(long long)bk * HW + i] = up * acc;
  }
}

}  // namespace tvs

using tvs_host::TvsError;
using tvs_host::guarded;

namespace {
void loss_check(const float* pred, const float* gt, const float* image, const float* residual, int B, int K, int H,
                int W, int terms) {
  if (!pred || !gt) throw TvsError(TVS_E_INVALID, "null pred / gt");
  if (B < 1 || K < 1 || H < 1 || W < 1) throw TvsError(TVS_E_INVALID, "bad shape B/K/H/W");
  if (terms & ~3) throw TvsError(TVS_E_INVALID, "terms: bit 0 = sum constraint, bit 1 = gradient Huber");
  if ((terms & 1) && (!image || !residual)) throw TvsError(TVS_E_INVALID, "the sum constraint needs image and residual");
}
dim3 loss_grid(int B, int K, int H, int W) {
  const long long HW = (long long)H * W;
  const long long want = std::max(1LL, std::min<long long>((HW + tvs::kLossTB * 4 - 1) / (tvs::kLossTB * 4),
                                                           std::max(1LL, 1184LL / ((long long)B * K))));
  return dim3((unsigned)want, (unsigned)(B * K));
}
}  // namespace

extern "C" {

int tvs_loss_sums(const float* pred, const float* gt, const float* image, const float* residual, int B, int K, int H,
                  int W, int terms, float huber_delta, double* sums, float* values, void* stream) {
  return guarded([&] {
    loss_check(pred, gt, image, residual, B, K, H, W, terms);
    if (!sums || !values) throw TvsError(TVS_E_INVALID, "null sums / values");
    if ((long long)B * K > 65535) throw TvsError(TVS_E_UNSUPPORTED, "B * K must be at most 65535");
    cudaStream_t st = (cudaStream_t)stream;
    TVS_CUDA(cudaMemsetAsync(sums, 0, ((size_t)B * K * 4 + (size_t)B * 2) * sizeof(double), st));
    tvs::loss_sums_kernel<<<loss_grid(B, K, H, W), tvs::kLossTB, 0, st>>>(pred, gt, image, residual, B, K, H, W, terms,
                                                                          huber_delta, sums);
    TVS_CUDA(cudaGetLastError());
    tvs::loss_value_kernel<<<1, 32, 0, st>>>(sums, B, K, terms, values);
    TVS_CUDA(cudaGetLastError());
  });
}

int tvs_loss_grad(const float* pred, const float* gt, const float* image, const float* residual, int B, int K, int H,
                  int W, int terms, float huber_delta, const double* sums, const float* g_total, float* grad_pred,
                  void* stream) {
  return guarded([&] {
    loss_check(pred, gt, image, residual, B, K, H, W, terms);
    if (!sums || !g_total || !grad_pred) throw TvsError(TVS_E_INVALID, "null sums / g_total / grad_pred");
    if ((long long)B * K > 65535) throw TvsError(TVS_E_UNSUPPORTED, "B * K must be at most 65535");
    cudaStream_t st = (cudaStream_t)stream;
    tvs::loss_grad_kernel<<<loss_grid(B, K, H, W), tvs::kLossTB, 0, st>>>(pred, gt, image, residual, B, K, H, W, terms,
                                                                          huber_delta, sums, g_total, grad_pred);
    TVS_CUDA(cudaGetLastError());
  });
}

}  // extern "C"
