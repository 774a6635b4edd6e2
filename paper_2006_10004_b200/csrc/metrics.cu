// metrics.cu — batched band scoring on the GPU:
// per (image, band) plane the statistics behind spectv's band_metrics
// (/root/reference/pkg/src/spectv/metrics.py):
//   psnr  (metrics.py:28-37)   : MSE over the plane
//   ssim  (metrics.py:61-112)  : 11x11 Gaussian (sigma 1.5) windowed SSIM,
//                                mean over the interior [r, H-r) x [r, W-r)
//   slmse (metrics.py:126-150) : sums of squared error / squared prediction
//                                over 16x16 patches at stride 8 (+ a clipped
//                                tail patch); overlapping patch sums are one
//                                weighted reduction, weight(y,x) = number of
//                                row patches x number of column patches that
//                                cover the pixel
//   data range (metrics.py:222-225): gt max - min, floored at 1e-9
// All arithmetic in fp64 like the reference.  Interior SSIM windows never
// reach the border, so the reference's symmetric padding never enters the
// score and is not needed here.
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>
#include "common.cuh"
#include <cstdint>

namespace tvs {

constexpr int kStatFields = 8;  // per plane: mse_sum, num, den, max, min, ssim_sum, n_interior, pad
constexpr int kR = 5;           // SSIM window radius
constexpr int kTile = 32;       // SSIM output tile
constexpr int kSpan = kTile + 2 * kR;

__device__ __forceinline__ double atomic_max_d(double* addr, double v) {
  unsigned long long* p = reinterpret_cast<unsigned long long*>(addr);
  unsigned long long old = *p, assumed;
  do {
    assumed = old;
    if (__longlong_as_double(assumed) >= v) break;
    old = atomicCAS(p, assumed, __double_as_longlong(v));
  } while (old != assumed);
  return __longlong_as_double(old);
}
__device__ __forceinline__ double atomic_min_d(double* addr, double v) {
  unsigned long long* p = reinterpret_cast<unsigned long long*>(addr);
  unsigned long long old = *p, assumed;
  do {
    assumed = old;
    if (__longlong_as_double(assumed) <= v) break;
    old = atomicCAS(p, assumed, __double_as_longlong(v));
  } while (old != assumed);
  return __longlong_as_double(old);
}

// number of patch starts s (0, 8, 16, ..., plus dim-16 if unaligned) with s <= i < s+16
__device__ __forceinline__ int patch_cover(int i, int dim) {
  const int last = dim - 16;
  int cnt = 0;
  // regular starts: multiples of 8 in [max(0, i-15), min(i, last)]
  const int lo = max(0, i - 15), hi = min(i, last);
  if (hi >= lo) cnt = hi / 8 - (lo + 7) / 8 + 1;
  // the clipped tail patch, when last is not a multiple of 8
  if (last % 8 != 0 && i >= last && i < dim) cnt += 1;
  return cnt;
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = (l < (int)(blockDim.x >> 5)) ? red[l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffff, t, o);
  }
  return t;  // valid in thread 0
}

// pass 1: one block-row of a plane per block (grid.x = plane, grid.y = row chunk)
__global__ void __launch_bounds__(256) plane_stats_kernel(const float* __restrict__ gt, const float* __restrict__ pred,
                                                          int H, int W, double* __restrict__ stats) {
  __shared__ double red[8];
  const int plane = blockIdx.x;
  const long long base = (long long)plane * H * W;
  double mse = 0.0, num = 0.0, den = 0.0, mx = -DBL_MAX, mn = DBL_MAX;
  const int rows_per = (H + gridDim.y - 1) / gridDim.y;
  const int y0 = blockIdx.y * rows_per, y1 = min(H, y0 + rows_per);
  const bool slm = H >= 16 && W >= 16;
  for (int y = y0; y < y1; ++y) {
    const int cy = slm ? patch_cover(y, H) : 0;
    for (int x = threadIdx.x; x < W; x += blockDim.x) {
      const double b = gt[base + (long long)y * W + x], h = pred[base + (long long)y * W + x];
      const double d = b - h;
      mse += d * d;
      mx = fmax(mx, b);
      mn = fmin(mn, b);
      if (cy) {
        const double wgt = (double)(cy * patch_cover(x, W));
        num += wgt * d * d;
        den += wgt * h * h;
      }
    }
  }
  double* s = stats + (long long)plane * kStatFields;
  const double t0 = block_sum(mse, red);
  if (threadIdx.x == 0) atomicAdd(&s[0], t0);
  const double t1 = block_sum(num, red);
  if (threadIdx.x == 0) atomicAdd(&s[1], t1);
  const double t2 = block_sum(den, red);
  if (threadIdx.x == 0) atomicAdd(&s[2], t2);
  // max / min: warp reduce then atomics
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffff, mx, o));
    mn = fmin(mn, __shfl_xor_sync(0xffffffff, mn, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomic_max_d(&s[3], mx);
    atomic_min_d(&s[4], mn);
  }
}

// pass 2: SSIM over the interior, 32x32 output tiles, fp64 separable filters
__global__ void __launch_bounds__(256) ssim_kernel(const float* __restrict__ gt, const float* __restrict__ pred, int H,
                                                   int W, const double* __restrict__ range_override,
                                                   double* __restrict__ stats, int tiles_x, int tiles_y) {
  extern __shared__ double sm[];
  double* sb = sm;                           // [kSpan][kSpan] gt
  double* sh = sb + kSpan * kSpan;           // [kSpan][kSpan] pred
  double* hz = sh + kSpan * kSpan;           // [5][kSpan][kTile] horizontally filtered maps
  __shared__ double red[8];
  __shared__ double g[2 * kR + 1];
  const int plane = blockIdx.x / (tiles_x * tiles_y);
  const int t = blockIdx.x % (tiles_x * tiles_y);
  const int oy = kR + (t / tiles_x) * kTile, ox = kR + (t % tiles_x) * kTile;  // first output pixel
  const long long base = (long long)plane * H * W;
  double* s = stats + (long long)plane * kStatFields;
  if (threadIdx.x == 0) {  // metrics.py:40-44 (k / k.sum(); numpy sums 11 terms pairwise = in order here)
    double k[2 * kR + 1], tot = 0.0;
    for (int i = 0; i <= 2 * kR; ++i) {
      const double xv = i - kR;
      k[i] = exp(__ddiv_rn(-__dmul_rn(xv, xv), __dmul_rn(__dmul_rn(2.0, 1.5), 1.5)));
    }
    for (int i = 0; i <= 2 * kR; ++i) tot = __dadd_rn(tot, k[i]);
    for (int i = 0; i <= 2 * kR; ++i) g[i] = __ddiv_rn(k[i], tot);
  }
  for (int i = threadIdx.x; i < kSpan * kSpan; i += blockDim.x) {
    const int yy = oy - kR + i / kSpan, xx = ox - kR + i % kSpan;
    const bool in = yy < H && xx < W;
    sb[i] = in ? (double)gt[base + (long long)yy * W + xx] : 0.0;
    sh[i] = in ? (double)pred[base + (long long)yy * W + xx] : 0.0;
  }
  __syncthreads();
  // horizontal pass: rows [0,kSpan), output cols [0,kTile)
  for (int i = threadIdx.x; i < kSpan * kTile; i += blockDim.x) {
    const int r = i / kTile, c = i % kTile;
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0;
    // same operation order as the reference's float64 numpy passes, with
    // contraction into FMA disabled (explicit _rn intrinsics), so the filtered
    // maps and the SSIM map are bit-identical to metrics.py:44-58, 93-112
#pragma unroll
    for (int k = 0; k <= 2 * kR; ++k) {
      const double b = sb[r * kSpan + c + k], h = sh[r * kSpan + c + k], wk = g[k];
      a0 = __dadd_rn(a0, __dmul_rn(wk, b));
      a1 = __dadd_rn(a1, __dmul_rn(wk, h));
      a2 = __dadd_rn(a2, __dmul_rn(wk, __dmul_rn(b, b)));
      a3 = __dadd_rn(a3, __dmul_rn(wk, __dmul_rn(h, h)));
      a4 = __dadd_rn(a4, __dmul_rn(wk, __dmul_rn(b, h)));
    }
    hz[(0 * kSpan + r) * kTile + c] = a0;
    hz[(1 * kSpan + r) * kTile + c] = a1;
    hz[(2 * kSpan + r) * kTile + c] = a2;
    hz[(3 * kSpan + r) * kTile + c] = a3;
    hz[(4 * kSpan + r) * kTile + c] = a4;
  }
  __syncthreads();
  const double rng = range_override ? range_override[plane] : fmax(__dsub_rn(s[3], s[4]), 1e-9);
  const double c1 = __dmul_rn(__dmul_rn(0.01, rng), __dmul_rn(0.01, rng));
  const double c2 = __dmul_rn(__dmul_rn(0.03, rng), __dmul_rn(0.03, rng));
  double acc = 0.0, cnt = 0.0;
  for (int i = threadIdx.x; i < kTile * kTile; i += blockDim.x) {
    const int r = i / kTile, c = i % kTile;
    const int y = oy + r, x = ox + c;
    if (y >= H - kR || x >= W - kR) continue;
    double u[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k <= 2 * kR; ++k) {
      const double wk = g[k];
#pragma unroll
      for (int m = 0; m < 5; ++m) u[m] = __dadd_rn(u[m], __dmul_rn(wk, hz[(m * kSpan + r + k) * kTile + c]));
    }
    const double vx = fmax(__dsub_rn(u[2], __dmul_rn(u[0], u[0])), 0.0);
    const double vy = fmax(__dsub_rn(u[3], __dmul_rn(u[1], u[1])), 0.0);
    const double cap = __dsqrt_rn(__dmul_rn(vx, vy));
    const double vxy = fmin(fmax(__dsub_rn(u[4], __dmul_rn(u[0], u[1])), -cap), cap);
    const double A = __dadd_rn(__dmul_rn(__dmul_rn(2.0, u[0]), u[1]), c1);
    const double Bv = __dadd_rn(__dmul_rn(2.0, vxy), c2);
    const double Cv = __dadd_rn(__dadd_rn(__dmul_rn(u[0], u[0]), __dmul_rn(u[1], u[1])), c1);
    const double D = __dadd_rn(__dadd_rn(vx, vy), c2);
    acc += __ddiv_rn(__dmul_rn(A, Bv), __dmul_rn(Cv, D));
    cnt += 1.0;
  }
  const double ts = block_sum(acc, red);
  if (threadIdx.x == 0) atomicAdd(&s[5], ts);
  const double tc = block_sum(cnt, red);
  if (threadIdx.x == 0) atomicAdd(&s[6], tc);
}

__global__ void init_stats_kernel(double* stats, int planes) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < planes) {
    double* s = stats + (long long)i * kStatFields;
    s[0] = s[1] = s[2] = s[5] = s[6] = s[7] = 0.0;
    s[3] = -DBL_MAX;
    s[4] = DBL_MAX;
  }
}

size_t band_stats_ssim_smem() { return (size_t)(2 * kSpan * kSpan + 5 * kSpan * kTile) * sizeof(double); }

cudaError_t launch_band_stats(const float* gt, const float* pred, int planes, int H, int W,
                              const double* range_override, double* stats, cudaStream_t st) {
  init_stats_kernel<<<(planes + 255) / 256, 256, 0, st>>>(stats, planes);
  const int ychunks = (H + 31) / 32;
  plane_stats_kernel<<<dim3(planes, ychunks), 256, 0, st>>>(gt, pred, H, W, stats);
  const int ih = H - 2 * kR, iw = W - 2 * kR;
  if (ih > 0 && iw > 0) {
    const int tx = (iw + kTile - 1) / kTile, ty = (ih + kTile - 1) / kTile;
    static std::mutex mu;
    static uint64_t done = 0;
    cudaError_t e = once_per_device(mu, done, [] {
      return cudaFuncSetAttribute(ssim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)band_stats_ssim_smem());
    });
    if (e != cudaSuccess) return e;
    ssim_kernel<<<planes * tx * ty, 256, band_stats_ssim_smem(), st>>>(gt, pred, H, W, range_override, stats, tx,
                                                                         ty);
  }
  return cudaGetLastError();
}

}  // namespace tvs
