// tvflow.cu — model-driven spectral TV decomposition on the GPU (SURVEY.md
// §8(f) row 3: the ground-truth producer the surrogate replaces).
//
// Restates, per image, /root/reference/pkg/src/spectv:
//   rof_prox / _primal_dual   solver.py:242-372  accelerated PDHG for the ROF
//                             prox, relative duality gap certified every 10
//                             iterations with the best feasible dual scaling
//                             (_certified_pair :134-150), adaptive restart
//                             (:307-315), flat-input shortcut (:358-366)
//   ModelDrivenDecomposer.analyze  pipeline.py:105-145: streamed flow,
//                             phi_i = i*(u_{i+1} - 2u_i + u_{i-1})/dt summed
//                             into dyadic bands, spectrum S_i = sum|phi_i|,
//                             residual f_r = u_N - N(u_N - u_{N-1})
// Arithmetic is fp64 with the reference's operation order (explicit _rn
// intrinsics, no FMA contraction) so iterates track the numpy solver to the
// last bits; only reductions (sums) are ordered differently.
//
// Two kernels, chosen per image size:
//  * tvflow_cluster_kernel (the fast path): the PDHG state of an image (u, v,
//    vbar, qx, qy: 40 B/px) lives entirely in SHARED memory, split by rows
//    over a thread-block cluster of G = 1..16 CTAs (<= 5.5 K px per CTA, so up
//    to 256x344 at G = 16).  One iteration = two fully parallel phases (dual
//    step, primal step) separated by cluster barriers; the one halo row each
//    phase needs is read from the neighbouring CTA over DSMEM.  Gap-certificate
//    sums are reduced per CTA and combined in rank order by every CTA, so all
//    CTAs take identical stop/restart decisions.  HBM is touched once per flow
//    step (u_prev and the band being accumulated), never per iteration.
//  * tvflow_kernel (any size with W <= 2048): one persistent CTA per image,
//    state in global memory.  One PDHG iteration is ONE in-place row sweep: the dual update of row y needs vbar
// rows y, y+1 (not yet overwritten), and the divergence at row y needs the
// new dual of row y-1, kept in registers, and the new x-dual of the left
// neighbour, exchanged through shared memory.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <mutex>

#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"

namespace tvs {

constexpr int kTvThreads = 256;
constexpr int kTvMaxCols = kTvMaxW / kTvThreads;  // columns per thread

__device__ __forceinline__ double block_sum_d(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = (l < (int)(blockDim.x >> 5)) ? red[l] : 0.0;
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffff, t, o);
  return t;  // valid in every lane of every warp
}

// a / b for b > 0 with rb = RN(1/b): q = RN(a rb) is within 1 ulp of a/b and
// one FMA correction makes it the correctly rounded quotient (Markstein's
// theorem; no over/underflow in this range), i.e. bitwise equal to a / b.
__device__ __forceinline__ double div_recip(double a, double b, double rb) {
  const double q = __dmul_rn(a, rb);
  const double r = __fma_rn(-q, b, a);
  return __fma_rn(r, rb, q);
}

// Dual projection of solver.py:278-282: scale = max(|q|/dt, 1); q /= scale.
// |q| is evaluated as the correctly rounded sqrt of RN(qx^2 + qy^2) (within
// an ulp of libm's hypot); pairs provably inside the ball keep scale == 1
// exactly and skip the (then exact) unit division.
__device__ __forceinline__ void project_ball(double& px, double& py, double dt, double rdt, double dt2_lo) {
  const double s2 = __dadd_rn(__dmul_rn(px, px), __dmul_rn(py, py));
  if (s2 < dt2_lo) return;
  const double sc = fmax(div_recip(__dsqrt_rn(s2), dt, rdt), 1.0);
  if (sc != 1.0) {
    const double r = __drcp_rn(sc);
    px = div_recip(px, sc, r);
    py = div_recip(py, sc, r);
  }
}

__device__ __forceinline__ double relative_gap(double primal, double dual, double floor_) {
  return __ddiv_rn(__dsub_rn(primal, dual), fmax(fmax(fabs(primal), fabs(dual)), floor_));
}

__global__ void __launch_bounds__(kTvThreads) tvflow_kernel(const TvFlowArgs a) {
  __shared__ double red[32];
  __shared__ double s_row[kTvMaxCols * kTvThreads];  // new x-dual of the current row
  const int img = blockIdx.x;
  const int H = a.H, W = a.W;
  const long long plane = (long long)H * W;
  double* wk = a.work + (long long)img * 6 * plane;
  double* P[3] = {wk, wk + plane, wk + 2 * plane};
  double* vbar = wk + 3 * plane;
  double* qx = wk + 4 * plane;
  double* qy = wk + 5 * plane;
  double* bands = a.bands + (long long)img * a.n_bands * plane;
  const double dt = a.dt;
  const double rdt = __drcp_rn(dt);
  const double dt2_lo = dt * dt * (1.0 - 1e-12);
  const int tid = threadIdx.x;

  // u_prev = f ; zero bands ; dual = 0
  const double* fimg = a.f + (long long)img * plane;
  for (long long i = tid; i < plane; i += blockDim.x) {
    P[0][i] = fimg[i];
    qx[i] = 0.0;
    qy[i] = 0.0;
  }
  for (long long i = tid; i < plane * a.n_bands; i += blockDim.x) bands[i] = 0.0;
  __syncthreads();

  int iu = 0;  // index of the prox input u in P; u_prev / u_next rotate around it
  int iprev = -1;
  int band_idx = 0;
  for (int step = 0; step < a.n_steps; ++step) {
    double* u = P[iu];
    const int iv = (iu + 1) % 3;  // prox output buffer (u_next); never aliases u_prev (see rotation)
    double* v = P[iv];
    // ---- rof_prox (solver.py:323-372) --------------------------------------
    // flat-input shortcut: mean, flat_gap, scale floor
    double su = 0.0, suu = 0.0;
    for (long long i = tid; i < plane; i += blockDim.x) {
      const double x = u[i];
      su += x;
      suu = __dadd_rn(suu, __dmul_rn(x, x));
    }
    su = block_sum_d(su, red);
    suu = block_sum_d(suu, red);
    const double mean = su / (double)plane;
    const double floor_ = 1e-12 * (1.0 + suu);
    double sfl = 0.0;
    for (long long i = tid; i < plane; i += blockDim.x) {
      const double d = __dsub_rn(u[i], mean);
      sfl = __dadd_rn(sfl, __dmul_rn(d, d));
    }
    const double flat_gap = 0.5 * block_sum_d(sfl, red);
    int iters = 0;
    bool converged = true;
    if (flat_gap <= a.gap_tol * floor_) {
      for (long long i = tid; i < plane; i += blockDim.x) {
        v[i] = mean;
        qx[i] = 0.0;
        qy[i] = 0.0;
      }
      __syncthreads();
    } else {
      // _primal_dual (solver.py:242-320); warm dual already in q (radius dt)
      double tau = a.tau0, sigma = a.sigma0, theta = 1.0, prev_rel = INFINITY, c = 1.0;
      for (long long i = tid; i < plane; i += blockDim.x) {
        v[i] = u[i];
        vbar[i] = u[i];
      }
      __syncthreads();
      while (true) {
        const int n_inner = min(10, a.max_iters - iters);
        for (int it = 0; it < n_inner; ++it) {
          const double th = a.accel ? 1.0 / sqrt(__dadd_rn(1.0, __dmul_rn(2.0, tau))) : theta;
          const double opt = __dadd_rn(1.0, tau);
          const double ropt = __drcp_rn(opt);
          double qy_prev[kTvMaxCols];
          for (int y = 0; y < H; ++y) {
            const long long ro = (long long)y * W;
            double qxn[kTvMaxCols], qyn[kTvMaxCols];
#pragma unroll
            for (int k = 0; k < kTvMaxCols; ++k) {
              const int x = tid + k * kTvThreads;
              if (x >= W) break;
              const double vb = vbar[ro + x];
              double gx = 0.0, gy = 0.0;
              if (x < W - 1) gx = __dmul_rn(__dsub_rn(vbar[ro + x + 1], vb), sigma);
              if (y < H - 1) gy = __dmul_rn(__dsub_rn(vbar[ro + W + x], vb), sigma);
              double px = __dadd_rn(qx[ro + x], gx), py = __dadd_rn(qy[ro + x], gy);
              project_ball(px, py, dt, rdt, dt2_lo);
              qxn[k] = px;
              qyn[k] = py;
              s_row[x] = px;
            }
            __syncthreads();  // all vbar(y, .) reads done; new x-duals of row y visible
#pragma unroll
            for (int k = 0; k < kTvMaxCols; ++k) {
              const int x = tid + k * kTvThreads;
              if (x >= W) break;
              const double uu = u[ro + x];
              double dq;  // div(q) + u with the reference's boundary folding
              if (W > 1) {
                if (x == 0) dq = __dadd_rn(qxn[k], uu);
                else if (x == W - 1) dq = __dsub_rn(uu, s_row[x - 1]);
                else dq = __dadd_rn(__dsub_rn(qxn[k], s_row[x - 1]), uu);
              } else {
                dq = uu;
              }
              if (H > 1) {
                if (y == 0) dq = __dadd_rn(dq, qyn[k]);
                else if (y == H - 1) dq = __dsub_rn(dq, qy_prev[k]);
                else dq = __dsub_rn(__dadd_rn(dq, qyn[k]), qy_prev[k]);
              }
              const double vo = v[ro + x];
              const double vn = div_recip(__dadd_rn(__dmul_rn(dq, tau), vo), opt, ropt);
              const double vbn = __dadd_rn(__dmul_rn(__dsub_rn(vn, vo), th), vn);
              qx[ro + x] = qxn[k];
              qy[ro + x] = qyn[k];
              v[ro + x] = vn;
              vbar[ro + x] = vbn;
              qy_prev[k] = qyn[k];
            }
            __syncthreads();  // s_row is rewritten by the next row
          }
          if (a.accel) {
            theta = th;
            tau = __dmul_rn(tau, th);
            sigma = __ddiv_rn(sigma, th);
          }
          ++iters;
        }
        // certificate (_certified_pair with w = div(q))
        double s_res = 0.0, s_tv = 0.0, s_uw = 0.0, s_ww = 0.0;
        for (int y = 0; y < H; ++y) {
          const long long ro = (long long)y * W;
          for (int x = tid; x < W; x += blockDim.x) {
            const double vv = v[ro + x], uu = u[ro + x];
            const double d = __dsub_rn(uu, vv);
            s_res = __dadd_rn(s_res, __dmul_rn(d, d));
            const double gx = (x < W - 1) ? __dsub_rn(v[ro + x + 1], vv) : 0.0;
            const double gy = (y < H - 1) ? __dsub_rn(v[ro + W + x], vv) : 0.0;
            s_tv = __dadd_rn(s_tv, __dsqrt_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy))));
            double w = 0.0;  // divergence (grid.py:64-91)
            if (W > 1) {
              if (x == 0) w = qx[ro];
              else if (x == W - 1) w = -qx[ro + x - 1];
              else w = __dsub_rn(qx[ro + x], qx[ro + x - 1]);
            }
            if (H > 1) {
              if (y == 0) w = __dadd_rn(w, qy[ro + x]);
              else if (y == H - 1) w = __dsub_rn(w, qy[ro - W + x]);
              else w = __dsub_rn(__dadd_rn(w, qy[ro + x]), qy[ro - W + x]);
            }
            s_uw = __dadd_rn(s_uw, __dmul_rn(uu, w));
            s_ww = __dadd_rn(s_ww, __dmul_rn(w, w));
          }
        }
        s_res = block_sum_d(s_res, red);
        s_tv = block_sum_d(s_tv, red);
        s_uw = block_sum_d(s_uw, red);
        s_ww = block_sum_d(s_ww, red);
        const double primal = __dadd_rn(__dmul_rn(0.5, s_res), __dmul_rn(dt, s_tv));
        c = (s_ww == 0.0) ? 1.0 : fmin(fmax(-s_uw / s_ww, 0.0), 1.0);
        const double dual = __dsub_rn(__dmul_rn(-c, s_uw), __dmul_rn(__dmul_rn(0.5 * c, c), s_ww));
        const double rel = relative_gap(primal, dual, floor_);
        if (rel <= a.gap_tol || iters >= a.max_iters) {
          converged = rel <= a.gap_tol;
          break;
        }
        if (a.accel && rel > 0.98 * prev_rel) {  // adaptive restart (solver.py:307-315)
          tau = a.tau0;
          sigma = a.sigma0;
          theta = 1.0;
          for (long long i = tid; i < plane; i += blockDim.x) vbar[i] = v[i];
          __syncthreads();
        }
        prev_rel = rel;
      }
      // warm start for the next prox: dual_field = c*q/dt (solver.py:320), which
      // rof_prox multiplies back by dt (:369-371) — rounded exactly that way
      for (long long i = tid; i < plane; i += blockDim.x) {
        qx[i] = __dmul_rn(div_recip(__dmul_rn(c, qx[i]), dt, rdt), dt);
        qy[i] = __dmul_rn(div_recip(__dmul_rn(c, qy[i]), dt, rdt), dt);
      }
      __syncthreads();
    }
    if (tid == 0) a.iters[(long long)img * a.n_steps + step] = converged ? iters : -(iters + 1);
    // ---- band accumulation (pipeline.py:120-137) ---------------------------
    if (step >= 1) {
      const int i = step;  // phi_i with u_prev = P[iprev], u_curr = u, u_next = v
      while (i > a.schedule[band_idx]) ++band_idx;
      double* band = bands + (long long)band_idx * plane;
      const double* up = P[iprev];
      double s_abs = 0.0;
      for (long long k = tid; k < plane; k += blockDim.x) {
        const double t = __dadd_rn(__dsub_rn(v[k], __dmul_rn(2.0, u[k])), up[k]);
        const double phi = div_recip(__dmul_rn((double)i, t), dt, rdt);
        band[k] = __dadd_rn(band[k], phi);
        s_abs = __dadd_rn(s_abs, fabs(phi));
      }
      s_abs = block_sum_d(s_abs, red);
      if (tid == 0) a.spectrum[(long long)img * (a.n_steps - 1) + (i - 1)] = s_abs;
    }
    __syncthreads();
    // rotate: u_prev <- u, u <- v (the freed buffer becomes the next output)
    iprev = iu;
    iu = iv;
  }
  // bands *= dt ; f_r = u_curr - n (u_curr - u_prev) ; bands[-1] += f_r
  const double* uc = P[iu];
  const double* up = P[iprev];
  const double n = (double)a.n_steps;
  double* res = a.residual + (long long)img * plane;
  for (long long k = tid; k < plane; k += blockDim.x) {
    const double fr = __dsub_rn(uc[k], __dmul_rn(n, __dsub_rn(uc[k], up[k])));
    res[k] = fr;
    for (int b = 0; b < a.n_bands; ++b) {
      double val = __dmul_rn(bands[(long long)b * plane + k], dt);
      if (b == a.n_bands - 1) val = __dadd_rn(val, fr);
      bands[(long long)b * plane + k] = val;
    }
  }
}


// ---------------------------------------------------------------------------
// Cluster / shared-memory resident variant.
namespace cg = cooperative_groups;

constexpr int kTcThreads = 1024;

// Every CTA of the cluster obtains the same K sums: per-CTA block sums are
// published in shared memory and read back by all CTAs in rank order.
template <int K>
__device__ __forceinline__ void cluster_sum(double (&v)[K], double* red, double* slot, double* bcast,
                                            const cg::cluster_group& cl) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double t = v[k];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffff, t, o);
    if (l == 0) red[k * 32 + w] = t;
  }
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double t = (l < nw) ? red[k * 32 + l] : 0.0;
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffff, t, o);
      if (l == 0) slot[k] = t;
    }
  }
  cl.sync();
  if (threadIdx.x < K) {
    double t = 0.0;
    for (int r = 0; r < (int)cl.num_blocks(); ++r) t += cl.map_shared_rank(slot, r)[threadIdx.x];
    bcast[threadIdx.x] = t;
  }
  cl.sync();  // remote reads of `slot` done before it is rewritten; bcast visible
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = bcast[k];
}

// Per-thread pixel geometry, fixed for the whole launch.
constexpr int kTcPix = 4;  // pixels per thread: a CTA holds at most kTcPix * kTcThreads pixels
constexpr int kTcMaxPx = kTcPix * kTcThreads;  // plane stride in shared memory (5 fp64 planes = 160 KB)
constexpr int kPU = 0, kPV = kTcMaxPx, kPVB = 2 * kTcMaxPx, kPQX = 3 * kTcMaxPx, kPQY = 4 * kTcMaxPx;
constexpr unsigned kFx0 = 1u << 16, kFxL = 1u << 17, kFyN = 1u << 18, kFyR = 1u << 19, kFy0 = 1u << 20,
                   kFyL = 1u << 21, kFlp = 1u << 22;

__global__ void __launch_bounds__(kTcThreads, 1) tvflow_cluster_kernel(const TvFlowArgs a, int rows_per) {
  extern __shared__ __align__(16) double sm[];  // planes u | v | vbar | qx | qy, stride kTcMaxPx
  __shared__ double red[4 * 32];
  __shared__ double slot[4];
  __shared__ double bcast[4];
  const cg::cluster_group cl = cg::this_cluster();
  const int G = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int img = blockIdx.x / G;
  const int H = a.H, W = a.W;
  const int row0 = min(H, rank * rows_per);
  const int nrows = min(H, row0 + rows_per) - row0;
  const int nloc = nrows * W;
  const bool has_next = row0 + nrows < H;  // rows below live on rank+1
  const bool has_prev = row0 > 0;          // rows above live on rank-1
  const long long plane = (long long)H * W;
  const long long goff = (long long)row0 * W;
  double* uprev = a.work + (long long)img * 6 * plane + goff;  // global: u_{i-1}, own rows
  double* bands = a.bands + (long long)img * a.n_bands * plane + goff;
  const double dt = a.dt;
  const double dt2_lo = dt * dt * (1.0 - 1e-12);
  const double rdt = __drcp_rn(dt);
  const int tid = threadIdx.x;
  constexpr int nt = kTcThreads;
  const double npx = (double)plane;
  const bool wide = W > 1, tall = H > 1;
  auto bar = [&]() {
    if (G == 1) __syncthreads();
    else cl.sync();
  };
  // remote halo rows (DSMEM): row 0 of rank+1, last row of rank-1
  const double* vb_next0 = has_next ? cl.map_shared_rank(sm + kPVB, rank + 1) : nullptr;
  const double* v_next0 = has_next ? cl.map_shared_rank(sm + kPV, rank + 1) : nullptr;
  const double* qy_prev0 = has_prev ? cl.map_shared_rank(sm + kPQY, rank - 1) + (rows_per - 1) * W : nullptr;
  // Halo addresses are used by boundary-row pixels only: re-derive them inside
  // each sweep (opaque copy) instead of letting the compiler hoist one 64-bit
  // address per pixel into registers.
  auto opaque = [](const double* q) {
    asm volatile("" : "+l"(q));
    return q;
  };

  // pixel k of this thread is p = tid + k * nt (valid while p < nloc)
  unsigned pfl[kTcPix];
#pragma unroll
  for (int k = 0; k < kTcPix; ++k) {
    const int p = tid + k * nt;
    pfl[k] = 0;
    if (p < nloc) {
      const int ly = p / W, x = p - ly * W, y = row0 + ly;
      pfl[k] = (unsigned)x | (x == 0 ? kFx0 : 0) | (x == W - 1 ? kFxL : 0) | (ly + 1 < nrows ? kFyN : 0) |
               (ly + 1 == nrows && has_next ? kFyR : 0) | (y == 0 ? kFy0 : 0) | (y == H - 1 ? kFyL : 0) |
               (ly > 0 ? kFlp : 0);
    }
  }

  const double* fimg = a.f + (long long)img * plane + goff;
#pragma unroll
  for (int k = 0; k < kTcPix; ++k) {
    const int p = tid + k * nt;
    if (p >= nloc) continue;
    const double x = fimg[p];
    sm[kPU + p] = x;
    uprev[p] = x;
    sm[kPQX + p] = 0.0;
    sm[kPQY + p] = 0.0;
  }
  for (int p = tid; p < a.n_bands * nloc; p += nt) {
    const int b = p / nloc, q = p - b * nloc;
    bands[(long long)b * plane + q] = 0.0;
  }
  __syncthreads();

  // div(q) (+ u when with_u) at one pixel, the reference's boundary folding
  auto divq = [&](int p, unsigned fl, const double* qy_prevc, double base, bool with_u) -> double {
    double d;
    if (wide) {
      const double qx = sm[kPQX + p];
      if (fl & kFx0) d = with_u ? __dadd_rn(qx, base) : qx;
      else if (fl & kFxL) d = with_u ? __dsub_rn(base, sm[kPQX + p - 1]) : -sm[kPQX + p - 1];
      else d = with_u ? __dadd_rn(__dsub_rn(qx, sm[kPQX + p - 1]), base) : __dsub_rn(qx, sm[kPQX + p - 1]);
    } else {
      d = with_u ? base : 0.0;
    }
    if (tall) {
      if (fl & kFy0) {
        d = __dadd_rn(d, sm[kPQY + p]);
      } else {
        const double qyp = (fl & kFlp) ? sm[kPQY + p - W] : qy_prevc[fl & 0xffff];
        d = (fl & kFyL) ? __dsub_rn(d, qyp) : __dsub_rn(__dadd_rn(d, sm[kPQY + p]), qyp);
      }
    }
    return d;
  };

  int band_idx = 0;
  for (int step = 0; step < a.n_steps; ++step) {
    // ---- rof_prox flat shortcut (solver.py:358-366) -------------------------
    double s2v[2] = {0.0, 0.0};
#pragma unroll
    for (int k = 0; k < kTcPix; ++k) {
      const int p = tid + k * nt;
      if (p >= nloc) continue;
      const double x = sm[kPU + p];
      s2v[0] += x;
      s2v[1] = __dadd_rn(s2v[1], __dmul_rn(x, x));
    }
    cluster_sum<2>(s2v, red, slot, bcast, cl);
    const double mean = s2v[0] / npx;
    const double floor_ = 1e-12 * (1.0 + s2v[1]);
    double s1v[1] = {0.0};
#pragma unroll
    for (int k = 0; k < kTcPix; ++k) {
      const int p = tid + k * nt;
      if (p >= nloc) continue;
      const double d = __dsub_rn(sm[kPU + p], mean);
      s1v[0] = __dadd_rn(s1v[0], __dmul_rn(d, d));
    }
    cluster_sum<1>(s1v, red, slot, bcast, cl);
    int iters = 0;
    bool converged = true;
    if (0.5 * s1v[0] <= a.gap_tol * floor_) {
#pragma unroll
      for (int k = 0; k < kTcPix; ++k) {
        const int p = tid + k * nt;
        if (p >= nloc) continue;
        sm[kPV + p] = mean;
        sm[kPQX + p] = 0.0;
        sm[kPQY + p] = 0.0;
      }
    } else {
      double tau = a.tau0, sigma = a.sigma0, theta = 1.0, prev_rel = INFINITY, c = 1.0;
#pragma unroll
      for (int k = 0; k < kTcPix; ++k) {
        const int p = tid + k * nt;
        if (p >= nloc) continue;
        sm[kPV + p] = sm[kPU + p];
        sm[kPVB + p] = sm[kPU + p];
      }
      bar();
      while (true) {
        const int n_inner = min(10, a.max_iters - iters);
        for (int it = 0; it < n_inner; ++it) {
          const double th = a.accel ? 1.0 / sqrt(__dadd_rn(1.0, __dmul_rn(2.0, tau))) : theta;
          const double* vb_next = opaque(vb_next0);
          // phase A: q += sigma grad(vbar); project onto the ball of radius dt
#pragma unroll
          for (int k = 0; k < kTcPix; ++k) {
            const int p = tid + k * nt;
            if (p >= nloc) continue;
            const unsigned fl = pfl[k];
            const double vb = sm[kPVB + p];
            const double gx = (fl & kFxL) ? 0.0 : __dmul_rn(__dsub_rn(sm[kPVB + p + 1], vb), sigma);
            double gy = 0.0;
            if (fl & kFyN) gy = __dmul_rn(__dsub_rn(sm[kPVB + p + W], vb), sigma);
            else if (fl & kFyR) gy = __dmul_rn(__dsub_rn(vb_next[fl & 0xffff], vb), sigma);
            double px = __dadd_rn(sm[kPQX + p], gx), py = __dadd_rn(sm[kPQY + p], gy);
            project_ball(px, py, dt, rdt, dt2_lo);
            sm[kPQX + p] = px;
            sm[kPQY + p] = py;
          }
          bar();
          // phase B: v = (v + tau (div q + u)) / (1 + tau); vbar = v + theta (v - v_old)
          const double opt = __dadd_rn(1.0, tau);
          const double ropt = __drcp_rn(opt);
          const double* qy_prevc = opaque(qy_prev0);
#pragma unroll
          for (int k = 0; k < kTcPix; ++k) {
            const int p = tid + k * nt;
            if (p >= nloc) continue;
            const double dq = divq(p, pfl[k], qy_prevc, sm[kPU + p], true);
            const double vo = sm[kPV + p];
            const double vn = div_recip(__dadd_rn(__dmul_rn(dq, tau), vo), opt, ropt);
            sm[kPV + p] = vn;
            sm[kPVB + p] = __dadd_rn(__dmul_rn(__dsub_rn(vn, vo), th), vn);
          }
          bar();
          if (a.accel) {
            theta = th;
            tau = __dmul_rn(tau, th);
            sigma = __ddiv_rn(sigma, th);
          }
          ++iters;
        }
        // certificate (_certified_pair with w = div(q), solver.py:134-150)
        double cs[4] = {0.0, 0.0, 0.0, 0.0};
        const double* v_next = opaque(v_next0);
        const double* qy_prevc = opaque(qy_prev0);
#pragma unroll
        for (int k = 0; k < kTcPix; ++k) {
          const int p = tid + k * nt;
          if (p >= nloc) continue;
          const unsigned fl = pfl[k];
          const double vv = sm[kPV + p], uu = sm[kPU + p];
          const double d = __dsub_rn(uu, vv);
          cs[0] = __dadd_rn(cs[0], __dmul_rn(d, d));
          const double gx = (fl & kFxL) ? 0.0 : __dsub_rn(sm[kPV + p + 1], vv);
          const double gy = (fl & kFyN) ? __dsub_rn(sm[kPV + p + W], vv)
                                        : ((fl & kFyR) ? __dsub_rn(v_next[fl & 0xffff], vv) : 0.0);
          cs[1] = __dadd_rn(cs[1], __dsqrt_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy))));
          const double w = divq(p, fl, qy_prevc, 0.0, false);
          cs[2] = __dadd_rn(cs[2], __dmul_rn(uu, w));
          cs[3] = __dadd_rn(cs[3], __dmul_rn(w, w));
        }
        cluster_sum<4>(cs, red, slot, bcast, cl);
        const double primal = __dadd_rn(__dmul_rn(0.5, cs[0]), __dmul_rn(dt, cs[1]));
        c = (cs[3] == 0.0) ? 1.0 : fmin(fmax(-cs[2] / cs[3], 0.0), 1.0);
        const double dual = __dsub_rn(__dmul_rn(-c, cs[2]), __dmul_rn(__dmul_rn(0.5 * c, c), cs[3]));
        const double rel = relative_gap(primal, dual, floor_);
        if (rel <= a.gap_tol || iters >= a.max_iters) {
          converged = rel <= a.gap_tol;
          break;
        }
        if (a.accel && rel > 0.98 * prev_rel) {
          tau = a.tau0;
          sigma = a.sigma0;
          theta = 1.0;
#pragma unroll
          for (int k = 0; k < kTcPix; ++k) {
            const int p = tid + k * nt;
            if (p < nloc) sm[kPVB + p] = sm[kPV + p];
          }
          bar();
        }
        prev_rel = rel;
      }
#pragma unroll
      for (int k = 0; k < kTcPix; ++k) {
        const int p = tid + k * nt;
        if (p >= nloc) continue;
        sm[kPQX + p] = __dmul_rn(div_recip(__dmul_rn(c, sm[kPQX + p]), dt, rdt), dt);
        sm[kPQY + p] = __dmul_rn(div_recip(__dmul_rn(c, sm[kPQY + p]), dt, rdt), dt);
      }
    }
    if (rank == 0 && tid == 0) a.iters[(long long)img * a.n_steps + step] = converged ? iters : -(iters + 1);
    // ---- band accumulation (pipeline.py:120-137); u_prev <- u; u <- v -------
    double sa[1] = {0.0};
    const int i = step;
    double* band = nullptr;
    if (i >= 1) {
      while (i > a.schedule[band_idx]) ++band_idx;
      band = bands + (long long)band_idx * plane;
    }
#pragma unroll
    for (int k = 0; k < kTcPix; ++k) {
      const int p = tid + k * nt;
      if (p >= nloc) continue;
      const double uc = sm[kPU + p], un = sm[kPV + p];
      if (i >= 1) {
        const double t = __dadd_rn(__dsub_rn(un, __dmul_rn(2.0, uc)), uprev[p]);
        const double phi = div_recip(__dmul_rn((double)i, t), dt, rdt);
        band[p] = __dadd_rn(band[p], phi);
        sa[0] = __dadd_rn(sa[0], fabs(phi));
      }
      uprev[p] = uc;
      sm[kPU + p] = un;
    }
    if (i >= 1) {
      cluster_sum<1>(sa, red, slot, bcast, cl);
      if (rank == 0 && tid == 0) a.spectrum[(long long)img * (a.n_steps - 1) + (i - 1)] = sa[0];
    } else {
      cl.sync();
    }
  }
  const double n = (double)a.n_steps;
  double* res = a.residual + (long long)img * plane + goff;
#pragma unroll
  for (int k = 0; k < kTcPix; ++k) {
    const int p = tid + k * nt;
    if (p >= nloc) continue;
    const double uc = sm[kPU + p];
    const double fr = __dsub_rn(uc, __dmul_rn(n, __dsub_rn(uc, uprev[p])));
    res[p] = fr;
    for (int b = 0; b < a.n_bands; ++b) {
      double val = __dmul_rn(bands[(long long)b * plane + p], dt);
      if (b == a.n_bands - 1) val = __dadd_rn(val, fr);
      bands[(long long)b * plane + p] = val;
    }
  }
  cl.sync();  // no CTA exits while a neighbour may still read its shared memory
}

namespace {
constexpr int kTvSmemMax = 224 * 1024;  // dynamic; static (~1 KB) + dynamic <= 227 KB opt-in
static_assert(kTcMaxPx * 5 * 8 <= kTvSmemMax, "cluster kernel state exceeds shared memory");
// largest usable cluster size per device ordinal (attributes and occupancy are
// per device context), probed once per device under a lock
std::mutex g_cluster_mu;
int g_max_cluster[64] = {};

int usable_cluster_max() {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_cluster_mu);
  if (dev < 64 && g_max_cluster[dev]) return g_max_cluster[dev];
  cudaFuncSetAttribute(tvflow_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTvSmemMax);
  cudaFuncSetAttribute(tvflow_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int best = 1;
  for (int g = 2; g <= 16; g *= 2) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = g;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(g);
    cfg.blockDim = dim3(kTcThreads);
    cfg.dynamicSmemBytes = kTvSmemMax;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, tvflow_cluster_kernel, &cfg) == cudaSuccess && n > 0) best = g;
    cudaGetLastError();
  }
  if (dev < 64) g_max_cluster[dev] = best;
  return best;
}
}  // namespace

// Smallest cluster whose shared memory holds the image, then widened (more
// CTAs per image, fewer pixels per CTA) while the whole batch still fits in
// one wave of SMs: small batches get more SMs per image.
int tvflow_cluster_size(int N, int H, int W) {
  const int gmax = usable_cluster_max();
  int g = 0;
  for (int c = 1; c <= gmax; c *= 2) {
    const long long rows = (H + c - 1) / c;
    if (rows * W <= kTcMaxPx) {
      g = c;
      break;
    }
  }
  if (g == 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  while (g * 2 <= gmax && (long long)N * g * 2 <= sms && (H + 2 * g - 1) / (2 * g) >= 2) g *= 2;
  return g;
}

cudaError_t launch_tvflow(const TvFlowArgs& a, cudaStream_t st) {
  const char* env = getenv("TVS_TVFLOW_KERNEL");  // "global" forces the row-sweep kernel
  const int g = (env && env[0] == 'g') ? 0 : tvflow_cluster_size(a.N, a.H, a.W);
  if (g == 0) {
    tvflow_kernel<<<a.N, kTvThreads, 0, st>>>(a);
    return cudaGetLastError();
  }
  const int rows_per = (a.H + g - 1) / g;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = g;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(a.N * g);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = (size_t)kTcMaxPx * 5 * sizeof(double);
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, tvflow_cluster_kernel, a, rows_per);
}

}  // namespace tvs
