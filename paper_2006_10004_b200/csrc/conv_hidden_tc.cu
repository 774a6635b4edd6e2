// conv_hidden_tc.cu — K2: one hidden TVSpecNET layer (Conv2d(64,64,3,p=1,no
// bias) -> BatchNorm2d(eval) -> ReLU, /root/reference/pkg/trainer/src/
// tvsurrogate/model.py:40-43) as a tcgen05 implicit GEMM on sm_100a.
//
// Data: activations are fp16 NHWC [B][H][W][64] in HBM (128 B per pixel =
// exactly one 128-byte swizzle row).  BN is folded host-side into W and a
// bias; the weights are rounded to fp16 with tap-sum compensation
// (pack_hidden_f16 below) and kept resident in shared memory.
//
// GEMM mapping (per CTA, persistent over work units = image x 128-px strip x
// band of output rows):
//   * M = 128 output pixels of one row (TMEM lanes),
//   * N = 192 = [W(dy=+1) | W(dy=0) | W(dy=-1)] stacked along N, so ONE
//     input row r updates the accumulators of output rows r-1, r, r+1 which
//     live in consecutive 64-column TMEM slots (slot = row sequence mod 8),
//   * K = 64 input channels x 3 dx taps; a dx tap is a +-128 B shift of the
//     A descriptor start inside the SW128 input-row buffer (one 130-px halo
//     row loaded by TMA, OOB zero fill = Conv2d zero padding).
// N >= 128 keeps the MMA at full rate (N=64 SS MMAs are shared-memory bound
// at 2/3 rate on B200 — measured, tools/ubench_tcgen05.cu).
//
// Warp roles (192 threads): w0 TMA producer, w1 TMEM alloc + MMA issuer,
// w2..w5 epilogue (TMEM -> +bias, ReLU, fp16 -> SW128 smem -> TMA store,
// then zero the slot and hand it back to the MMA warp).
#include "common.cuh"
#include "sm100.cuh"

namespace tvs {

struct UnitGeom {
  int b, x0, ya, yb;
};
TVS_DEV UnitGeom unit_geom(const HiddenArgs& a, int u) {
  UnitGeom g;
  const int s = u % a.strips;
  const int t = u / a.strips;
  const int band = t % a.bands;
  g.b = t / a.bands;
  g.x0 = s * kStripPx;
  g.ya = band * a.band_rows;
  g.yb = min(a.H, g.ya + a.band_rows);
  return g;
}

__global__ void __launch_bounds__(kHiddenThreads, 1)
conv3x3_hidden_f16_kernel(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_out,
                          const HiddenArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;
  uint8_t* sIn = sW + kWBytes;
  uint8_t* sOut = sIn + kStages * kInRowStride;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sOut + 2 * kOutRowBytes);
  uint64_t* full = bars;                 // [kStages]
  uint64_t* empty = full + kStages;      // [kStages]
  uint64_t* slot_full = empty + kStages; // [kSlots]
  uint64_t* slot_empty = slot_full + kSlots;
  uint64_t* wbar = slot_empty + kSlots;
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(wbar + 1);
  float* sBias = reinterpret_cast<float*>(tmem_base_smem + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < kSlots; ++i) { mbar_init(&slot_full[i], 1); mbar_init(&slot_empty[i], 4); }
    mbar_init(wbar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < kC) sBias[threadIdx.x] = a.bias[threadIdx.x];
  if (warp == 1) tmem_alloc<512>(tmem_base_smem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_base_smem;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer ----
    if (elect_one()) {
      prefetch_tmap(&tm_in);
      mbar_arrive_expect_tx(wbar, kWBytes);
      for (int i = 0; i < 3; ++i) bulk_load(sW + i * kWdxBytes, a.wpack + i * kWdxBytes, kWdxBytes, wbar);
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
        const UnitGeom g = unit_geom(a, u);
        const int r0 = max(g.ya - 1, 0), r1 = min(g.yb, a.H - 1);
        for (int r = r0; r <= r1; ++r) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], kInRowBytes);
          tma_load_4d(sIn + stage * kInRowStride, &tm_in, &full[stage], 0, g.x0 - 1, r, g.b);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer ----
    if (elect_one()) {
      const uint32_t idesc64 = make_idesc(128, 64, kFmtF16, kFmtF16);
      const uint32_t idesc128 = make_idesc(128, 128, kFmtF16, kFmtF16);
      const uint32_t idesc192 = make_idesc(128, 192, kFmtF16, kFmtF16);
      const uint32_t sW_u = smem_u32(sW), sIn_u = smem_u32(sIn);
      mbar_wait(wbar, 0);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t seq = 0;  // output-row sequence number: slot = seq & 7, use = seq >> 3
      for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
        const UnitGeom g = unit_geom(a, u);
        const int r0 = max(g.ya - 1, 0), r1 = min(g.yb, a.H - 1);
        for (int r = r0; r <= r1; ++r) {
          const int q_lo = max(r - 1, g.ya), q_hi = min(r + 1, g.yb - 1);
          // accumulators first touched by this input row must be zeroed & free
          for (int q = q_lo; q <= q_hi; ++q) {
            if (max(q - 1, 0) == r) {
              const uint32_t sq = seq + (uint32_t)(q - g.ya);
              mbar_wait(&slot_empty[sq & 7], (sq >> 3) & 1);
            }
          }
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          // split the target slot range at the ring wrap
          const uint32_t s_lo = (seq + (uint32_t)(q_lo - g.ya)) & 7;
          const int cnt = q_hi - q_lo + 1;
          const int c0 = min(cnt, 8 - (int)s_lo);
          const int c1 = cnt - c0;
          const uint32_t brow0 = (uint32_t)(q_lo - (r - 1)) * 64u;  // first W(dy) block of piece 0
          const uint32_t brow1 = brow0 + (uint32_t)c0 * 64u;
          const uint32_t id0 = c0 == 3 ? idesc192 : (c0 == 2 ? idesc128 : idesc64);
          const uint32_t id1 = c1 == 2 ? idesc128 : idesc64;
          const uint32_t a_base = sIn_u + stage * kInRowStride;
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t ad = make_smem_desc(a_base + dx * 128 + k * 32, 0, 1024, kLayoutSW128);
              const uint32_t wb = sW_u + dx * kWdxBytes + k * 32;
              mma_f16_ss(tmem + s_lo * 64, ad, make_smem_desc(wb + brow0 * 128, 0, 1024, kLayoutSW128), id0, 1);
              if (c1 > 0)
                mma_f16_ss(tmem, ad, make_smem_desc(wb + brow1 * 128, 0, 1024, kLayoutSW128), id1, 1);
            }
          }
          mma_commit(&empty[stage]);
          for (int q = q_lo; q <= q_hi; ++q) {
            if (min(q + 1, a.H - 1) == r) mma_commit(&slot_full[(seq + (uint32_t)(q - g.ya)) & 7]);
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        seq += (uint32_t)(g.yb - g.ya);
      }
    }
  } else {
    // ------------------------------------------------ epilogue (w2..w5) ----
    const int quarter = warp & 3;             // TMEM lane quarter this warp may access
    const int px = quarter * 32 + lane;       // pixel within the strip == TMEM lane
    const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
    const bool leader = (threadIdx.x == 64);
    // zero all slots once, then release them
#pragma unroll 1
    for (int c = 0; c < kSlots * 64; c += 16) tmem_st16_zero(tmem + lane_addr + c);
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0)
      for (int i = 0; i < kSlots; ++i) mbar_arrive(&slot_empty[i]);
    if (leader) prefetch_tmap(&tm_out);

    uint32_t seq = 0;
    int buf = 0;
    for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
      const UnitGeom g = unit_geom(a, u);
      for (int q = g.ya; q < g.yb; ++q, ++seq) {
        const uint32_t slot = seq & 7;
        mbar_wait(&slot_full[slot], (seq >> 3) & 1);
        tc_fence_after();
        uint32_t v[4][16];
#pragma unroll
        for (int j = 0; j < 4; ++j) tmem_ld16(tmem + lane_addr + slot * 64 + j * 16, v[j]);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 4; ++j) reg_fence16(v[j]);
#pragma unroll
        for (int j = 0; j < 4; ++j) tmem_st16_zero(tmem + lane_addr + slot * 64 + j * 16);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&slot_empty[slot]);

        // staging buffer `buf` must be drained by its previous TMA store
        if (leader) bulk_wait_read<1>();
        named_bar_sync(1, 128);
        uint8_t* row = sOut + buf * kOutRowBytes + px * 128;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t packed[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int c = j * 16 + h * 8 + e * 2;
              float f0 = fmaxf(__uint_as_float(v[j][h * 8 + e * 2]) + sBias[c], 0.0f);
              float f1 = fmaxf(__uint_as_float(v[j][h * 8 + e * 2 + 1]) + sBias[c + 1], 0.0f);
              __half2 hv = __floats2half2_rn(f0, f1);
              packed[e] = *reinterpret_cast<uint32_t*>(&hv);
            }
            const int chunk = j * 2 + h;  // 16-byte chunk = 8 channels
            *reinterpret_cast<uint4*>(row + ((chunk ^ (px & 7)) << 4)) =
                make_uint4(packed[0], packed[1], packed[2], packed[3]);
          }
        }
        fence_async_smem();
        named_bar_sync(1, 128);
        if (leader) {
          tma_store_4d(&tm_out, sOut + buf * kOutRowBytes, 0, g.x0, q, g.b);
          bulk_commit();
        }
        buf ^= 1;
      }
    }
    if (leader) bulk_wait<0>();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// --------------------------------------------------------------------------
// Weight pack: folded fp32 W[co][ci][3][3] -> fp16 SW128 tiles (kWBytes).
// Rounding is round-to-nearest, then per (co, ci) the rounding direction of
// individual taps is flipped (cheapest first) while that brings the sum of
// rounding residuals over the 9 taps closer to zero.  This keeps each
// filter's response to locally-constant input (the DC term that dominates
// with non-negative ReLU activations) exact to fp32 precision; it halves the
// fp16 error of the 17-layer stack (tools/emulate_precision.py: 1.04e-2 ->
// 6.1e-3 worst band on config 1).
// --------------------------------------------------------------------------
__device__ __forceinline__ float half_other_side(float w, __half rn) {
  const float r = __half2float(rn);
  if (r == w) return r;
  unsigned short bits = __half_as_ushort(rn);
  const bool toward_up = (r < w);              // need a value above r
  const bool neg = (bits & 0x8000u) != 0;
  if (r == 0.0f) {
    bits = toward_up ? 0x0001u : 0x8001u;      // smallest subnormal of the right sign
  } else {
    // magnitude increases when moving away from zero
    const bool grow = (toward_up != neg);
    bits = grow ? (unsigned short)(bits + 1) : (unsigned short)(bits - 1);
  }
  return __half2float(__ushort_as_half(bits));
}

__global__ void pack_hidden_f16_kernel(const float* __restrict__ w, const float* __restrict__ scale,
                                       uint8_t* __restrict__ out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // co*64 + ci
  if (idx >= kC * kC) return;
  const int co = idx / kC, ci = idx % kC;
  float wv[9], rn[9], alt[9], cost[9];
  float s = 0.0f;
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    wv[t] = w[idx * 9 + t] * scale[co];  // BatchNorm fold W' = W*s (fp32)
    const __half h = __float2half_rn(wv[t]);
    rn[t] = __half2float(h);
    alt[t] = half_other_side(wv[t], h);
    cost[t] = fabsf(alt[t] - wv[t]) - fabsf(rn[t] - wv[t]);
    s += rn[t] - wv[t];
  }
  bool used[9] = {false, false, false, false, false, false, false, false, false};
  for (int it = 0; it < 9; ++it) {
    int best = -1;
    float bc = 3.4e38f;
#pragma unroll
    for (int t = 0; t < 9; ++t)
      if (!used[t] && cost[t] < bc) { bc = cost[t]; best = t; }
    used[best] = true;
    const float d = (alt[best] - wv[best]) - (rn[best] - wv[best]);
    if (fabsf(s + d) < fabsf(s)) { s += d; rn[best] = alt[best]; }
  }
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    const int ky = t / 3, kx = t % 3;
    *reinterpret_cast<__half*>(out + wpack_offset(co, ci, ky, kx)) = __float2half_rn(rn[t]);
  }
}

cudaError_t launch_hidden_f16(const CUtensorMap& tm_in, const CUtensorMap& tm_out, const HiddenArgs& a, int grid,
                              cudaStream_t st) {
  conv3x3_hidden_f16_kernel<<<grid, kHiddenThreads, kHiddenSmem, st>>>(tm_in, tm_out, a);
  return cudaGetLastError();
}

cudaError_t launch_pack_hidden_f16(const float* w, const float* scale, uint8_t* out, cudaStream_t st) {
  pack_hidden_f16_kernel<<<(kC * kC + 127) / 128, 128, 0, st>>>(w, scale, out);
  return cudaGetLastError();
}

__global__ void fill_kernel(float* dst, float v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = v;
}
cudaError_t launch_fill(float* dst, float v, int n, cudaStream_t st) {
  fill_kernel<<<(n + 255) / 256, 256, 0, st>>>(dst, v, n);
  return cudaGetLastError();
}

cudaError_t configure_edge_kernels();
cudaError_t configure_kernels() {
  cudaError_t e = cudaFuncSetAttribute(conv3x3_hidden_f16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kHiddenSmem);
  if (e != cudaSuccess) return e;
  return configure_edge_kernels();
}

}  // namespace tvs
