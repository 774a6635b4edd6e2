// conv_pair.cu — two consecutive hidden layers in one kernel (north-star item
// 4: multi-layer fusion keeping activation tiles on chip).
//
// Layer L+1 (Conv2d(64,64)+BN+ReLU, model.py:40-43) consumes layer L's output
// rows straight from shared memory, so each fused pair reads one activation
// and writes one (256 B/px) instead of two of each: the fast hidden stack is
// HBM-bound at burst clocks, this halves its traffic.
//
// Geometry: a thread-block cluster of S CTAs covers the S 128-px strips of the
// image rows it owns (S = ceil(W/128) <= 8).  Every CTA
//   * TMA-loads layer L's 130-px halo input rows (2-stage ring),
//   * runs layer L on tcgen05 into TMEM ring A (4 slots x 64 columns),
//   * writes L's ReLU'd fp16 output rows into a 2-slot "mid" ring in shared
//     memory in the SW128 operand layout, and sends its edge pixels to the
//     neighbouring strips' mid rows over DSMEM (the 1-px halo layer L+1 needs),
//   * runs layer L+1 from the mid ring into TMEM ring B (4 slots x 64),
//   * stores L+1's fp16 output rows to HBM from registers.
// The MMA warp interleaves the layers with layer L+1 two rows behind L.
// Segments of rows recompute one halo row of layer L at each end.
//
// Warp roles: w0 TMA producer, w1 TMEM alloc + MMA issuer, w2-5 epilogue L
// (-> mid ring), w6-9 epilogue L+1 (-> global).
#include "common.cuh"
#include "sm100.cuh"

namespace tvs {

// Protocol watchdog: a wait that times out records (cta, warp, barrier, parity,
// row) here, raises the abort flag so every other wait gives up, and the kernel
// runs to completion (results invalid) instead of hanging the GPU.
__device__ int g_pair_dbg[8];

TVS_DEV void pwait(uint64_t* bar, uint32_t parity, int id, int info) {
  const uint32_t a = smem_u32(bar);
  for (uint32_t i = 0;; ++i) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(ok) : "r"(a), "r"(parity) : "memory");
    if (ok) return;
    if ((i & 1023) == 1023 && *(volatile int*)&g_pair_dbg[0] != 0) return;
    if (i > (1u << 24)) {
      if (atomicCAS(&g_pair_dbg[0], 0, 1) == 0) {
        g_pair_dbg[1] = blockIdx.x;
        g_pair_dbg[2] = threadIdx.x >> 5;
        g_pair_dbg[3] = id;
        g_pair_dbg[4] = (int)parity;
        g_pair_dbg[5] = info;
        __threadfence();
      }
      return;
    }
  }
}

namespace {
constexpr int kPairThreads = 32 * 10;
constexpr int kPairW = 3 * 3 * 64 * 128;                   // one layer's packed B (= mode 0 pack)
constexpr int kPairRing = 2;                               // input / mid ring slots
constexpr size_t kPairSmem = 1024 + 2 * kPairW + 2 * kPairRing * kInRowStride;  // 218112

struct PairSeg {
  int b, ya, yb;  // image, output rows [ya, yb) of the pair
};
// Contiguous range of the B*H image rows per cluster, split at image boundaries.
struct PairIter {
  long long cur, end;
  TVS_DEV PairIter(const PairArgs& a, int cluster, int nclusters) {
    const long long T = (long long)a.B * a.H;
    cur = T * cluster / nclusters;
    end = T * (cluster + 1) / nclusters;
  }
  TVS_DEV bool next(const PairArgs& a, PairSeg& g) {
    if (cur >= end) return false;
    g.b = (int)(cur / a.H);
    g.ya = (int)(cur - (long long)g.b * a.H);
    const long long n = min((long long)(a.H - g.ya), end - cur);
    g.yb = g.ya + (int)n;
    cur += n;
    return true;
  }
};
}  // namespace

__global__ void __launch_bounds__(kPairThreads, 1)
conv3x3_pair_kernel(const __grid_constant__ CUtensorMap tm_in, const PairArgs a) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t full[kPairRing], empty[kPairRing];            // input ring
  __shared__ uint64_t mfull[kPairRing], mempty[kPairRing];          // mid ring
  __shared__ uint64_t lfree[kPairRing], rfree[kPairRing];           // left / right neighbour's mid slot free
  __shared__ uint64_t afull[4], aempty[4], bfull[4], bempty[4], wbar;  // TMEM rings A (layer L), B (L+1)
  __shared__ uint32_t tmem_base_smem;
  __shared__ __align__(16) float sShift[2][kC];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW0 = smem;
  uint8_t* sW1 = sW0 + kPairW;
  uint8_t* sIn = sW1 + kPairW;
  uint8_t* sMid = sIn + kPairRing * kInRowStride;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = a.S;
  const int rank = (int)cluster_ctarank();
  const int cluster = blockIdx.x / S, nclusters = gridDim.x / S;
  const int x0 = rank * kStripPx;
  const bool halo_x = !(a.dbg & 1);
  if (threadIdx.x == 0 && (a.dbg & 16)) {  // bring-up: record the cluster geometry this CTA sees
    uint32_t nc;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(nc));
    if ((int)nc != S || rank != (int)(blockIdx.x % S)) {
      if (atomicCAS(&g_pair_dbg[0], 0, 2) == 0) {
        g_pair_dbg[1] = blockIdx.x;
        g_pair_dbg[2] = rank;
        g_pair_dbg[3] = (int)nc;
        g_pair_dbg[4] = S;
      }
    }
  }
  const bool has_left = halo_x && rank > 0, has_right = halo_x && rank < S - 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kPairRing; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&mfull[i], 4 + ((a.dbg & 128) ? 0 : (has_left ? 1 : 0) + (has_right ? 1 : 0)));
      mbar_init(&mempty[i], 1);
      mbar_init(&lfree[i], 1);
      mbar_init(&rfree[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&afull[i], 1);
      mbar_init(&aempty[i], 4);
      mbar_init(&bfull[i], 1);
      mbar_init(&bempty[i], 4);
    }
    mbar_init(&wbar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 2 * kC) sShift[threadIdx.x / kC][threadIdx.x % kC] = (threadIdx.x < kC ? a.shift0 : a.shift1)[threadIdx.x % kC];
  if (warp == 1) tmem_alloc<512>(&tmem_base_smem);
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&wbar, 2 * kPairW);
    for (int i = 0; i < 3; ++i) {
      bulk_load(sW0 + i * (kPairW / 3), a.wpack0 + i * (kPairW / 3), kPairW / 3, &wbar);
      bulk_load(sW1 + i * (kPairW / 3), a.wpack1 + i * (kPairW / 3), kPairW / 3, &wbar);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // every CTA's barriers exist before any remote arrive
  tc_fence_after();
  const uint32_t tmem = tmem_base_smem;
  pdl_launch_dependents();
  pdl_wait();

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer ----
    if (elect_one()) {
      prefetch_tmap(&tm_in);
      int stage = 0;
      uint32_t phase = 0;
      PairIter it(a, cluster, nclusters);
      PairSeg g;
      while (it.next(a, g)) {
        const int qa0 = max(g.ya - 1, 0), qa1 = min(g.yb, a.H - 1);
        for (int r = max(qa0 - 1, 0); r <= min(qa1 + 1, a.H - 1); ++r) {
          pwait(&empty[stage], phase ^ 1, 1, r);
          mbar_arrive_expect_tx(&full[stage], kInRowBytes);
          tma_load_4d(sIn + stage * kInRowStride, &tm_in, &full[stage], 0, x0 - 1, r, g.b);
          if (++stage == kPairRing) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------- MMA issuer ----
    const uint32_t idesc1 = make_idesc(128, 64, kFmtF16, kFmtF16);
    const uint32_t idesc2 = make_idesc(128, 128, kFmtF16, kFmtF16);
    const uint32_t idesc3 = make_idesc(128, 192, kFmtF16, kFmtF16);
    const uint64_t dIn = make_smem_desc(smem_u32(sIn), 0, 1024, kLayoutSW128);
    const uint64_t dMid = make_smem_desc(smem_u32(sMid), 0, 1024, kLayoutSW128);
    const uint64_t dW0 = make_smem_desc(smem_u32(sW0), 0, 1024, kLayoutSW128);
    const uint64_t dW1 = make_smem_desc(smem_u32(sW1), 0, 1024, kLayoutSW128);
    const bool leader = elect_one();
    pwait(&wbar, 0, 2, 0);
    auto idesc_of = [&](int c) { return c == 3 ? idesc3 : (c == 2 ? idesc2 : idesc1); };
    // One input row r of a layer: targets output rows [max(r-1, lo), min(r+1, hi)]
    // (ring slots seq_lo + (q - lo) mod 4); newly entered rows start with
    // accumulate = 0; rows whose last input row is r are committed.
    auto issue_row = [&](uint32_t ring_col, uint64_t* sfull, uint64_t* sempty, uint32_t seq_lo, int lo, int hi,
                         int r, uint64_t a_row, uint64_t b_base, uint64_t* in_full, uint32_t in_parity,
                         uint64_t* in_empty) {
      const int q_lo = max(r - 1, lo), q_hi = min(r + 1, hi);
      const int q_new = (r == 0) ? q_lo : r + 1;
      for (int q = max(q_new, q_lo); q <= q_hi; ++q) {
        const uint32_t sq = seq_lo + (uint32_t)(q - lo);
        pwait(&sempty[sq & 3], ((sq >> 2) & 1) ^ 1, 3 + (ring_col ? 10 : 0), r);
      }
      pwait(in_full, in_parity, 4 + (ring_col ? 10 : 0), r);
      tc_fence_after();
      if (leader && (ring_col == 0 || !(a.dbg & 2))) {
        const uint32_t s_lo = (seq_lo + (uint32_t)(q_lo - lo)) & 3;
        const int cnt = q_hi - q_lo + 1;
        const int c0 = min(cnt, 4 - (int)s_lo), c1 = cnt - c0;
        auto brow16 = [&](int q) { return (uint32_t)(q - (r - 1)) * (uint32_t)(64 * 128 / 16); };
        const uint32_t R0t = tmem + ring_col + s_lo * 64, R0b = brow16(q_lo), R0i = idesc_of(c0);
        const uint32_t R1t = tmem + ring_col, R1b = brow16(q_lo + c0), R1i = idesc_of(c1);
        const int s0e = q_lo + c0 - 1, s1b = q_lo + c0;
        const int A_e = min(s0e, q_new - 1), B_b = max(q_lo, q_new);
        const int C_e = min(q_hi, q_new - 1), D_b = max(s1b, q_new);
        const bool vA = q_lo <= A_e, vB = B_b <= s0e, vC = c1 > 0 && s1b <= C_e, vD = c1 > 0 && D_b <= q_hi;
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = a_row + (uint64_t)((dx * 128 + k * 32) >> 4);
            const uint64_t bd = b_base + (uint64_t)((dx * 3 * 64 * 128 + k * 32) >> 4);
            if (dx == 0 && k == 0) {
              if (vA) mma_f16_ss(R0t, ad, bd + R0b, idesc_of(A_e - q_lo + 1), 1u);
              if (vB) mma_f16_ss(R0t + (uint32_t)(B_b - q_lo) * 64, ad, bd + brow16(B_b), idesc_of(s0e - B_b + 1), 0u);
              if (vC) mma_f16_ss(R1t, ad, bd + R1b, idesc_of(C_e - s1b + 1), 1u);
              if (vD) mma_f16_ss(R1t + (uint32_t)(D_b - s1b) * 64, ad, bd + brow16(D_b), idesc_of(q_hi - D_b + 1), 0u);
            } else {
              mma_f16_ss(R0t, ad, bd + R0b, R0i, 1u);
              if (c1 > 0) mma_f16_ss(R1t, ad, bd + R1b, R1i, 1u);
            }
          }
        }
        mma_commit(in_empty);
        for (int q = q_lo; q <= q_hi; ++q)
          if (min(q + 1, a.H - 1) == r) mma_commit(&sfull[(seq_lo + (uint32_t)(q - lo)) & 3]);
      } else if (leader) {  // bring-up: layer skipped, keep the protocol
        mma_commit(in_empty);
        for (int q = q_lo; q <= q_hi; ++q)
          if (min(q + 1, a.H - 1) == r) mma_commit(&sfull[(seq_lo + (uint32_t)(q - lo)) & 3]);
      }
      __syncwarp();
    };
    uint32_t seqA = 0, seqB = 0;  // output-row sequences of rings A (= mid rows) and B
    int stage = 0;
    uint32_t phase = 0;
    PairIter it(a, cluster, nclusters);
    PairSeg g;
    while (it.next(a, g)) {
      const int qa0 = max(g.ya - 1, 0), qa1 = min(g.yb, a.H - 1);
      const int ra0 = max(qa0 - 1, 0), ra1 = min(qa1 + 1, a.H - 1);
      int ib = qa0;  // next mid row (layer L+1 input row)
      auto issue_b = [&](int rb) {
        const uint32_t ms = seqA + (uint32_t)(rb - qa0);  // mid-row sequence
        const uint32_t m = ms & 1;
        issue_row(256, bfull, bempty, seqB, g.ya, g.yb - 1, rb, dMid + (uint64_t)((m * kInRowStride) >> 4), dW1,
                  &mfull[m], (ms >> 1) & 1, &mempty[m]);
      };
      for (int ra = ra0; ra <= ra1; ++ra) {
        issue_row(0, afull, aempty, seqA, qa0, qa1, ra, dIn + (uint64_t)((stage * kInRowStride) >> 4), dW0,
                  &full[stage], phase, &empty[stage]);
        if (++stage == kPairRing) { stage = 0; phase ^= 1; }
        while (ib <= qa1 && ib + 2 <= ra) issue_b(ib++);
      }
      while (ib <= qa1) issue_b(ib++);
      seqA += (uint32_t)(qa1 - qa0 + 1);
      seqB += (uint32_t)(g.yb - g.ya);
    }
  } else if (warp < 6) {
    // ------------------------------------------- epilogue L -> mid ring ----
    const int quarter = warp & 3;
    const int px = quarter * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
    const uint32_t shift_u = smem_u32(&sShift[0][0]);
    const uint32_t mid_u = smem_u32(sMid);
    uint32_t seqA = 0;
    PairIter it(a, cluster, nclusters);
    PairSeg g;
    while (it.next(a, g)) {
      const int qa0 = max(g.ya - 1, 0), qa1 = min(g.yb, a.H - 1);
      for (int q = qa0; q <= qa1; ++q, ++seqA) {
        const uint32_t s = seqA & 3, m = seqA & 1;
        pwait(&afull[s], (seqA >> 2) & 1, 5, q);
        tc_fence_after();
        uint32_t v[4][16];
#pragma unroll
        for (int j = 0; j < 4; ++j) tmem_ld16(tmem + lane_addr + s * 64 + j * 16, v[j]);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 4; ++j) reg_fence16(v[j]);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&aempty[s]);
        const bool inside = x0 + px < a.W;
        uint32_t packed[8][4];
#pragma unroll
        for (int chunk = 0; chunk < 8; ++chunk) {
          const float4 s0 = ld_shared_f4(shift_u + chunk * 32);
          const float4 s1 = ld_shared_f4(shift_u + chunk * 32 + 16);
          const float sh[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int c = chunk * 8 + e * 2;
            const float f0 = inside ? fmaxf(__uint_as_float(v[c >> 4][c & 15]) + sh[2 * e], 0.0f) : 0.0f;
            const float f1 = inside ? fmaxf(__uint_as_float(v[c >> 4][(c & 15) + 1]) + sh[2 * e + 1], 0.0f) : 0.0f;
            __half2 hv = __floats2half2_rn(f0, f1);
            packed[chunk][e] = *reinterpret_cast<uint32_t*>(&hv);
          }
        }
        // my mid slot m is free once layer L+1 consumed its previous row
        pwait(&mempty[m], ((seqA >> 1) & 1) ^ 1, 6, q);
        // tell the neighbours they may write their halo pixel into it: use 0 of a
        // slot is free from the start (the waiters' parity convention), so only
        // uses >= 1 are signalled
        if (warp == 2 && lane == 0 && seqA >= 2 && !(a.dbg & 32)) {
          if (has_left) mbar_arrive_remote(mapa_shared(smem_u32(&rfree[m]), rank - 1));
          if (has_right) mbar_arrive_remote(mapa_shared(smem_u32(&lfree[m]), rank + 1));
        }
        const uint32_t row_u = mid_u + m * kInRowStride;
        const int pos = px + 1;  // mid-row position: 0 = x0-1, 1..128 = strip, 129 = x0+128
        if (!(a.dbg & 4))
#pragma unroll
          for (int chunk = 0; chunk < 8; ++chunk)
            st_shared_v4(row_u + pos * 128 + ((chunk ^ (pos & 7)) << 4), packed[chunk][0], packed[chunk][1],
                         packed[chunk][2], packed[chunk][3]);
        // image-edge halo positions are the next layer's zero padding
        if (!has_left && px == 0)
#pragma unroll
          for (int chunk = 0; chunk < 8; ++chunk) st_shared_v4(row_u + ((chunk ^ 0) << 4), 0u, 0u, 0u, 0u);
        if (!has_right && px == 127)
#pragma unroll
          for (int chunk = 0; chunk < 8; ++chunk)
            st_shared_v4(row_u + 129 * 128 + ((chunk ^ (129 & 7)) << 4), 0u, 0u, 0u, 0u);
        // edge pixels -> neighbours' halo positions (129 of the left CTA, 0 of the right CTA)
        if (has_left && px == 0) {
          if (!(a.dbg & 64)) pwait(&lfree[m], ((seqA >> 1) & 1) ^ 1, 7, q);
          const uint32_t rrow = mapa_shared(row_u, rank - 1);
          if (!(a.dbg & 8))
#pragma unroll
            for (int chunk = 0; chunk < 8; ++chunk)
              st_cluster_v4(rrow + 129 * 128 + ((chunk ^ (129 & 7)) << 4), packed[chunk][0], packed[chunk][1],
                            packed[chunk][2], packed[chunk][3]);
          fence_proxy_async_all();
          if (!(a.dbg & 128)) mbar_arrive_remote(mapa_shared(smem_u32(&mfull[m]), rank - 1));
        }
        if (has_right && px == 127) {
          if (!(a.dbg & 64)) pwait(&rfree[m], ((seqA >> 1) & 1) ^ 1, 8, q);
          const uint32_t rrow = mapa_shared(row_u, rank + 1);
          if (!(a.dbg & 8))
#pragma unroll
            for (int chunk = 0; chunk < 8; ++chunk)
              st_cluster_v4(rrow + ((chunk ^ 0) << 4), packed[chunk][0], packed[chunk][1], packed[chunk][2],
                            packed[chunk][3]);
          fence_proxy_async_all();
          if (!(a.dbg & 128)) mbar_arrive_remote(mapa_shared(smem_u32(&mfull[m]), rank + 1));
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&mfull[m]);
      }
    }
  } else {
    // ------------------------------------------ epilogue L+1 -> global ----
    const int quarter = warp & 3;
    const int px = quarter * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
    const uint32_t shift_u = smem_u32(&sShift[1][0]);
    uint32_t seqB = 0;
    PairIter it(a, cluster, nclusters);
    PairSeg g;
    while (it.next(a, g)) {
      for (int q = g.ya; q < g.yb; ++q, ++seqB) {
        const uint32_t s = seqB & 3;
        pwait(&bfull[s], (seqB >> 2) & 1, 9, q);
        tc_fence_after();
        uint32_t v[4][16];
#pragma unroll
        for (int j = 0; j < 4; ++j) tmem_ld16(tmem + lane_addr + 256 + s * 64 + j * 16, v[j]);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 4; ++j) reg_fence16(v[j]);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bempty[s]);
        const int xg = x0 + px;
        if (xg < a.W) {
          uint4* dst = reinterpret_cast<uint4*>(a.act_out + (((long long)g.b * a.H + q) * a.W + xg) * 128);
#pragma unroll
          for (int chunk = 0; chunk < 8; ++chunk) {
            const float4 s0 = ld_shared_f4(shift_u + chunk * 32);
            const float4 s1 = ld_shared_f4(shift_u + chunk * 32 + 16);
            const float sh[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
            uint32_t packed[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int c = chunk * 8 + e * 2;
              const float f0 = fmaxf(__uint_as_float(v[c >> 4][c & 15]) + sh[2 * e], 0.0f);
              const float f1 = fmaxf(__uint_as_float(v[c >> 4][(c & 15) + 1]) + sh[2 * e + 1], 0.0f);
              __half2 hv = __floats2half2_rn(f0, f1);
              packed[e] = *reinterpret_cast<uint32_t*>(&hv);
            }
            dst[chunk] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while a neighbour may still write into its mid ring
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

cudaError_t launch_conv_pair(const CUtensorMap& tm_in, const PairArgs& a, int max_ctas, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(conv3x3_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kPairSmem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int nclusters = std::max(1, max_ctas / a.S);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(nclusters * a.S);
  cfg.blockDim = dim3(kPairThreads);
  cfg.dynamicSmemBytes = kPairSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = a.S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, conv3x3_pair_kernel, tm_in, a);
}

}  // namespace tvs

// bring-up diagnostics of the fused pair kernel (not part of the public ABI)
extern "C" int tvs_debug_pair(int* out8, int reset) {
  if (cudaMemcpyFromSymbol(out8, tvs::g_pair_dbg, 8 * sizeof(int)) != cudaSuccess) return -1;
  if (reset) {
    int z[8] = {0};
    cudaMemcpyToSymbol(tvs::g_pair_dbg, z, sizeof(z));
  }
  return 0;
}
