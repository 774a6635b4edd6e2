// common.cuh — shared constants and small helpers for the TVSpecNET kernels.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <mutex>

namespace tvs {

// Kernel attributes (max dynamic smem, cluster sizes) belong to a device
// context: run `f` once per device ordinal, thread-safely.
template <typename F>
cudaError_t once_per_device(std::mutex& mu, uint64_t& done_mask, F&& f) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && ((done_mask >> dev) & 1ull)) return cudaSuccess;
  e = f();
  if (e == cudaSuccess && dev < 64) done_mask |= 1ull << dev;
  return e;
}

constexpr int kC = 64;            // hidden feature maps (ARCH_SPEC["channels"], model.py:19-26)
constexpr int kStripPx = 128;     // output pixels per strip = tcgen05 M
constexpr int kHaloPx = kStripPx + 2;
constexpr int kInRowBytes = kHaloPx * kC * 2;          // 16640: one halo'd input row, fp16 NHWC
constexpr int kInRowStride = 17408;                    // 1024-aligned ring stride (17 KB)
constexpr int kSlots = 8;                              // TMEM accumulator slots (one per output row)
// B operand pack (fp16, SW128 K-major rows of 64 input channels): for dx block
// kx, row n = dyslot*NB + j with dyslot = 2 - ky (dy=+1 -> 0, 0 -> 1, -1 -> 2),
// byte = kx*3*NB*128 + n*128 + ((ci/8) ^ (n&7))*16 + (ci%8)*2.

// tcgen05 conv kernels (conv_tc.cu)
constexpr int kStages = 6;             // input-row ring depth
constexpr int kEpiGroups = 3;          // epilogue row groups (output row seq % 3)
#ifndef TVS_EPI_GROUPS_PLAIN
#define TVS_EPI_GROUPS_PLAIN 3
#endif
#ifndef TVS_WIDE_MCAST
#define TVS_WIDE_MCAST 0
#endif
#ifndef TVS_STAGES_PLAIN
#define TVS_STAGES_PLAIN 6
#endif
constexpr int kEpiGroupsPlain = TVS_EPI_GROUPS_PLAIN;  // modes 0 / 8
constexpr int kStagesPlain = TVS_STAGES_PLAIN;
static_assert(kStagesPlain <= kStages, "barrier arrays are sized by kStages");

// Device-side duration of one kernel launch (plan option "span"): every CTA
// reduces the globaltimer after its PDL wait (so spans of dependent launches
// on one stream never overlap) into `start` and at exit into `end`, with
// fire-and-forget atomics; the host sums end - start over the launch records.
struct KernelSpan {
  unsigned long long start;  // ~0 when armed
  unsigned long long end;
};
// status flag store (host-mapped memory: plain stores, no system-scope atomics)
__device__ __forceinline__ void flag_set(int* p) { *(volatile int*)p = 1; }

// Fused band-sum reconstruction check (north_star item 3; the closure identity
// of inference.py:34-42 / pkg/trainer/tests/test_inference.py:31-38): every
// head epilogue that writes the closure plane c = x - sum_k b_k also evaluates
// r = x - (sum_k b_k + c) from the values it stores and adds r^2 and x^2 (fp64)
// to recon[2b], recon[2b+1].  Called by all 32 lanes of a warp (lanes without
// a pixel pass r = x = 0); one pair of atomics per warp and row.
__device__ __forceinline__ void recon_accumulate(double* recon, int b, float r, float x) {
  double r2 = (double)r * (double)r, x2 = (double)x * (double)x;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    x2 += __shfl_xor_sync(0xffffffffu, x2, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(recon + 2 * b, r2);
    atomicAdd(recon + 2 * b + 1, x2);
  }
}

struct ConvArgs {
  int B, H, W;
  int strips;            // ceil(W / 128)
  int row0, rows;        // output rows computed: [row0, row0 + rows)
  const uint8_t* wpack;  // packed fp16 B operand (SW128)
  const float* shift;    // per output channel (hidden: beta - mu*s; head: conv bias)
  int nshift;
  // head only
  const float* x;        // (B,1,H,W) input plane for the closure
  float* bands;          // (B,K,rows,W)
  float* closure;        // (B,1,rows,W) or null
  double* recon;         // null, or (B,2) fused reconstruction check sums (recon_accumulate)
  int K;
  // fp32-accurate split hidden layer: output fp16 pair rows [B][H][W][hi 64 | lo 64]
  uint8_t* act_out;
  // layer-stack kernel (conv_tc.cu mode 8): all `nlayers` hidden layers in one
  // persistent launch; wpack / shift hold every layer back to back and
  // rowcnt[(b*strips + s)*H + y] counts the epilogue warps (4 per layer) that
  // have stored output row y of strip s of image b
  int out_single;  // wide hidden (modes 5 / 9): write single fp16 output instead of the hi/lo pair
  int nlayers;
  int* rowcnt;
  // work items {image, layer << 16 | strip, first row, end row} (image -1:
  // padding, skipped) in a topological order, CTA i taking entries i, i+G, ...
  const int4* items;
  int nitems;
  // head after a layer stack (mode 1): > 0 = gate every input row on the
  // stack's row flags (rowcnt >= gate_target) instead of waiting for the
  // whole stack grid (griddepcontrol.wait), so the head runs on the SMs the
  // stack's CTAs free at its tail
  int gate_target;
  int watcher;  // layer stack: a dedicated warp polls the row flags (conv_tc.cu StackWatcher)
  // per-image input exponent e_b (tvs_api.cu, input_scale_kernel): the
  // activations of image b are computed as 2^-e_b times the model's (exact:
  // ReLU commutes with powers of two), keeping them inside the fp16 range.
  // Hidden epilogues scale the BN shift by 2^-e_b, heads rescale by 2^e_b.
  // Null = no scaling.
  const int* escale;
  // per-forward status words (kStat*): a slot of pinned, mapped host memory
  // the host zeroes before the forward (kernels only ever store 1 into it)
  int* status;
  int* abort;  // layer stack: device word set when a watchdog fired (zeroed with rowcnt)
  // training (train.cu): modes 0 / 3 write the raw fp32 accumulator (no
  // shift, no ReLU) as fp32 NHWC [B][H][W][64] to act_out, times 2^-(*out_exp)
  // when out_exp is set (the dgrad conv undoes its input's gradient scale)
  int raw_f32;
  const int* out_exp;
  // wide fp32-accurate mode (tvs_api.cu, 128 channels as 2 x 2 blocks of the
  // 64-channel split kernels): a hidden launch on the second input block adds
  // the first block's raw fp32 partial sums acc_in [B][H][W][64] before the
  // shift and ReLU; a head launch with acc_bands adds the bands already in
  // `bands` (the first block's partial output)
  const float* acc_in;
  int acc_bands;
  // training forward (mode 13, raw_f32): per-channel batch sums of the raw
  // output, [0, 64) sum y and [64, 128) sum y^2 (fp64, zeroed by the host): the
  // epilogue reduces each row across the warp's 32 pixels and every lane
  // carries one channel, so BatchNorm's statistics need no pass over y
  double* bn_sums;
  unsigned long long watchdog_ns;  // layer stack: give up a row-flag wait after this long
  KernelSpan* span;                // null, or accumulate this launch's device duration
  // TVS_CONV_DBG / plan option "debug" (results invalid except kDbgWithholdFlag,
  // which exercises the watchdog): 1 no stack flag waits, 16 epilogue skips its
  // work, 32 no input loads, 64 no MMAs, ... (conv_tc.cu)
  int dbg;
};
// status words (ConvArgs::status)
constexpr int kStatWatchdog = 0;    // a layer-stack row-flag wait expired: that forward's output is invalid
constexpr int kStatNonFiniteOut = 1;  // a head wrote a NaN / Inf band value
constexpr int kStatNonFiniteIn = 2;   // the input held NaN / Inf (the reference propagates them)
constexpr int kStatWords = 4;
constexpr int kDbgWithholdFlag = 1 << 17;
constexpr int kDbgTrace = 1 << 19;
constexpr int kDbgNoStoreWait = 1 << 20;  // ablation: stack publishes a row without its store-completion wait (invalid)
constexpr int kDbgSpinGate = 1 << 21;     // ablation: StackGate polls without __nanosleep  // stack: globaltimer per row of image 0 strip 0 (g_trace, tvs_debug_trace)
constexpr int kDbgNoPdlStack = 1 << 18;     // launch the stack without programmatic serialization  // stack: never publish row 1 of (image 0, strip 0, layer 2)
// 2^k as an exact fp32 (|k| <= 126)
__host__ __device__ __forceinline__ float pow2i(int k) {
  union { unsigned u; float f; } v;
  v.u = (unsigned)(127 + k) << 23;
  return v.f;
}
// per-image scale factor 2^-e (1 when the plan does not scale)
__device__ __forceinline__ float image_scale(const int* escale, int b) { return escale ? pow2i(-__ldg(escale + b)) : 1.0f; }
// Second pair of tensor maps of the layer-stack kernel (layer j reads buffer j&1
// and writes buffer (j+1)&1; tm_in / tm_out cover buffer 0 input / buffer 1 output)
struct StackMaps {
  CUtensorMap in1;   // buffer 1, 130-px halo rows
  CUtensorMap out0;  // buffer 0, 32-px store boxes
};
cudaError_t launch_conv_stack(const CUtensorMap& tm_in0, const CUtensorMap& tm_out1, const StackMaps& sm,
                              const ConvArgs& a, int grid, cudaStream_t st);
// the stack kernel can run on this device: cooperative launch supported and
// one CTA per SM fits (all `grid` CTAs co-resident)
bool conv_stack_fits(int num_sms, int grid);
int debug_cycles(unsigned long long* out, int reset);  // TVS_CONV_DBG bit 15 counters
int debug_trace(unsigned long long* out, int reset);   // kDbgTrace row timeline

// fp32 hidden layer (conv_edge.cu)
constexpr int kF32TileRows = 4, kF32TilePx = 32, kF32CiChunk = 16;
constexpr int kF32InRows = kF32TileRows + 2, kF32InPx = kF32TilePx + 2;
constexpr size_t f32_smem(int C) { return (size_t)(kF32InRows * kF32InPx * kF32CiChunk + kF32CiChunk * 9 * C) * 4; }
constexpr int kMaxC = 128;  // channels supported by the CUDA-core (fp32) path
constexpr int kMaxBands = 8;

// host-side launchers (defined next to their kernels)
size_t conv_wpack_bytes(bool head);
size_t conv_wpack_split_bytes();  // fp32-accurate hidden layer: hi pack | lo pack
size_t conv_wpack_wide_bytes(bool head);  // wide variant (128 ch) on tcgen05: 4 quarter packs / head pack
size_t conv_wpack_unshuf_head_bytes();    // unshuffle = 2 variant: Conv2d(64, 4K) head pack
cudaError_t launch_pack_head_unshuf(const float* w, int K4, uint8_t* out, cudaStream_t st);
// unshuffle = 2: Conv2d(4, 64) + ReLU over pixel_unshuffle(x, 2); H, W = half-res grid
cudaError_t launch_conv0_unshuffle(const float* x, void* act, const float* w, const float* b, const int* escale, int B,
                                   int H, int W, cudaStream_t st);
struct Conv0Params;
cudaError_t launch_conv_tc(int mode, const CUtensorMap& tm_in, const CUtensorMap& tm_out, const ConvArgs& a,
                           int grid, cudaStream_t st);
cudaError_t launch_pack_hidden_f16(const float* w, const float* scale, uint8_t* out, cudaStream_t st);
// (cin, co0, ci0): pack the 64 x 64 block at output channel co0, input channel
// ci0 of a [Cout][cin][3][3] weight (the wide fp32 mode's 2 x 2 blocks)
cudaError_t launch_pack_hidden_split(const float* w, const float* scale, uint8_t* out, cudaStream_t st, int cin = 64,
                                     int co0 = 0, int ci0 = 0);
cudaError_t launch_pack_hidden_f16_t(const float* w, uint8_t* out, cudaStream_t st);  // training dgrad pack
cudaError_t launch_pack_head_f16_t(const float* w, int K, uint8_t* out, cudaStream_t st);  // training head dgrad pack
// training step: split (forward) + transposed fp16 (dgrad) packs of n hidden layers, one launch per 32 layers
constexpr int kTrainPackLayers = 32;
struct TrainPackPtrs { const float* w[kTrainPackLayers]; };
cudaError_t launch_train_pack_hidden(const float* const* w_dev, int n, uint8_t* wsplit, uint8_t* wt, cudaStream_t st);
// training wgrad on tcgen05 (wgrad_tc.cu): dW = alpha * sum_p G[p] (x) A[p + tap offset] over the
// zero-bordered pixel list; `part` holds wgrad_part_bytes(num_sms) of split-K partials
size_t wgrad_part_bytes(int num_sms);
CUtensorMap make_wgrad_gmap(const void* base, long long rows);  // [rows][64] fp16 gradient operand
CUtensorMap make_wgrad_amap(const void* base, long long rows);  // [rows][128] fp16 pair activations (hi half read)
cudaError_t launch_wgrad_tc(const CUtensorMap& gmap, const CUtensorMap& amap, long long PP, int guard, int W,
                            int rows, const float* alpha, float* part, float* dw, int num_sms, cudaStream_t st);
// parts = 4: output-channel quarters (modes 5 / 9); 2: halves (mode 11)
cudaError_t launch_pack_hidden_wide(const float* w, const float* scale, uint8_t* out, cudaStream_t st, int parts,
                                    bool lo8);
cudaError_t launch_pack_head_wide(const float* w, int K, uint8_t* out, cudaStream_t st);
cudaError_t launch_pack_head_f16(const float* w, int K, uint8_t* out, cudaStream_t st, int cin = 64, int ci0 = 0);
cudaError_t launch_fill(float* dst, float v, int n, cudaStream_t st);
struct Conv0Params {  // passed by value: lives in the kernel's constant bank
  float w[kMaxC * 9];  // [co][ky*3+kx]
  float b[kMaxC];
};
// act_fmt: 0 = fp16 NHWC, 1 = fp32 NHWC, 2 = fp16 hi/lo pair NHWC (4*C bytes/px: hi C | lo C)
constexpr int kActF16 = 0, kActF32 = 1, kActSplit = 2;
cudaError_t launch_conv0(int act_fmt, int C, const float* x, void* act, const Conv0Params& p, const int* escale,
                         int B, int H, int W, cudaStream_t st);
// per-image input exponents: e_b = 0 while the conv0 output bound
// M_b = max|x_b| * w0_l1 + b0_max lies in [2^-6, 2^6], else round(log2 M_b) - 2;
// counts non-finite inputs into status[kStatNonFiniteIn]
cudaError_t launch_input_scale(const float* x, int B, long long px_per_image, float w0_l1, float b0_max, int* escale,
                               int* scratch, int* status, cudaStream_t st);
// the input-scale kernel's scratch: 2 * B ints, zero on first use; the kernel
// leaves it zeroed for the next forward
cudaError_t launch_head_f32(int C, const float* act, const float* x, const float* wh, const float* bh, float* bands,
                            double* recon,
                            float* closure, int B, int H, int W, int K, int row0, int rows, int* status,
                            cudaStream_t st);
cudaError_t launch_hidden_f32(int C, const float* in, float* out, const float* w, const float* scale,
                              const float* shift, int B, int H, int W, cudaStream_t st);
cudaError_t configure_kernels();  // one-time smem opt-ins
// conv0_tc.cu: K1 on tcgen05 (fast path, fp16 NHWC output), TF32 hi/lo split;
// in_ch = 1 (reference conv0) or 4 (unshuffle = 2 variant, H/W = half-res grid)
size_t conv0_tc_pack_bytes(int in_ch);
cudaError_t launch_pack_conv0_tc(const float* w, int in_ch, uint8_t* out, cudaStream_t st);
// pdl: launched programmatically after the input-scale kernel (x may be read
// before griddepcontrol.wait; escale and the activation writes come after it)
cudaError_t launch_conv0_tc(int in_ch, const float* x, const CUtensorMap& out_map, const uint8_t* bpack,
                            const float* bias, const int* escale, int B, int H, int W, int num_sms, bool pdl,
                            cudaStream_t st);
// metrics.cu: per-plane scoring statistics (8 doubles per plane)
cudaError_t launch_band_stats(const float* gt, const float* pred, int planes, int H, int W,
                              const double* range_override, double* stats, cudaStream_t st);
// tvflow.cu: model-driven TV-flow decomposition (ground-truth producer)
constexpr int kTvMaxW = 2048;
constexpr int kTvMaxBands = 16;
struct TvFlowArgs {
  int N, H, W;
  double dt;
  int n_steps, n_bands;
  int schedule[kTvMaxBands];  // inclusive band end indices on the fine grid 1..n_steps-1
  int max_iters, accel;
  double gap_tol, tau0, sigma0;
  const double* f;   // (N, H, W)
  double* work;      // (N, 6, H, W): three rotating flow states, vbar, qx, qy
  double* bands;     // (N, n_bands, H, W)
  double* spectrum;  // (N, n_steps-1)
  double* residual;  // (N, H, W)
  int* iters;        // (N, n_steps), -(iters+1) when not certified
};
cudaError_t launch_tvflow(const TvFlowArgs& a, cudaStream_t st);

}  // namespace tvs
