// tvs_api.cu — host runtime behind include/tvs_b200.h: plans, packed
// weights, TMA descriptors, activation scratch and the per-layer launch
// sequence.  See DESIGN.md for the data layout.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>

#include <nvtx3/nvToolsExt.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <array>
#include <cmath>
#include <deque>
#include <vector>

#include "../../include/tvs_b200.h"
#include "common.cuh"
#include "host_util.h"


namespace tvs_host {
std::string& last_error() {
  thread_local std::string msg;
  return msg;
}
}  // namespace tvs_host

using tvs_host::DeviceGuard;
using tvs_host::TvsError;
using tvs_host::get_encode;
using tvs_host::guarded;
using tvs_host::make_act_map;

struct tvs_plan {
  int device = 0, depth = 17, channels = 64, out_bands = 5, mode = TVS_MODE_FAST;
  int num_sms = 148;
  bool weights_ready = false;

  // Plan options (tvs_plan_set_option).  The defaults are the
  // measured-best settings; the rest exist so a maintainer can A/B a design
  // choice.  Options marked (pack) change the weight layout and take effect at
  // the next tvs_plan_set_weights.
  struct Options {
    int stack = -1;             // layer stack K4: -1 auto (item-rich chunks), 0 off, 1 whenever legal
    int stack_band_rows = 0;    // layer-stack item height: 0 auto, R > 0 rows per item (>= H: whole columns)
    int stack_skew = 1;         // layer-stack row bands: layer j's band edges sit at j*skew mod R
    int head_gate = 1;          // head after a stack: gate rows on the stack's flags (runs in the stack's tail)
    int head_grid = 4;          // gated head: CTAs per SM of its grid (tools/ab.py: 4 best, -1.5%)
    int stack_watcher = 1;      // layer stack: a dedicated warp polls the row flags
    int fp32_pairs = 1;         // fp32-accurate hidden layers on CTA pairs (mode 12) instead of mode 3
    int conv0_tc = 1;           // K1 on tcgen05 (TF32 hi/lo) instead of the CUDA-core K1
    int wide_pair_layers = 12;  // (pack) wide variant: leading hidden layers on fp16 hi/lo pairs
    int wide_halves = 1;        // (pack) wide single-input layers on output-channel halves (mode 11)
    int fp32_cuda = 0;          // (pack) fp32 mode on the CUDA-core fp32 kernels
    int wide_cuda = 0;          // (pack) wide variant on the CUDA-core fp32 kernels
    long long chunk_mb = 16384;  // activation budget per batch chunk (x2 ping-pong); lazily sized to the batch
    int check = 1;              // per-forward status: 0 off, 1 synchronous, 2 deferred (tvs_plan_sync)
    int watchdog_ms = 2000;     // layer-stack row-flag wait limit
    int input_scale = 1;        // per-image power-of-two activation scale (fp16 range guard)
    int span = 0;               // accumulate the hidden-layer kernels' device spans (tvs_profile_span)
    int debug = 0;              // kernel debug/ablation bits (ConvArgs::dbg)
  } opt;

  // conv0 [64][1][3][3] + bias, head [K][64][3][3] + bias (fp32, folded)
  tvs::Conv0Params conv0{};  // host copy, passed by value to the CUDA-core K1
  tvs::Conv0Params conv0_blk[2]{};  // wide fp32 mode: the two 64-output-channel blocks of conv0
  float w0_l1 = 0.f, b0_max = 0.f;  // input-scale bound: max_co sum|W0|, max|b0|
  float* wh = nullptr;
  float* bh = nullptr;
  // hidden: packed per path (see set_weights); head packs
  uint8_t* wpack = nullptr;
  uint8_t* hpack = nullptr;
  // opt-in unshuffle = 2 variant: conv0 Conv2d(4, 64) weights on the device
  int unshuffle = 1;
  float* w0u = nullptr;
  float* b0u = nullptr;
  float* whid = nullptr;
  float* bhid = nullptr;  // per hidden layer: shift (beta - mu*s)
  float* shid = nullptr;  // per hidden layer: BatchNorm scale s (fp32 mode epilogue; folded in FAST)
  uint8_t* c0pack = nullptr;  // K1 on tcgen05: packed TF32 hi/lo B operand
  float* c0bias = nullptr;
  // the path the packed weights were built for (options may change later)
  bool packed_tc = false, packed_split = false, packed_wide = false, packed_wide_split = false;
  int packed_pairs = 12, packed_halves = 1;

  // activation ping-pong scratch
  void* act[2] = {nullptr, nullptr};
  size_t act_bytes = 0;
  // wide fp32 mode: raw fp32 partial sums of one 64-channel output block
  void* act_raw = nullptr;
  size_t act_raw_bytes = 0;
  // device records of the hidden-layer launches (option "span"), one per launch
  static constexpr int kSpanSlots = 8192;
  tvs::KernelSpan* span = nullptr;
  int span_next = 0;
  // per-image input exponents
  int* escale = nullptr;
  size_t escale_n = 0;
  // per-forward status words (tvs::kStat*): a ring of slots in pinned, mapped
  // host memory that the kernels write directly (no per-forward memset or copy)
  static constexpr int kRing = 32;
  int* status_host = nullptr;  // kRing x kStatWords
  int* status_dev = nullptr;   // the same memory, device view
  cudaEvent_t status_ev[kRing] = {};
  int status_next = 0;
  std::deque<int> status_pending;  // deferred mode: slots not yet evaluated
  // host-API staging
  float* dx = nullptr;  // [x | bands | closure] staging for tvs_forward_host
  size_t io_bytes = 0;
  int last_launches = 0;
  int last_stack = 0;  // the last forward ran the layer stack
  // optional per-kernel event timing
  struct Rec { cudaEvent_t a, b; int kind; double flops; };
  bool profiling = false;
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> event_pool;
  double prof_ms[3] = {0, 0, 0};
  long long prof_n[3] = {0, 0, 0};
  double prof_flops[3] = {0, 0, 0};
  // layer stack: co-residency verified for this device (cooperative launch,
  // occupancy); cleared if the driver ever refuses the cooperative launch
  bool stack_ok = false;
  static constexpr int kStackMinItems = 6;
  static constexpr int kStackMaxColH = 1024;
  // row-band stack items (auto): images at least kStackMinBandH tall whose
  // per-layer launches give each SM at most kBandMaxRowsPerSm strip-rows
  static constexpr int kStackMinBandH = 128;
  static constexpr double kBandMaxRowsPerSm = 8.0;
  static constexpr int kStackBandRows = 6;
  int* rowcnt = nullptr;  // row flags (B*strips*H ints), zeroed per chunk
  size_t rowcnt_n = 0;
  // work-item tables per (B, strips, layers, bands, order), uploaded once and
  // never overwritten (a running stack kernel may be reading an older one)
  struct Items { long long key[6]; int4* dev; int4* host; size_t n; };
  std::vector<Items> items;

  int n_hidden() const { return depth - 2; }
  // tcgen05 fp16 path: FAST mode with 64 channels
  bool tc_path() const { return mode == TVS_MODE_FAST && channels == 64; }
  // fp32-accurate mode on tcgen05 with split fp16 operands (conv_tc.cu modes 3/4)
  bool split_path() const { return mode == TVS_MODE_FP32 && channels == 64 && !opt.fp32_cuda; }
  // wide variant (128 channels) fast mode on tcgen05 (modes 5/6/9/10/11)
  bool wide_path() const { return mode == TVS_MODE_FAST && channels == 128 && !opt.wide_cuda; }
  // wide variant, fp32-accurate mode on tcgen05: every 128 -> 128 layer as 2 x 2
  // blocks of the 64-channel split kernels (modes 12 / 3 / 4), activations as two
  // 64-channel hi|lo pair planes
  bool wide_split_path() const {
    return mode == TVS_MODE_FP32 && channels == 128 && !opt.fp32_cuda && !opt.wide_cuda;
  }
  size_t act_px_bytes() const { return tc_path() ? 128 : (size_t)channels * 4; }
  // the power-of-two input scale guards the fp16-range formats (fast, split,
  // wide); the CUDA-core fp32 kernels compute at fp32 range and do not need it
  bool scaled() const {
    return opt.input_scale && (tc_path() || split_path() || wide_path() || wide_split_path());
  }
};

namespace {


void free_weights(tvs_plan* p) {
  void* ptrs[] = {p->wh, p->bh, p->wpack, p->hpack, p->whid, p->bhid, p->shid, p->w0u, p->b0u, p->c0pack, p->c0bias};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  p->wh = p->bh = p->whid = p->bhid = p->shid = p->w0u = p->b0u = p->c0bias = nullptr;
  p->wpack = p->hpack = p->c0pack = nullptr;
  p->weights_ready = false;
}

void free_all(tvs_plan* p) {
  for (auto& r : p->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : p->event_pool) cudaEventDestroy(e);
  p->recs.clear();
  p->event_pool.clear();
  for (auto& it : p->items) { cudaFree(it.dev); cudaFreeHost(it.host); }
  p->items.clear();
  for (auto& e : p->status_ev)
    if (e) cudaEventDestroy(e);
  if (p->status_host) cudaFreeHost(p->status_host);
  free_weights(p);
  void* ptrs[] = {p->act[0], p->act[1], p->act_raw, p->dx, p->rowcnt, p->escale, p->span};
  for (void* q : ptrs)
    if (q) cudaFree(q);
}

void ensure_act(tvs_plan* p, size_t bytes) {
  if (bytes <= p->act_bytes) return;
  for (int i = 0; i < 2; ++i) {
    if (p->act[i]) TVS_CUDA(cudaFree(p->act[i]));
    p->act[i] = nullptr;
  }
  p->act_bytes = 0;
  for (int i = 0; i < 2; ++i) TVS_CUDA(cudaMalloc(&p->act[i], bytes));
  p->act_bytes = bytes;
}

void ensure_raw(tvs_plan* p, size_t bytes) {
  if (bytes <= p->act_raw_bytes) return;
  if (p->act_raw) TVS_CUDA(cudaFree(p->act_raw));
  p->act_raw = nullptr;
  p->act_raw_bytes = 0;
  TVS_CUDA(cudaMalloc(&p->act_raw, bytes));
  p->act_raw_bytes = bytes;
}

// Work items of the layer-stack kernel (conv_tc.cu ItemIter) for a chunk of B
// images, `strips` strips, L hidden layers and H rows, image-major, then
// layer, then row band, then strip: an item only depends on layer j-1 items of
// its image, which sort before it.  CTA i runs entries i, i+G, ... in table
// order, so every CTA's sequence is topologically sorted too.
//
// Row bands (R < H) are skewed: layer j's band edges sit at rows congruent to
// j*skew (mod R).  A band [a, a+R) of layer j then reads rows a-1 .. a+R of
// layer j-1, which are rows skew-1 and skew of two layer j-1 bands: both are
// produced early in those items, so every layer trails the one before it by a
// few rows.  With aligned edges (skew 0) row a-1 is the LAST row of the band
// above, and band k of layer j could only start once band k-1 of layer j-1 had
// finished: a diagonal wavefront costing a whole band per layer
// (tools/stack_trace.py).
const int4* stack_items(tvs_plan* p, int B, int strips, int L, int H, int R, int skew, cudaStream_t st,
                        size_t* n_out) {
  const long long key[6] = {B, strips, L, H, R, skew};
  for (auto& it : p->items)
    if (std::equal(key, key + 6, it.key)) {
      *n_out = it.n;
      return it.dev;
    }
  std::vector<int4> v;
  for (int i = 0; i < B; ++i)
    for (int j = 0; j < L; ++j) {
      const int s0 = R < H ? (int)(((long long)j * skew) % R) : 0;  // first band edge below row 0
      for (int ya = 0; ya < H;) {
        const int yb = std::min(H, ya == 0 && s0 > 0 ? s0 : ya + R);
        for (int s = 0; s < strips; ++s) v.push_back(make_int4(i, j << 16 | s, ya, yb));
        ya = yb;
      }
    }
  tvs_plan::Items it{{key[0], key[1], key[2], key[3], key[4], key[5]}, nullptr, nullptr, v.size()};
  TVS_CUDA(cudaMallocHost(&it.host, v.size() * sizeof(int4)));
  std::copy(v.begin(), v.end(), it.host);
  if (cudaMalloc(&it.dev, v.size() * sizeof(int4)) != cudaSuccess) {
    cudaFreeHost(it.host);
    throw TvsError(TVS_E_CUDA, "cudaMalloc of the layer-stack item table failed");
  }
  TVS_CUDA(cudaMemcpyAsync(it.dev, it.host, v.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
  p->items.push_back(it);
  *n_out = it.n;
  return it.dev;
}

int conv_grid(int max_ctas, const tvs::ConvArgs& a) {
  const long long total = (long long)a.B * a.strips * a.rows;
  return (int)std::max(1LL, std::min<long long>(max_ctas, (total + 2) / 3));
}

cudaEvent_t pool_event(tvs_plan* p) {
  if (!p->event_pool.empty()) {
    cudaEvent_t e = p->event_pool.back();
    p->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  TVS_CUDA(cudaEventCreate(&e));
  return e;
}

// Launch `f` bracketed by events when profiling is on.
// NVTX ranges (SURVEY §5 tracing): one host range per forward and per kernel
// launch, visible in Nsight Systems / ncu --nvtx; no-ops without a tool
// attached (NVTX v3 is header-only and injection-based).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
const char* kind_name(int kind) {
  return kind == TVS_KIND_CONV0 ? "tvs.conv0" : (kind == TVS_KIND_HIDDEN ? "tvs.hidden" : "tvs.head");
}

template <typename F>
void timed_launch(tvs_plan* p, cudaStream_t st, int kind, double flops, F&& f) {
  NvtxRange nr(kind_name(kind));
  if (!p->profiling) {
    TVS_CUDA(f());
    p->last_launches++;
    return;
  }
  tvs_plan::Rec r{pool_event(p), pool_event(p), kind, flops};
  TVS_CUDA(cudaEventRecord(r.a, st));
  TVS_CUDA(f());
  TVS_CUDA(cudaEventRecord(r.b, st));
  p->recs.push_back(r);
  p->last_launches++;
}

void drain_profile(tvs_plan* p) {
  for (auto& r : p->recs) {
    TVS_CUDA(cudaEventSynchronize(r.b));
    float ms = 0.f;
    TVS_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    p->prof_ms[r.kind] += ms;
    p->prof_n[r.kind] += 1;
    p->prof_flops[r.kind] += r.flops;
    p->event_pool.push_back(r.a);
    p->event_pool.push_back(r.b);
  }
  p->recs.clear();
}

void run_chunk(tvs_plan* p, const float* x, float* bands, float* closure, int B, int H, int W, int row0, int rows,
               cudaStream_t st, const int* escale, int* status, bool conv0_pdl, double* recon) {
  void* const* act = p->act;
  const int max_ctas = p->num_sms;
  const bool fast = p->tc_path();
  const bool split = p->split_path();
  const bool wide = p->wide_path();
  const bool wsplit = p->wide_split_path();
  const int C = p->channels;
  const double px = (double)B * H * W;
  // wide fp32 mode: act[i] holds two 64-channel pair planes of the chunk
  const size_t plane_bytes = (size_t)B * H * W * 256;
  auto plane = [&](int buf, int blk) { return static_cast<uint8_t*>(act[buf]) + (size_t)blk * plane_bytes; };
  const int us = p->unshuffle;  // 2: the layer stack runs on the (H/2, W/2) grid
  // layer stack (FAST path): all CTAs of the persistent grid co-resident
  // (cooperative launch, verified at plan creation)
  bool stack = false;
  const int Hs = H / us, strips_s = (W / us + tvs::kStripPx - 1) / tvs::kStripPx;
  const long long stack_cols = (long long)B * strips_s * p->n_hidden();  // whole-column items
  int band_rows = Hs;  // rows per stack item
  if (fast && p->opt.stack != 0 && p->stack_ok && strips_s < 65536 && p->n_hidden() < 32768) {
    // auto: enough whole-column items per SM with a nearly full last round
    // (equal-length items; a partial round idles SMs), else row-band items
    // when the image is tall enough to cut (batch-1 latency: the reference's
    // own calling pattern, inference.py:25-32)
    const long long rounds = (stack_cols + p->num_sms - 1) / p->num_sms;
    // (columns taller than kStackMaxColH keep the per-layer kernels: with
    // 2160-row columns the layers drift apart and the hand-off misses L2;
    // config 4 measured 945 vs 965 MP/s, tools/ab.py chunk_mb=120000)
    const bool columns = stack_cols >= (long long)tvs_plan::kStackMinItems * p->num_sms &&
                         (double)stack_cols >= 0.95 * (double)(rounds * p->num_sms) && Hs <= tvs_plan::kStackMaxColH;
    // row bands: when the per-layer kernels would give each SM only a few
    // strip-rows per layer (batch 1 at 256^2: 3.5), the 15 launches are
    // latency-bound and a row-band stack wins (tools/stack_sweep.py: 4-8-row
    // bands with skew 1 best on config 1, 6% under the per-layer kernels;
    // config 3 at 55 rows per SM per layer is faster per layer)
    const double rows_per_sm = (double)B * strips_s * Hs / p->num_sms;
    const bool few_rows = rows_per_sm <= tvs_plan::kBandMaxRowsPerSm && Hs >= tvs_plan::kStackMinBandH;
    if (p->opt.stack_band_rows > 0)
      band_rows = std::min(Hs, p->opt.stack_band_rows);
    else if (!columns && (few_rows || p->opt.stack == 1) && Hs > tvs_plan::kStackBandRows)
      band_rows = tvs_plan::kStackBandRows;
    const bool banded = band_rows < Hs;
    stack = p->opt.stack == 1 || columns || (banded && few_rows);
  }
  const int stack_nbands = (Hs + band_rows - 1) / band_rows + (band_rows < Hs ? 1 : 0);
  const int stack_grid = (int)std::min<long long>(p->num_sms, stack_cols * stack_nbands);
  if (stack) {
    // row flags + the watchdog's abort word, zeroed per launch
    const size_t n = (size_t)B * ((W / us + tvs::kStripPx - 1) / tvs::kStripPx) * (H / us) + 1;
    if (n > p->rowcnt_n) {
      if (p->rowcnt) TVS_CUDA(cudaFree(p->rowcnt));
      p->rowcnt = nullptr;
      p->rowcnt_n = 0;
      TVS_CUDA(cudaMalloc(&p->rowcnt, n * sizeof(int)));
      p->rowcnt_n = n;
    }
    TVS_CUDA(cudaMemsetAsync(p->rowcnt, 0, n * sizeof(int), st));
    conv0_pdl = false;  // the memset sits between the input-scale kernel and K1
  }
  // K1
  // wide fast stack: hidden layer j reads an fp16 hi / e4m3 lo pair for j < P,
  // single fp16 after; the head (j == n_hidden) always reads single fp16
  const int nh = p->n_hidden();
  const int P = std::max(0, std::min(p->packed_pairs, nh));
  auto pair_in = [&](int j) { return j < P && j < nh; };
  const int fmt = fast ? tvs::kActF16
                       : (split ? tvs::kActSplit : (wide ? (pair_in(0) ? tvs::kActSplit : tvs::kActF16) : tvs::kActF32));
  if (us == 2 && p->opt.conv0_tc)
    timed_launch(p, st, TVS_KIND_CONV0, px * 2.0 * 9 * C, [&] {
      return tvs::launch_conv0_tc(4, x, make_act_map(act[0], B, H / 2, W / 2, 128), p->c0pack, p->c0bias, escale, B,
                                  H / 2, W / 2, p->num_sms,
                                  conv0_pdl, st);
    });
  else if (us == 2)
    timed_launch(p, st, TVS_KIND_CONV0, px * 2.0 * 9 * C,
                 [&] { return tvs::launch_conv0_unshuffle(x, act[0], p->w0u, p->b0u, escale, B, H / 2, W / 2, st); });
  else if (fast && p->opt.conv0_tc)
    timed_launch(p, st, TVS_KIND_CONV0, px * 2.0 * 9 * C, [&] {
      return tvs::launch_conv0_tc(1, x, make_act_map(act[0], B, H, W, 128), p->c0pack, p->c0bias, escale, B, H, W,
                                  p->num_sms, conv0_pdl, st);
    });
  else if (wsplit)
    for (int o = 0; o < 2; ++o)
      timed_launch(p, st, TVS_KIND_CONV0, px * 2.0 * 9 * 64, [&] {
        return tvs::launch_conv0(tvs::kActSplit, 64, x, plane(0, o), p->conv0_blk[o], escale, B, H, W, st);
      });
  else
    timed_launch(p, st, TVS_KIND_CONV0, px * 2.0 * 9 * C,
                 [&] { return tvs::launch_conv0(fmt, C, x, act[0], p->conv0, escale, B, H, W, st); });
  // one span record per hidden-layer launch (option "span")
  auto next_span = [&]() -> tvs::KernelSpan* {
    return (p->opt.span && p->span_next < tvs_plan::kSpanSlots) ? p->span + p->span_next++ : nullptr;
  };
  // common per-launch fields
  auto base_args = [&](int Hg, int Wg, int strips, int r0, int nrows) {
    tvs::ConvArgs a{};
    a.B = B; a.H = Hg; a.W = Wg; a.strips = strips;
    a.row0 = r0; a.rows = nrows;
    a.escale = escale;
    a.status = status;
    a.watchdog_ns = (unsigned long long)std::max(1, p->opt.watchdog_ms) * 1000000ull;
    a.dbg = p->opt.debug;
    return a;
  };
  // K2 x (depth-2), K3
  int cur = 0;
  if (wide) {
    // wide variant: split activations (hi 128 | lo 128 halves per pixel), groups
    // of 4 CTAs per strip-row range (one 32-channel quarter each)
    const int strips = (W + tvs::kStripPx - 1) / tvs::kStripPx;
    CUtensorMap pair_map[2], single_map[2];
    for (int i = 0; i < 2; ++i) {
      pair_map[i] = make_act_map(act[i], B, H, W, tvs::kHaloPx, 192);  // [hi 128 fp16 | lo 128 e4m3] = 192 fp16 units
      single_map[i] = make_act_map(act[i], B, H, W, tvs::kHaloPx, 128);
    }
    for (int l = 0; l < nh; ++l) {
      tvs::ConvArgs a = base_args(H, W, strips, 0, H);
      a.wpack = p->wpack + (size_t)l * tvs::conv_wpack_wide_bytes(false);
      a.shift = p->bhid + (size_t)l * C;
      a.nshift = C;
      a.act_out = static_cast<uint8_t*>(act[cur ^ 1]);
      a.out_single = pair_in(l + 1) ? 0 : 1;
      a.span = next_span();
      const CUtensorMap& m = pair_in(l) ? pair_map[cur] : single_map[cur];
      // 4 (quarters) or 2 (halves) CTAs per strip-row range: size the grid by groups
      const int mode = pair_in(l) ? 5 : (p->packed_halves ? 11 : 9);
      const int parts = mode == 11 ? 2 : 4;
      const int grid = parts * std::max(1, std::min(max_ctas / parts, conv_grid(max_ctas, a)));
      timed_launch(p, st, TVS_KIND_HIDDEN, px * 2.0 * 9 * C * C,
                   [&] { return tvs::launch_conv_tc(mode, m, m, a, grid, st); });
      cur ^= 1;
    }
    tvs::ConvArgs a = base_args(H, W, strips, row0, rows);
    a.wpack = p->hpack;
    a.shift = p->bh;
    a.nshift = p->out_bands;
    a.x = x; a.bands = bands; a.closure = closure; a.recon = recon; a.K = p->out_bands;
    const int grid = conv_grid(max_ctas, a);
    const CUtensorMap& mh = single_map[cur];
    timed_launch(p, st, TVS_KIND_HEAD, (double)B * rows * W * 2.0 * 9 * C * p->out_bands,
                 [&] { return tvs::launch_conv_tc(10, mh, mh, a, grid, st); });
  } else if (wsplit) {
    // wide fp32-accurate mode: out_o = ReLU(conv(P0, W[o][0]) + conv(P1, W[o][1]) + shift_o),
    // each block conv on the 64-channel split kernel; the first writes its raw
    // fp32 sums, the second adds them in its epilogue (ConvArgs::acc_in)
    const int strips = (W + tvs::kStripPx - 1) / tvs::kStripPx;
    CUtensorMap in_map[2][2];
    for (int i = 0; i < 2; ++i)
      for (int k = 0; k < 2; ++k) in_map[i][k] = make_act_map(plane(i, k), B, H, W, tvs::kHaloPx, 128);
    const int mode = p->opt.fp32_pairs ? 12 : 3;
    for (int l = 0; l < nh; ++l) {
      for (int o = 0; o < 2; ++o)
        for (int k = 0; k < 2; ++k) {
          tvs::ConvArgs a = base_args(H, W, strips, 0, H);
          a.wpack = p->wpack + ((size_t)(l * 2 + o) * 2 + k) * tvs::conv_wpack_split_bytes();
          a.shift = p->bhid + (size_t)l * C + o * 64;
          a.nshift = 64;
          if (k == 0) {
            a.act_out = static_cast<uint8_t*>(p->act_raw);
            a.raw_f32 = 1;
          } else {
            a.act_out = plane(cur ^ 1, o);
            a.acc_in = static_cast<const float*>(p->act_raw);
          }
          a.span = next_span();
          const int grid = mode == 12 ? 2 * conv_grid(max_ctas / 2, a) : conv_grid(max_ctas, a);
          timed_launch(p, st, TVS_KIND_HIDDEN, px * 2.0 * 9 * 64 * 64,
                       [&] { return tvs::launch_conv_tc(mode, in_map[cur][k], in_map[cur][k], a, grid, st); });
        }
      cur ^= 1;
    }
    for (int k = 0; k < 2; ++k) {
      tvs::ConvArgs a = base_args(H, W, strips, row0, rows);
      a.wpack = p->hpack + (size_t)k * tvs::conv_wpack_bytes(true);
      a.K = p->out_bands;
      a.x = x; a.bands = bands;
      if (k == 1) {  // + block 0's partial bands, bias, closure, checks
        a.shift = p->bh;
        a.nshift = p->out_bands;
        a.acc_bands = 1;
        a.closure = closure; a.recon = recon;
      }
      const int grid = conv_grid(max_ctas, a);
      timed_launch(p, st, TVS_KIND_HEAD, (double)B * rows * W * 2.0 * 9 * 64 * p->out_bands,
                   [&] { return tvs::launch_conv_tc(4, in_map[cur][k], in_map[cur][k], a, grid, st); });
    }
  } else if (split) {
    // fp32-accurate: split-operand tcgen05 layers on fp16 hi|lo pair rows
    const int strips = (W + tvs::kStripPx - 1) / tvs::kStripPx;
    CUtensorMap in_map[2];
    for (int i = 0; i < 2; ++i) in_map[i] = make_act_map(act[i], B, H, W, tvs::kHaloPx, 128);
    for (int l = 0; l < nh; ++l) {
      tvs::ConvArgs a = base_args(H, W, strips, 0, H);
      a.wpack = p->wpack + (size_t)l * tvs::conv_wpack_split_bytes();
      a.shift = p->bhid + (size_t)l * tvs::kC;
      a.nshift = tvs::kC;
      a.act_out = static_cast<uint8_t*>(act[cur ^ 1]);
      a.span = next_span();
      // CTA pairs (mode 12): both output-channel halves of a strip-row range at
      // once, input rows multicast to the pair; a pair covers what one mode-3
      // CTA covers in two visits, so the grid counts pairs of CTAs
      const int mode = p->opt.fp32_pairs ? 12 : 3;
      const int grid = mode == 12 ? 2 * conv_grid(max_ctas / 2, a) : conv_grid(max_ctas, a);
      timed_launch(p, st, TVS_KIND_HIDDEN, px * 2.0 * 9 * 64 * 64,
                   [&] { return tvs::launch_conv_tc(mode, in_map[cur], in_map[cur], a, grid, st); });
      cur ^= 1;
    }
    tvs::ConvArgs a = base_args(H, W, strips, row0, rows);
    a.wpack = p->hpack;
    a.shift = p->bh;
    a.nshift = p->out_bands;
    a.x = x; a.bands = bands; a.closure = closure; a.recon = recon; a.K = p->out_bands;
    const int grid = conv_grid(max_ctas, a);
    timed_launch(p, st, TVS_KIND_HEAD, (double)B * rows * W * 2.0 * 9 * 64 * p->out_bands,
                 [&] { return tvs::launch_conv_tc(4, in_map[cur], in_map[cur], a, grid, st); });
  } else if (fast) {
    const int Hg = H / us, Wg = W / us;  // layer grid (half-res when unshuffled)
    const double pxg = px / (us * us);
    const int strips = (Wg + tvs::kStripPx - 1) / tvs::kStripPx;
    CUtensorMap in_map[2], out_map[2];
    for (int i = 0; i < 2; ++i) {
      in_map[i] = make_act_map(act[i], B, Hg, Wg, tvs::kHaloPx);
      out_map[i] = make_act_map(act[i], B, Hg, Wg, 32);
    }
    int l0 = 0;
    if (stack) {
      tvs::ConvArgs a = base_args(Hg, Wg, strips, 0, Hg);
      a.wpack = p->wpack;
      a.shift = p->bhid;
      a.nshift = tvs::kC;
      a.nlayers = nh;
      a.rowcnt = p->rowcnt;
      a.abort = p->rowcnt + (p->rowcnt_n - 1);
      size_t nitems = 0;
      a.items = stack_items(p, B, strips, a.nlayers, Hg, band_rows, p->opt.stack_skew, st, &nitems);
      a.watcher = p->opt.stack_watcher;
      a.nitems = (int)nitems;
      a.span = next_span();
      tvs::StackMaps sm{};
      sm.in1 = in_map[1];
      sm.out0 = out_map[0];
      cudaError_t e = cudaSuccess;
      timed_launch(p, st, TVS_KIND_HIDDEN, a.nlayers * pxg * 2.0 * 9 * 64 * 64, [&] {
        e = tvs::launch_conv_stack(in_map[0], out_map[1], sm, a, stack_grid, st);
        return e == cudaErrorCooperativeLaunchTooLarge ? cudaSuccess : e;
      });
      if (e == cudaErrorCooperativeLaunchTooLarge) {
        // the driver cannot make the grid co-resident here (MPS SM limits,
        // green contexts): nothing ran, use the per-layer kernels from now on
        cudaGetLastError();
        p->stack_ok = false;
        p->last_launches--;
      } else {
        l0 = a.nlayers;
        cur = l0 & 1;
        p->last_stack = 1;
      }
    }
    for (int l = l0; l < nh; ++l) {
      tvs::ConvArgs a = base_args(Hg, Wg, strips, 0, Hg);
      a.wpack = p->wpack + (size_t)l * tvs::conv_wpack_bytes(false);
      a.shift = p->bhid + (size_t)l * tvs::kC;
      a.nshift = tvs::kC;
      a.x = x;
      a.span = next_span();
      const int grid = conv_grid(max_ctas, a);
      timed_launch(p, st, TVS_KIND_HIDDEN, pxg * 2.0 * 9 * 64 * 64,
                   [&] { return tvs::launch_conv_tc(0, in_map[cur], out_map[cur ^ 1], a, grid, st); });
      cur ^= 1;
    }
    tvs::ConvArgs a = base_args(Hg, Wg, strips, row0 / us, rows / us);
    a.wpack = p->hpack;
    a.shift = p->bh;
    a.nshift = p->out_bands * us * us;
    if (l0 == nh && nh > 0 && us == 1 && p->opt.head_gate) {
      // the head starts on the SMs the stack's CTAs free and acquires layer
      // nh-1's rows through the stack's row flags (conv_tc.cu gate_target)
      a.rowcnt = p->rowcnt;
      a.abort = p->rowcnt + (p->rowcnt_n - 1);
      a.gate_target = 4 * nh;
    }
    a.x = x; a.bands = bands; a.closure = closure; a.recon = recon; a.K = p->out_bands;
    // a gated head gets more, shorter CTAs: the block scheduler hands them to
    // the SMs in the order the stack's CTAs free them (dynamic balance)
    const int grid = a.gate_target ? conv_grid(max_ctas * std::max(1, p->opt.head_grid), a) : conv_grid(max_ctas, a);
    timed_launch(p, st, TVS_KIND_HEAD, (double)B * rows * W * 2.0 * 9 * 64 * p->out_bands,
                 [&] { return tvs::launch_conv_tc(us == 2 ? 7 : 1, in_map[cur], in_map[cur], a, grid, st); });
  } else {
    for (int l = 0; l < nh; ++l) {
      timed_launch(p, st, TVS_KIND_HIDDEN, px * 2.0 * 9 * C * C, [&] {
        return tvs::launch_hidden_f32(C, (const float*)act[cur], (float*)act[cur ^ 1],
                                      p->whid + (size_t)l * C * C * 9, p->shid + (size_t)l * C,
                                      p->bhid + (size_t)l * C, B, H, W, st);
      });
      cur ^= 1;
    }
    timed_launch(p, st, TVS_KIND_HEAD, (double)B * rows * W * 2.0 * 9 * C * p->out_bands, [&] {
      return tvs::launch_head_f32(C, (const float*)act[cur], x, p->wh, p->bh, bands, recon, closure, B, H, W, p->out_bands,
                                  row0, rows, status, st);
    });
  }
}

// Evaluate one forward's status words (host copy).
void evaluate_status(const int* s) {
  if (s[tvs::kStatWatchdog])
    throw TvsError(TVS_E_CUDA,
                   "layer-stack row-flag wait expired (watchdog): that forward's output is invalid; later forwards "
                   "are unaffected (plan option stack=0 selects the per-layer kernels)");
  if (s[tvs::kStatNonFiniteOut] && !s[tvs::kStatNonFiniteIn])
    throw TvsError(TVS_E_NUMERIC,
                   "non-finite band values from a finite input: the activations left the fp16 range of this mode "
                   "(use precision fp32 with plan option fp32_cuda=1 for full fp32 range)");
}

// Poll deferred status checks; `wait` blocks on all of them.
void drain_status(tvs_plan* p, bool wait) {
  while (!p->status_pending.empty()) {
    const int slot = p->status_pending.front();
    if (wait) {
      TVS_CUDA(cudaEventSynchronize(p->status_ev[slot]));
    } else {
      const cudaError_t q = cudaEventQuery(p->status_ev[slot]);
      if (q == cudaErrorNotReady) return;
      if (q != cudaSuccess) TVS_CUDA(q);
    }
    p->status_pending.pop_front();
    evaluate_status(p->status_host + slot * tvs::kStatWords);
  }
}

void forward_impl(tvs_plan* p, const float* x, float* bands, float* closure, int B, int H, int W, int row0, int rows,
                  cudaStream_t st, double* recon = nullptr) {
  if (!p->weights_ready) throw TvsError(TVS_E_STATE, "tvs_forward before tvs_plan_set_weights");
  if (!x || !bands) throw TvsError(TVS_E_INVALID, "null x/bands pointer");
  if (B < 0 || H < 1 || W < 1) throw TvsError(TVS_E_INVALID, "bad shape B/H/W");
  if (rows < 0) { row0 = 0; rows = H; }
  if (row0 < 0 || rows < 1 || row0 + rows > H) throw TvsError(TVS_E_INVALID, "bad valid row window");
  if (p->unshuffle == 2 && (H % 2 || W % 2 || row0 % 2 || rows % 2))
    throw TvsError(TVS_E_INVALID, "unshuffle = 2 needs even H, W and an even row window");
  if (recon && !closure) throw TvsError(TVS_E_INVALID, "the reconstruction check needs the closure plane");
  p->last_launches = 0;
  p->last_stack = 0;
  if (B == 0) return;
  NvtxRange nr("tvs_forward");
  DeviceGuard dg(p->device);
  drain_status(p, false);  // report a finished earlier forward's failure (deferred mode)
  const size_t per_img = (size_t)H * W * p->act_px_bytes() / ((size_t)p->unshuffle * p->unshuffle);
  const size_t in_img = (size_t)H * W, out_img = (size_t)rows * W;
  const bool check = p->opt.check != 0;
  int* status = nullptr;
  int slot = -1;
  if (check) {
    if (p->status_pending.size() >= (size_t)tvs_plan::kRing) {  // deferred ring full: settle the oldest
      TVS_CUDA(cudaEventSynchronize(p->status_ev[p->status_pending.front()]));
      drain_status(p, false);
    }
    slot = p->status_next;
    p->status_next = (slot + 1) % tvs_plan::kRing;
    std::fill(p->status_host + slot * tvs::kStatWords, p->status_host + (slot + 1) * tvs::kStatWords, 0);
    status = p->status_dev + slot * tvs::kStatWords;
  }
  if (recon) TVS_CUDA(cudaMemsetAsync(recon, 0, (size_t)B * 2 * sizeof(double), st));
  const int* escale = nullptr;
  if (p->scaled()) {
    if ((size_t)B > p->escale_n) {
      if (p->escale) TVS_CUDA(cudaFree(p->escale));
      p->escale = nullptr;
      p->escale_n = 0;
      TVS_CUDA(cudaMalloc(&p->escale, (size_t)B * 3 * sizeof(int)));  // exponents | 2B scratch
      TVS_CUDA(cudaMemsetAsync(p->escale, 0, (size_t)B * 3 * sizeof(int), st));
      p->escale_n = B;
    }
    TVS_CUDA(tvs::launch_input_scale(x, B, (long long)H * W, p->w0_l1, p->b0_max, p->escale, p->escale + B,
                                     status, st));
    p->last_launches++;
    escale = p->escale;
  }
  int cb = (int)std::max<size_t>(1, (size_t)(p->opt.chunk_mb << 20) / std::max<size_t>(per_img, 1));
  cb = std::min(cb, B);
  ensure_act(p, per_img * cb);
  if (p->wide_split_path()) ensure_raw(p, (size_t)H * W * 256 * cb);
  for (int b0 = 0; b0 < B; b0 += cb) {
    const int nb = std::min(cb, B - b0);
    run_chunk(p, x + b0 * in_img, bands + (size_t)b0 * p->out_bands * out_img,
              closure ? closure + b0 * out_img : nullptr, nb, H, W, row0, rows, st, escale ? escale + b0 : nullptr,
              status, escale != nullptr && b0 == 0, recon ? recon + 2 * b0 : nullptr);
  }
  if (!check) return;
  TVS_CUDA(cudaEventRecord(p->status_ev[slot], st));
  if (p->opt.check == 1) {
    TVS_CUDA(cudaEventSynchronize(p->status_ev[slot]));
    evaluate_status(p->status_host + slot * tvs::kStatWords);
  } else {
    p->status_pending.push_back(slot);
  }
}


}  // namespace

extern "C" {

int tvs_abi_version(void) { return TVS_ABI_VERSION; }

const char* tvs_last_error(void) { return tvs_host::last_error().c_str(); }

int tvs_plan_create(int device, int depth, int channels, int out_bands, int mode, tvs_plan** out_plan) {
  return tvs_plan_create_ex(device, depth, channels, out_bands, mode, 1, out_plan);
}

int tvs_plan_create_ex(int device, int depth, int channels, int out_bands, int mode, int unshuffle,
                       tvs_plan** out_plan) {
  return guarded([&] {
    if (!out_plan) throw TvsError(TVS_E_INVALID, "out_plan is null");
    *out_plan = nullptr;
    if (unshuffle != 1 && unshuffle != 2) throw TvsError(TVS_E_INVALID, "unshuffle must be 1 or 2");
    if (unshuffle == 2 && (mode != TVS_MODE_FAST || channels != 64))
      throw TvsError(TVS_E_UNSUPPORTED, "unshuffle = 2 is built for FAST mode with 64 channels");
    if (depth < 3) throw TvsError(TVS_E_INVALID, "depth must be at least 3 (first, hidden, last)");
    if (channels != 64 && channels != 128)
      throw TvsError(TVS_E_UNSUPPORTED, "this build supports channels 64 and 128");
    if (out_bands < 1 || out_bands > 8) throw TvsError(TVS_E_UNSUPPORTED, "out_bands must be in [1, 8]");
    if (mode != TVS_MODE_FP32 && mode != TVS_MODE_FAST) throw TvsError(TVS_E_INVALID, "unknown mode");
    int ndev = 0;
    TVS_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw TvsError(TVS_E_INVALID, "bad device ordinal");
    DeviceGuard dg(device);
    cudaDeviceProp prop;
    TVS_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
      throw TvsError(TVS_E_UNSUPPORTED, "libtvsb200 is built for sm_100a (B200) only");
    auto* p = new tvs_plan();
    p->device = device; p->depth = depth; p->channels = channels; p->out_bands = out_bands; p->mode = mode;
    p->unshuffle = unshuffle;
    p->num_sms = prop.multiProcessorCount;
    if (const char* e = std::getenv("TVS_CONV_DBG")) p->opt.debug = std::atoi(e);  // debug builds of experiments
    try {
      TVS_CUDA(tvs::configure_kernels());
      p->stack_ok = tvs::conv_stack_fits(p->num_sms, p->num_sms);
      TVS_CUDA(cudaMalloc(&p->span, tvs_plan::kSpanSlots * sizeof(tvs::KernelSpan)));
      {
        std::vector<tvs::KernelSpan> armed(tvs_plan::kSpanSlots, tvs::KernelSpan{~0ull, 0ull});
        TVS_CUDA(cudaMemcpy(p->span, armed.data(), armed.size() * sizeof(tvs::KernelSpan), cudaMemcpyHostToDevice));
      }
      TVS_CUDA(cudaHostAlloc(&p->status_host, tvs_plan::kRing * tvs::kStatWords * sizeof(int), cudaHostAllocMapped));
      std::fill(p->status_host, p->status_host + tvs_plan::kRing * tvs::kStatWords, 0);
      TVS_CUDA(cudaHostGetDevicePointer((void**)&p->status_dev, p->status_host, 0));
      for (auto& e : p->status_ev) TVS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    } catch (...) {
      free_all(p);
      delete p;
      throw;
    }
    *out_plan = p;
  });
}

int tvs_plan_set_option(tvs_plan* p, const char* name, long long value) {
  return guarded([&] {
    if (!p || !name) throw TvsError(TVS_E_INVALID, "null plan/name");
    const std::string k(name);
    auto& o = p->opt;
    auto flag = [&](int& f) { if (value != 0 && value != 1) throw TvsError(TVS_E_INVALID, k + " takes 0 or 1"); f = (int)value; };
    if (k == "stack") {
      if (value < -1 || value > 1) throw TvsError(TVS_E_INVALID, "stack takes -1 (auto), 0 or 1");
      o.stack = (int)value;
    } else if (k == "stack_band_rows") {
      if (value < 0 || value > (1 << 20)) throw TvsError(TVS_E_INVALID, "stack_band_rows out of range");
      o.stack_band_rows = (int)value;
    } else if (k == "head_gate") flag(o.head_gate);
    else if (k == "stack_watcher") flag(o.stack_watcher);
    else if (k == "fp32_pairs") flag(o.fp32_pairs);
    else if (k == "head_grid") {
      if (value < 1 || value > 64) throw TvsError(TVS_E_INVALID, "head_grid takes 1..64");
      o.head_grid = (int)value;
    }
    else if (k == "stack_skew") {
      if (value < 0 || value > 64) throw TvsError(TVS_E_INVALID, "stack_skew takes 0..64");
      o.stack_skew = (int)value;
    } else if (k == "conv0_tc") flag(o.conv0_tc);
    else if (k == "wide_pair_layers") {
      if (value < 0 || value > 1024) throw TvsError(TVS_E_INVALID, "wide_pair_layers out of range");
      o.wide_pair_layers = (int)value;
      p->weights_ready = false;
    } else if (k == "wide_halves") { flag(o.wide_halves); p->weights_ready = false; }
    else if (k == "fp32_cuda") { flag(o.fp32_cuda); p->weights_ready = false; }
    else if (k == "wide_cuda") { flag(o.wide_cuda); p->weights_ready = false; }
    else if (k == "chunk_mb") {
      if (value < 1) throw TvsError(TVS_E_INVALID, "chunk_mb must be positive");
      o.chunk_mb = value;
    } else if (k == "check") {
      if (value < 0 || value > 2) throw TvsError(TVS_E_INVALID, "check takes 0 (off), 1 (sync) or 2 (deferred)");
      if (o.check == 2 && value != 2) {  // leaving deferred mode: settle what is outstanding
        DeviceGuard dg(p->device);
        drain_status(p, true);
      }
      o.check = (int)value;
    } else if (k == "watchdog_ms") {
      if (value < 1 || value > 3600000) throw TvsError(TVS_E_INVALID, "watchdog_ms out of range");
      o.watchdog_ms = (int)value;
    } else if (k == "input_scale") flag(o.input_scale);
    else if (k == "span") flag(o.span);
    else if (k == "debug") o.debug = (int)value;
    else throw TvsError(TVS_E_INVALID, "unknown plan option '" + k + "'");
  });
}

int tvs_plan_sync(tvs_plan* p, void* stream) {
  return guarded([&] {
    if (!p) throw TvsError(TVS_E_INVALID, "null plan");
    DeviceGuard dg(p->device);
    TVS_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    drain_status(p, true);
  });
}

int tvs_plan_set_weights(tvs_plan* p, const float* const* w_dev, const float* const* scale_dev,
                         const float* const* shift_dev, int n_layers, void* stream) {
  return guarded([&] {
    if (!p || !w_dev || !shift_dev) throw TvsError(TVS_E_INVALID, "null argument");
    if (n_layers != p->depth) throw TvsError(TVS_E_INVALID, "n_layers must equal depth");
    for (int i = 0; i < n_layers; ++i)
      if (!w_dev[i] || !shift_dev[i]) throw TvsError(TVS_E_INVALID, "null weight/shift pointer");
    auto scale_of = [&](int i) -> const float* { return scale_dev ? scale_dev[i] : nullptr; };
    if (scale_of(0) || scale_of(p->depth - 1))
      throw TvsError(TVS_E_UNSUPPORTED, "conv0/head take no BatchNorm scale (model.py:37,44)");
    DeviceGuard dg(p->device);
    cudaStream_t st = (cudaStream_t)stream;
    TVS_CUDA(cudaStreamSynchronize(st));  // earlier forwards may still read the old packs
    free_weights(p);
    const int nh = p->n_hidden();
    const int C = p->channels;
    const int us = p->unshuffle;
    // buffers for the path the current options select
    TVS_CUDA(cudaMalloc(&p->wh, (size_t)p->out_bands * C * 9 * 4));
    TVS_CUDA(cudaMalloc(&p->bh, (size_t)p->out_bands * us * us * 4));  // head bias (4K if unshuffled)
    TVS_CUDA(cudaMalloc(&p->bhid, (size_t)nh * C * 4));
    TVS_CUDA(cudaMalloc(&p->shid, (size_t)nh * C * 4));
    if (p->tc_path()) {
      TVS_CUDA(cudaMalloc(&p->wpack, (size_t)nh * tvs::conv_wpack_bytes(false)));
      TVS_CUDA(cudaMalloc(&p->hpack, us == 2 ? tvs::conv_wpack_unshuf_head_bytes() : tvs::conv_wpack_bytes(true)));
      if (us == 2) {
        TVS_CUDA(cudaMalloc(&p->w0u, (size_t)C * 36 * 4));
        TVS_CUDA(cudaMalloc(&p->b0u, (size_t)C * 4));
      }
      TVS_CUDA(cudaMalloc(&p->c0pack, tvs::conv0_tc_pack_bytes(us == 2 ? 4 : 1)));
      TVS_CUDA(cudaMalloc(&p->c0bias, 64 * sizeof(float)));
    } else if (p->split_path()) {
      TVS_CUDA(cudaMalloc(&p->wpack, (size_t)nh * tvs::conv_wpack_split_bytes()));
      TVS_CUDA(cudaMalloc(&p->hpack, tvs::conv_wpack_bytes(true)));
    } else if (p->wide_path()) {
      TVS_CUDA(cudaMalloc(&p->wpack, (size_t)nh * tvs::conv_wpack_wide_bytes(false)));
      TVS_CUDA(cudaMalloc(&p->hpack, tvs::conv_wpack_wide_bytes(true)));
    } else if (p->wide_split_path()) {  // 2 x 2 blocks per hidden layer, 2 head blocks
      TVS_CUDA(cudaMalloc(&p->wpack, (size_t)nh * 4 * tvs::conv_wpack_split_bytes()));
      TVS_CUDA(cudaMalloc(&p->hpack, 2 * tvs::conv_wpack_bytes(true)));
    } else {
      TVS_CUDA(cudaMalloc(&p->whid, (size_t)nh * C * C * 9 * 4));
    }
    // conv0 on the host side: CUDA-core K1 parameters and the input-scale bound
    const int taps0 = us == 2 ? 36 : 9;
    std::vector<float> w0((size_t)C * taps0), b0(C);
    TVS_CUDA(cudaMemcpyAsync(w0.data(), w_dev[0], w0.size() * 4, cudaMemcpyDeviceToHost, st));
    TVS_CUDA(cudaMemcpyAsync(b0.data(), shift_dev[0], (size_t)C * 4, cudaMemcpyDeviceToHost, st));
    TVS_CUDA(cudaStreamSynchronize(st));
    p->w0_l1 = 0.f;
    p->b0_max = 0.f;
    for (int co = 0; co < C; ++co) {
      float l1 = 0.f;
      for (int t = 0; t < taps0; ++t) l1 += std::fabs(w0[(size_t)co * taps0 + t]);
      p->w0_l1 = std::max(p->w0_l1, l1);
      p->b0_max = std::max(p->b0_max, std::fabs(b0[co]));
    }
    if (us == 2) {  // conv0 Conv2d(4, C) on the device; head Conv2d(C, 4K) packed below
      TVS_CUDA(cudaMemcpyAsync(p->w0u, w_dev[0], (size_t)C * 36 * 4, cudaMemcpyDeviceToDevice, st));
      TVS_CUDA(cudaMemcpyAsync(p->b0u, shift_dev[0], (size_t)C * 4, cudaMemcpyDeviceToDevice, st));
    } else {
      std::copy(w0.begin(), w0.end(), p->conv0.w);
      std::copy(b0.begin(), b0.end(), p->conv0.b);
      if (C == 128)
        for (int o = 0; o < 2; ++o) {
          std::copy(w0.begin() + o * 64 * 9, w0.begin() + (o + 1) * 64 * 9, p->conv0_blk[o].w);
          std::copy(b0.begin() + o * 64, b0.begin() + (o + 1) * 64, p->conv0_blk[o].b);
        }
      TVS_CUDA(cudaMemcpyAsync(p->wh, w_dev[p->depth - 1], (size_t)p->out_bands * C * 9 * 4,
                               cudaMemcpyDeviceToDevice, st));
    }
    if (p->tc_path()) {  // K1 on tcgen05: TF32 hi/lo B pack + bias
      TVS_CUDA(tvs::launch_pack_conv0_tc(w_dev[0], us == 2 ? 4 : 1, p->c0pack, st));
      TVS_CUDA(cudaMemcpyAsync(p->c0bias, shift_dev[0], 64 * sizeof(float), cudaMemcpyDeviceToDevice, st));
    }
    TVS_CUDA(cudaMemcpyAsync(p->bh, shift_dev[p->depth - 1], (size_t)p->out_bands * us * us * 4,
                             cudaMemcpyDeviceToDevice, st));
    p->packed_pairs = p->opt.wide_pair_layers;
    p->packed_halves = p->opt.wide_halves;
    const int P = std::max(0, std::min(p->packed_pairs, nh));
    for (int l = 0; l < nh; ++l) {
      const float* sc = scale_of(l + 1);
      float* dst_scale = p->shid + l * C;
      if (sc)
        TVS_CUDA(cudaMemcpyAsync(dst_scale, sc, C * 4, cudaMemcpyDeviceToDevice, st));
      else
        TVS_CUDA(tvs::launch_fill(dst_scale, 1.0f, C, st));
      TVS_CUDA(cudaMemcpyAsync(p->bhid + l * C, shift_dev[l + 1], C * 4, cudaMemcpyDeviceToDevice, st));
      if (p->tc_path()) {
        TVS_CUDA(tvs::launch_pack_hidden_f16(w_dev[l + 1], dst_scale,
                                             p->wpack + (size_t)l * tvs::conv_wpack_bytes(false), st));
      } else if (p->split_path()) {
        TVS_CUDA(tvs::launch_pack_hidden_split(w_dev[l + 1], dst_scale,
                                               p->wpack + (size_t)l * tvs::conv_wpack_split_bytes(), st));
      } else if (p->wide_split_path()) {
        for (int o = 0; o < 2; ++o)
          for (int k = 0; k < 2; ++k)
            TVS_CUDA(tvs::launch_pack_hidden_split(
                w_dev[l + 1], dst_scale, p->wpack + ((size_t)(l * 2 + o) * 2 + k) * tvs::conv_wpack_split_bytes(), st,
                128, o * 64, k * 64));
      } else if (p->wide_path()) {  // pair-input layers: quarters (mode 5); single-input: halves (mode 11)
        const bool pair_in = l < P || P >= nh;
        TVS_CUDA(tvs::launch_pack_hidden_wide(w_dev[l + 1], dst_scale,
                                              p->wpack + (size_t)l * tvs::conv_wpack_wide_bytes(false), st,
                                              pair_in || !p->packed_halves ? 4 : 2, pair_in));
      } else {
        TVS_CUDA(cudaMemcpyAsync(p->whid + (size_t)l * C * C * 9, w_dev[l + 1], (size_t)C * C * 9 * 4,
                                 cudaMemcpyDeviceToDevice, st));
      }
    }
    if (us == 2) {
      TVS_CUDA(tvs::launch_pack_head_unshuf(w_dev[p->depth - 1], 4 * p->out_bands, p->hpack, st));
    } else if (p->tc_path() || p->split_path()) {
      TVS_CUDA(tvs::launch_pack_head_f16(w_dev[p->depth - 1], p->out_bands, p->hpack, st));
    }
    if (p->wide_path()) TVS_CUDA(tvs::launch_pack_head_wide(w_dev[p->depth - 1], p->out_bands, p->hpack, st));
    if (p->wide_split_path())
      for (int k = 0; k < 2; ++k)
        TVS_CUDA(tvs::launch_pack_head_f16(w_dev[p->depth - 1], p->out_bands,
                                           p->hpack + (size_t)k * tvs::conv_wpack_bytes(true), st, 128, k * 64));
    p->packed_tc = p->tc_path();
    p->packed_split = p->split_path();
    p->packed_wide = p->wide_path();
    p->packed_wide_split = p->wide_split_path();
    p->weights_ready = true;
  });
}

int tvs_forward(tvs_plan* p, const float* x, float* bands, float* closure_or_null, int B, int H, int W,
                int valid_row0, int valid_rows, void* stream) {
  return guarded([&] {
    if (!p) throw TvsError(TVS_E_INVALID, "null plan");
    if (p->weights_ready && (p->packed_tc != p->tc_path() || p->packed_split != p->split_path() ||
                             p->packed_wide != p->wide_path() || p->packed_wide_split != p->wide_split_path()))
      throw TvsError(TVS_E_STATE, "plan options changed the weight layout: call tvs_plan_set_weights again");
    forward_impl(p, x, bands, closure_or_null, B, H, W, valid_row0, valid_rows, (cudaStream_t)stream);
  });
}

int tvs_forward_checked(tvs_plan* p, const float* x, float* bands, float* closure, double* recon, int B, int H, int W,
                        int valid_row0, int valid_rows, void* stream) {
  return guarded([&] {
    if (!p || !closure || !recon) throw TvsError(TVS_E_INVALID, "null plan/closure/recon");
    if (p->weights_ready && (p->packed_tc != p->tc_path() || p->packed_split != p->split_path() ||
                             p->packed_wide != p->wide_path() || p->packed_wide_split != p->wide_split_path()))
      throw TvsError(TVS_E_STATE, "plan options changed the weight layout: call tvs_plan_set_weights again");
    forward_impl(p, x, bands, closure, B, H, W, valid_row0, valid_rows, (cudaStream_t)stream, recon);
  });
}

int tvs_forward_host(tvs_plan* p, const float* x_host, float* bands_host, float* closure_host_or_null, int B, int H,
                     int W, void* stream) {
  return guarded([&] {
    if (!p || !x_host || !bands_host) throw TvsError(TVS_E_INVALID, "null argument");
    if (B < 0 || H < 1 || W < 1) throw TvsError(TVS_E_INVALID, "bad shape B/H/W");
    DeviceGuard dg(p->device);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t nx = (size_t)B * H * W, nb = nx * p->out_bands;
    const size_t need = (nx + nb + nx) * 4;
    if (need > p->io_bytes) {
      if (p->dx) cudaFree(p->dx);
      p->dx = nullptr; p->io_bytes = 0;
      TVS_CUDA(cudaMalloc(&p->dx, need));
      p->io_bytes = need;
    }
    float* dbands = p->dx + nx;
    float* dclos = dbands + nb;
    TVS_CUDA(cudaMemcpyAsync(p->dx, x_host, nx * 4, cudaMemcpyHostToDevice, st));
    forward_impl(p, p->dx, dbands, closure_host_or_null ? dclos : nullptr, B, H, W, 0, H, st);
    TVS_CUDA(cudaMemcpyAsync(bands_host, dbands, nb * 4, cudaMemcpyDeviceToHost, st));
    if (closure_host_or_null)
      TVS_CUDA(cudaMemcpyAsync(closure_host_or_null, dclos, nx * 4, cudaMemcpyDeviceToHost, st));
    TVS_CUDA(cudaStreamSynchronize(st));
    drain_status(p, true);
  });
}

int tvs_last_launch_count(const tvs_plan* p) { return p ? p->last_launches : 0; }
int tvs_last_used_stack(const tvs_plan* p) { return p ? p->last_stack : 0; }

int tvs_profile_enable(tvs_plan* p, int on) {
  return guarded([&] {
    if (!p) throw TvsError(TVS_E_INVALID, "null plan");
    DeviceGuard dg(p->device);
    drain_profile(p);
    for (int k = 0; k < 3; ++k) { p->prof_ms[k] = 0; p->prof_n[k] = 0; p->prof_flops[k] = 0; }
    p->profiling = on != 0;
  });
}

int tvs_profile_read(tvs_plan* p, int kind, double* total_ms, long long* launches, double* flops) {
  return guarded([&] {
    if (!p || kind < 0 || kind > 2) throw TvsError(TVS_E_INVALID, "bad plan/kind");
    DeviceGuard dg(p->device);
    drain_profile(p);
    if (total_ms) *total_ms = p->prof_ms[kind];
    if (launches) *launches = p->prof_n[kind];
    if (flops) *flops = p->prof_flops[kind];
  });
}

int tvs_profile_span(tvs_plan* p, double* total_ms, long long* launches, int reset) {
  return guarded([&] {
    if (!p) throw TvsError(TVS_E_INVALID, "null plan");
    DeviceGuard dg(p->device);
    TVS_CUDA(cudaDeviceSynchronize());
    const int n = p->span_next;
    std::vector<tvs::KernelSpan> h(std::max(1, n));
    if (n) TVS_CUDA(cudaMemcpy(h.data(), p->span, n * sizeof(tvs::KernelSpan), cudaMemcpyDeviceToHost));
    double ns = 0.0;
    long long cnt = 0;
    for (int i = 0; i < n; ++i)
      if (h[i].end > h[i].start) { ns += (double)(h[i].end - h[i].start); ++cnt; }
    if (total_ms) *total_ms = ns * 1e-6;
    if (launches) *launches = cnt;
    if (reset && n) {
      std::fill(h.begin(), h.begin() + n, tvs::KernelSpan{~0ull, 0ull});
      TVS_CUDA(cudaMemcpy(p->span, h.data(), n * sizeof(tvs::KernelSpan), cudaMemcpyHostToDevice));
      p->span_next = 0;
    }
  });
}

int tvs_band_stats(const float* gt, const float* pred, int planes, int H, int W, const double* range_or_null,
                   double* stats, void* stream) {
  return guarded([&] {
    if (!gt || !pred || !stats) throw TvsError(TVS_E_INVALID, "null pointer");
    if (planes < 0 || H < 1 || W < 1) throw TvsError(TVS_E_INVALID, "bad shape");
    if (planes == 0) return;
    TVS_CUDA(tvs::launch_band_stats(gt, pred, planes, H, W, range_or_null, stats, (cudaStream_t)stream));
  });
}

size_t tvs_tvflow_workspace_bytes(int N, int H, int W) {
  if (N < 0 || H < 1 || W < 1) return 0;
  return (size_t)N * 6 * (size_t)H * (size_t)W * sizeof(double);
}

int tvs_tvflow_analyze(const double* f, int N, int H, int W, double dt, int n_steps, const int* schedule,
                       int n_bands, int max_iters, double gap_tol, double pd_tau, double pd_sigma, int pd_accel,
                       void* workspace, double* bands, double* spectrum, double* residual, int* iters,
                       void* stream) {
  return guarded([&] {
    if (!f || !schedule || !workspace || !bands || !spectrum || !residual || !iters)
      throw TvsError(TVS_E_INVALID, "null pointer");
    if (N < 0 || H < 1 || W < 1) throw TvsError(TVS_E_INVALID, "bad shape");
    if (W > tvs::kTvMaxW) throw TvsError(TVS_E_INVALID, "image width exceeds 2048");
    if (!(dt > 0)) throw TvsError(TVS_E_INVALID, "dt must be positive");
    if (n_steps < 2) throw TvsError(TVS_E_INVALID, "n_steps must be >= 2");
    if (n_bands < 1 || n_bands > tvs::kTvMaxBands) throw TvsError(TVS_E_INVALID, "n_bands must lie in [1, 16]");
    int prev = 0;
    for (int b = 0; b < n_bands; ++b) {
      if (schedule[b] <= prev) throw TvsError(TVS_E_INVALID, "schedule indices must be strictly increasing");
      prev = schedule[b];
    }
    if (prev != n_steps - 1) throw TvsError(TVS_E_INVALID, "schedule must end at n_steps - 1");
    if (max_iters < 1) throw TvsError(TVS_E_INVALID, "max_iters must be >= 1");
    if (!(gap_tol > 0)) throw TvsError(TVS_E_INVALID, "gap_tol must be positive");
    if (!(pd_tau > 0) || !(pd_sigma > 0)) throw TvsError(TVS_E_INVALID, "primal-dual steps must be positive");
    if (pd_tau * pd_sigma * 8.0 > 1.0 + 1e-12) throw TvsError(TVS_E_INVALID, "pd_step_tau * pd_step_sigma * 8 must be <= 1");
    if (N == 0) return;
    tvs::TvFlowArgs a{};
    a.N = N;
    a.H = H;
    a.W = W;
    a.dt = dt;
    a.n_steps = n_steps;
    a.n_bands = n_bands;
    for (int b = 0; b < n_bands; ++b) a.schedule[b] = schedule[b];
    a.max_iters = max_iters;
    a.accel = pd_accel ? 1 : 0;
    a.gap_tol = gap_tol;
    a.tau0 = pd_tau;
    a.sigma0 = pd_sigma;
    a.f = f;
    a.work = (double*)workspace;
    a.bands = bands;
    a.spectrum = spectrum;
    a.residual = residual;
    a.iters = iters;
    TVS_CUDA(tvs::launch_tvflow(a, (cudaStream_t)stream));
  });
}

// diagnostics (not part of the public ABI): stack MMA-issuer cycle counters
int tvs_debug_cycles(unsigned long long* out, int reset) { return tvs::debug_cycles(out, reset); }
// diagnostics: the kDbgTrace row timeline, 5 x 32 x 1024 globaltimer stamps (conv_tc.cu g_trace)
int tvs_debug_trace(unsigned long long* out, int reset) { return tvs::debug_trace(out, reset); }

int tvs_plan_destroy(tvs_plan* p) {
  return guarded([&] {
    if (!p) return;
    DeviceGuard dg(p->device);
    cudaDeviceSynchronize();  // nothing of this plan may still be in flight
    free_all(p);
    delete p;
  });
}

}  // extern "C"
