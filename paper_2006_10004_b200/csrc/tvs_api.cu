// tvs_api.cu — host runtime behind include/tvs_b200.h: plans, packed
// weights, TMA descriptors, activation scratch and the per-layer launch
// sequence.  See DESIGN.md for the data layout.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <array>
#include <vector>

#include "../../include/tvs_b200.h"
#include "common.cuh"


namespace {

thread_local std::string g_last_error;

struct TvsError : std::runtime_error {
  int code;
  TvsError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define TVS_CUDA(call)                                                                                     \
  do {                                                                                                     \
    cudaError_t e_ = (call);                                                                               \
    if (e_ != cudaSuccess)                                                                                 \
      throw TvsError(TVS_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_) + " (" __FILE__ ":" + \
                                     std::to_string(__LINE__) + ")");                                      \
  } while (0)

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    TVS_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw TvsError(TVS_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// fp16 NHWC activation [B][H][W][C] (C = 64, or 128 = a hi|lo pair row) as a
// 4-D tensor map, SW128, box (64, box_px, 1, 1)
CUtensorMap make_act_map(void* base, int B, int H, int W, int box_px, int C = 64) {
  CUtensorMap m;
  const cuuint64_t rb = (cuuint64_t)C * 2;
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
  cuuint64_t strides[3] = {rb, (cuuint64_t)W * rb, (cuuint64_t)H * W * rb};
  cuuint32_t box[4] = {64, (cuuint32_t)box_px, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, base, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw TvsError(TVS_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

}  // namespace

struct tvs_plan {
  int device = 0, depth = 17, channels = 64, out_bands = 5, mode = TVS_MODE_FAST;
  int num_sms = 148;
  bool weights_ready = false;
  // conv0 [64][1][3][3] + bias, head [K][64][3][3] + bias (fp32, folded)
  tvs::Conv0Params conv0{};  // host copy, passed by value to K1
  float* wh = nullptr;
  float* bh = nullptr;
  // hidden: fast -> packed fp16 (n_hidden * conv_wpack_bytes(false)) ; fp32 -> [co][ci][9] fp32
  uint8_t* wpack = nullptr;
  uint8_t* hpack = nullptr;  // fast-mode head: fp16 hi/lo pack
  // opt-in unshuffle = 2 variant: conv0 Conv2d(4, 64) weights on the device
  int unshuffle = 1;
  float* w0u = nullptr;
  float* b0u = nullptr;
  float* whid = nullptr;
  float* bhid = nullptr;  // per hidden layer: shift (beta - mu*s)
  float* shid = nullptr;  // per hidden layer: BatchNorm scale s (fp32 mode epilogue; folded in FAST)
  // activation ping-pong scratch
  void* act[2] = {nullptr, nullptr};
  size_t act_bytes = 0;
  // concurrent L2-sized chunks (FAST path): stream s runs whole layer
  // sequences of its chunks on its own ping-pong buffers, grids of num_sms/S
  int l2_reverse_sub = 1;              // TVS_REVERSE_SUB: odd layers visit sub-ranges last-first (measured: no gain)
  int n_streams = 1;                   // TVS_STREAMS (measured: >1 does not help on B200)
  size_t l2_chunk_bytes = 16ull << 20; // TVS_L2_CHUNK_MB: activation bytes per chunk
  std::vector<cudaStream_t> streams;
  std::vector<void*> sact;             // 2 per stream
  size_t sact_bytes = 0;
  cudaEvent_t fork_ev = nullptr;
  std::vector<cudaEvent_t> join_ev;
  // host-API staging
  float* dx = nullptr;  // [x | bands | closure] staging for tvs_forward_host
  size_t io_bytes = 0;
  int last_launches = 0;
  // optional per-kernel event timing
  struct Rec { cudaEvent_t a, b; int kind; double flops; };
  bool profiling = false;
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> event_pool;
  double prof_ms[3] = {0, 0, 0};
  long long prof_n[3] = {0, 0, 0};
  double prof_flops[3] = {0, 0, 0};
  size_t chunk_budget = 2048ull << 20;
  // TVS_FUSE_CONV0=1: compute conv0 in the first hidden layer's producer warps
  // (saves the K1 kernel and 2x128 B/px of HBM traffic, but on B200 the
  // producer's ~600 FFMA/px-row currently cost more than they save)
  bool unfused_conv0 = true;  // activation bytes per chunk (TVS_CHUNK_MB)
  int l2_hints = 0;           // TVS_L2_HINTS (ConvArgs::l2_hints)
  // TVS_PAIR2=1: per-layer fast hidden layers on CTA pairs (cta_group::2,
  // conv_tc.cu conv3x3_pair2_kernel; prototype, disables the layer stack)
  bool pair2 = false;
  uint8_t* wpack2 = nullptr;
  // K1 on tcgen05 (conv0_tc.cu, TF32 hi/lo split) for the fast path: config 2
  // 149 vs 170 us (reference conv0, K = 9) and 96 vs 212 us (the unshuffle = 2
  // variant's Conv2d(4, 64), K = 36).  TVS_CONV0_TC=0 selects the CUDA-core K1.
  int conv0_tc = 1;
  uint8_t* c0pack = nullptr;  // packed TF32 hi/lo B operand
  float* c0bias = nullptr;
  bool pair_fuse = false;     // TVS_PAIR: fuse consecutive hidden layers (conv_pair.cu)
  // layer-stack kernel (conv_tc.cu mode 8, all hidden layers in one persistent
  // launch, activations handed between layers through L2): TVS_STACK = 0 off,
  // 1 whenever legal, -1 (default) when the chunk has >= kStackMinItems work
  // items per SM (short columns / few images keep the per-layer kernels)
  int stack = -1;
  // wide variant, fast mode: hidden layers reading fp16 hi/lo pairs (the rest
  // read single fp16; TVS_WIDE_PAIR).  12 of 24 keeps the worst band at
  // 6.6-8.0e-3 on config 5 (tools/emulate_wide.py), 0 is the plain-fp16
  // roofline probe (1.1-1.3e-2, over the 1e-2 gate)
  int wide_pair_layers = 12;
  // wide single-input layers on output-channel halves (mode 11, N = 192) instead
  // of quarters (mode 9, N = 96); TVS_WIDE_HALVES = 0 / 1
  bool wide_halves = true;
  static constexpr int kStackMinItems = 6;
  int* rowcnt = nullptr;  // row flags (B*strips*H ints), zeroed per chunk
  size_t rowcnt_n = 0;
  // work-item order (TVS_STACK_SKEW = A): items sorted by diagonal i*A + j, then
  // layer, then strip; A >= n_hidden is image-major, small A interleaves layer j
  // of image i with layer j+A of image i-1 (more slack between a layer and the
  // next, more activation rows live in L2)
  int stack_skew = 1 << 20;
  int2* items = nullptr;
  size_t items_cap = 0;
  long long items_key[4] = {-1, -1, -1, -1};

  int n_hidden() const { return depth - 2; }
  // tcgen05 fp16 path: FAST mode with 64 channels; everything else runs the
  // CUDA-core fp32 path (fp32-accurate mode, and the 128-channel wide variant)
  bool tc_path() const { return mode == TVS_MODE_FAST && channels == 64; }
  // fp32-accurate mode on tcgen05 with split fp16 operands (conv_tc.cu modes
  // 3/4).  TVS_FP32_CUDA=1 selects the CUDA-core fp32 kernels
  // (also used for the 128-channel wide variant).
  bool fp32_split = true;
  bool split_path() const { return mode == TVS_MODE_FP32 && channels == 64 && fp32_split; }
  // wide variant (128 channels) fast mode on tcgen05: split activations, fp16 weights
  // (conv_tc.cu modes 5/6); TVS_WIDE_CUDA=1 keeps it on the CUDA-core kernels
  bool wide_cuda = false;
  bool wide_path() const { return mode == TVS_MODE_FAST && channels == 128 && !wide_cuda; }
  size_t act_px_bytes() const { return tc_path() ? 128 : (size_t)channels * 4; }
};

namespace {

void ensure_device(const tvs_plan* p) { TVS_CUDA(cudaSetDevice(p->device)); }

void free_all(tvs_plan* p) {
  for (void* q : p->sact)
    if (q) cudaFree(q);
  p->sact.clear();
  for (auto st : p->streams) cudaStreamDestroy(st);
  p->streams.clear();
  for (auto e : p->join_ev) cudaEventDestroy(e);
  p->join_ev.clear();
  if (p->fork_ev) cudaEventDestroy(p->fork_ev);
  p->fork_ev = nullptr;
  for (auto& r : p->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : p->event_pool) cudaEventDestroy(e);
  p->recs.clear();
  p->event_pool.clear();
  void* ptrs[] = {p->wh, p->bh, p->wpack, p->hpack, p->whid, p->bhid, p->shid, p->act[0], p->act[1], p->dx,
                  p->w0u, p->b0u, p->rowcnt, p->items, p->c0pack, p->c0bias, p->wpack2};
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

// one CTA per SM, but never fewer than ~3 output rows per CTA (short
// segments pay two extra input rows each)
void ensure_streams(tvs_plan* p, int ns, size_t bytes) {
  if (!p->fork_ev) TVS_CUDA(cudaEventCreateWithFlags(&p->fork_ev, cudaEventDisableTiming));
  while ((int)p->streams.size() < ns) {
    cudaStream_t st;
    TVS_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    p->streams.push_back(st);
    cudaEvent_t e;
    TVS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    p->join_ev.push_back(e);
  }
  if (bytes > p->sact_bytes || (int)p->sact.size() < 2 * ns) {
    TVS_CUDA(cudaDeviceSynchronize());  // buffers may be in use by earlier forwards
    for (void* q : p->sact)
      if (q) TVS_CUDA(cudaFree(q));
    p->sact.assign(2 * p->streams.size(), nullptr);
    const size_t nbytes = std::max(bytes, p->sact_bytes);
    for (auto& q : p->sact) TVS_CUDA(cudaMalloc(&q, nbytes));
    p->sact_bytes = nbytes;
  }
}

// Work items of the layer-stack kernel for (B, strips, layers): a topological
// order (an item only depends on layer j-1 items of its image, which sort
// before it), uploaded once per shape.
const int2* stack_items(tvs_plan* p, int B, int strips, int L, cudaStream_t st) {
  const long long key[4] = {B, strips, L, p->stack_skew};
  if (std::equal(key, key + 4, p->items_key)) return p->items;
  const size_t n = (size_t)B * strips * L;
  std::vector<std::array<long long, 4>> v;
  v.reserve(n);
  const long long A = std::max(1, p->stack_skew);
  for (int i = 0; i < B; ++i)
    for (int j = 0; j < L; ++j)
      for (int s = 0; s < strips; ++s) v.push_back({i * A + j, j, s, i});
  std::sort(v.begin(), v.end());
  std::vector<int2> h(n);
  for (size_t k = 0; k < n; ++k) h[k] = make_int2((int)v[k][3], (int)(v[k][1] << 16 | v[k][2]));
  if (n > p->items_cap) {
    TVS_CUDA(cudaStreamSynchronize(st));
    if (p->items) TVS_CUDA(cudaFree(p->items));
    p->items = nullptr;
    p->items_cap = 0;
    TVS_CUDA(cudaMalloc(&p->items, n * sizeof(int2)));
    p->items_cap = n;
  }
  TVS_CUDA(cudaStreamSynchronize(st));  // a running stack kernel may still read the old table
  TVS_CUDA(cudaMemcpy(p->items, h.data(), n * sizeof(int2), cudaMemcpyHostToDevice));
  std::copy(key, key + 4, p->items_key);
  return p->items;
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
template <typename F>
void timed_launch(tvs_plan* p, cudaStream_t st, int kind, double flops, F&& f) {
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
               cudaStream_t st, void* const* act, int max_ctas) {
  const bool fast = p->tc_path();
  const bool split = p->split_path();
  const bool wide = p->wide_path();
  const int C = p->channels;
  const double px = (double)B * H * W;
  // layer stack (FAST path): every CTA of the persistent grid must be resident
  // at once, so only on the full device grid of the single-stream path
  bool stack = false;
  if (fast && p->stack != 0 && p->unfused_conv0 && !p->pair_fuse && !p->pair2 && max_ctas >= p->num_sms) {
    const int us0 = p->unshuffle;
    const long long items = (long long)B * ((W / us0 + tvs::kStripPx - 1) / tvs::kStripPx) * p->n_hidden();
    // auto: enough items per SM, and a last round that is nearly full (the
    // items are equal-length columns, a partial round idles SMs)
    const long long rounds = (items + p->num_sms - 1) / p->num_sms;
    stack = p->stack == 1 || (items >= (long long)tvs_plan::kStackMinItems * p->num_sms &&
                              (double)items >= 0.95 * (double)(rounds * p->num_sms));
  }
  if (stack) {
    const int us0 = p->unshuffle;
    const size_t n = (size_t)B * ((W / us0 + tvs::kStripPx - 1) / tvs::kStripPx) * (H / us0);
    if (n > p->rowcnt_n) {
      if (p->rowcnt) TVS_CUDA(cudaFree(p->rowcnt));
      p->rowcnt = nullptr;
      p->rowcnt_n = 0;
      TVS_CUDA(cudaMalloc(&p->rowcnt, n * sizeof(int)));
      p->rowcnt_n = n;
    }
    TVS_CUDA(cudaMemsetAsync(p->rowcnt, 0, n * sizeof(int), st));
  }
  // K1 (the FAST path can fuse it into the first hidden layer's producer)
  // wide fast stack: hidden layer j reads an fp16 hi/lo pair for j < P, single
  // fp16 after (j == n_hidden is the head); P = n_hidden keeps every layer paired
  const int nh = p->n_hidden();
  const int P = std::max(0, std::min(p->wide_pair_layers, nh));
  auto pair_in = [&](int j) { return j < P || P >= nh; };
  const int fmt = fast ? tvs::kActF16
                       : (split ? tvs::kActSplit : (wide ? (pair_in(0) ? tvs::kActSplit : tvs::kActF16) : tvs::kActF32));
  const int us = p->unshuffle;  // 2: the layer stack runs on the (H/2, W/2) grid
  if (us == 2 && p->conv0_tc)
    timed_launch(p, st, TVS_KIND_CONV0, px * 2.0 * 9 * C, [&] {
      return tvs::launch_conv0_tc(4, x, act[0], p->c0pack, p->c0bias, B, H / 2, W / 2, p->num_sms, st);
    });
  else if (us == 2)
    timed_launch(p, st, TVS_KIND_CONV0, px * 2.0 * 9 * C,
                 [&] { return tvs::launch_conv0_unshuffle(x, act[0], p->w0u, p->b0u, B, H / 2, W / 2, st); });
  else if (fast && p->unfused_conv0 && p->conv0_tc)
    timed_launch(p, st, TVS_KIND_CONV0, px * 2.0 * 9 * C, [&] {
      return tvs::launch_conv0_tc(1, x, act[0], p->c0pack, p->c0bias, B, H, W, p->num_sms, st);
    });
  else if (!fast || p->unfused_conv0)
    timed_launch(p, st, TVS_KIND_CONV0, px * 2.0 * 9 * C,
                 [&] { return tvs::launch_conv0(fmt, C, x, act[0], p->conv0, B, H, W, st); });
  // K2 x (depth-2), K3
  int cur = 0;
  if (wide) {
    // wide variant: split activations (hi 128 | lo 128 halves per pixel), groups
    // of 4 CTAs per strip-row range (one 32-channel quarter each)
    const int strips = (W + tvs::kStripPx - 1) / tvs::kStripPx;
    CUtensorMap pair_map[2], single_map[2];
    for (int i = 0; i < 2; ++i) {
      pair_map[i] = make_act_map(act[i], B, H, W, tvs::kHaloPx, 256);
      single_map[i] = make_act_map(act[i], B, H, W, tvs::kHaloPx, 128);
    }
    auto geom = [&](int r0, int nrows) {
      tvs::ConvArgs a{};
      a.B = B; a.H = H; a.W = W; a.strips = strips;
      a.row0 = r0; a.rows = nrows; a.nsub = 1;
      return a;
    };
    for (int l = 0; l < p->n_hidden(); ++l) {
      tvs::ConvArgs a = geom(0, H);
      a.wpack = p->wpack + (size_t)l * tvs::conv_wpack_wide_bytes(false);
      a.shift = p->bhid + (size_t)l * C;
      a.nshift = C;
      a.act_out = static_cast<uint8_t*>(act[cur ^ 1]);
      a.out_single = pair_in(l + 1) ? 0 : 1;
      const CUtensorMap& m = pair_in(l) ? pair_map[cur] : single_map[cur];
      // 4 (quarters) or 2 (halves) CTAs per strip-row range: size the grid by groups
      const int mode = pair_in(l) ? 5 : (p->wide_halves ? 11 : 9);
      const int parts = mode == 11 ? 2 : 4;
      const int grid = parts * std::max(1, std::min(max_ctas / parts, conv_grid(max_ctas, a)));
      timed_launch(p, st, TVS_KIND_HIDDEN, px * 2.0 * 9 * C * C,
                   [&] { return tvs::launch_conv_tc(mode, m, m, a, nullptr, grid, st); });
      cur ^= 1;
    }
    tvs::ConvArgs a = geom(row0, rows);
    a.wpack = p->hpack;
    a.shift = p->bh;
    a.nshift = p->out_bands;
    a.x = x; a.bands = bands; a.closure = closure; a.K = p->out_bands;
    const int grid = conv_grid(max_ctas, a);
    const CUtensorMap& mh = pair_in(nh) ? pair_map[cur] : single_map[cur];
    timed_launch(p, st, TVS_KIND_HEAD, (double)B * rows * W * 2.0 * 9 * C * p->out_bands,
                 [&] { return tvs::launch_conv_tc(pair_in(nh) ? 6 : 10, mh, mh, a, nullptr, grid, st); });
  } else if (split) {
    // fp32-accurate: split-operand tcgen05 layers on fp16 hi|lo pair rows
    const int strips = (W + tvs::kStripPx - 1) / tvs::kStripPx;
    CUtensorMap in_map[2];
    for (int i = 0; i < 2; ++i) in_map[i] = make_act_map(act[i], B, H, W, tvs::kHaloPx, 128);
    auto geom = [&](int r0, int nrows) {
      tvs::ConvArgs a{};
      a.B = B; a.H = H; a.W = W; a.strips = strips;
      a.row0 = r0; a.rows = nrows; a.nsub = 1;
      return a;
    };
    for (int l = 0; l < p->n_hidden(); ++l) {
      tvs::ConvArgs a = geom(0, H);
      a.wpack = p->wpack + (size_t)l * tvs::conv_wpack_split_bytes();
      a.shift = p->bhid + (size_t)l * tvs::kC;
      a.nshift = tvs::kC;
      a.act_out = static_cast<uint8_t*>(act[cur ^ 1]);
      const int grid = conv_grid(max_ctas, a);
      timed_launch(p, st, TVS_KIND_HIDDEN, px * 2.0 * 9 * 64 * 64,
                   [&] { return tvs::launch_conv_tc(3, in_map[cur], in_map[cur], a, nullptr, grid, st); });
      cur ^= 1;
    }
    tvs::ConvArgs a = geom(row0, rows);
    a.wpack = p->hpack;
    a.shift = p->bh;
    a.nshift = p->out_bands;
    a.x = x; a.bands = bands; a.closure = closure; a.K = p->out_bands;
    const int grid = conv_grid(max_ctas, a);
    timed_launch(p, st, TVS_KIND_HEAD, (double)B * rows * W * 2.0 * 9 * 64 * p->out_bands,
                 [&] { return tvs::launch_conv_tc(4, in_map[cur], in_map[cur], a, nullptr, grid, st); });
  } else if (fast) {
    const int Hg = H / us, Wg = W / us;  // layer grid (half-res when unshuffled)
    const double pxg = px / (us * us);
    const int strips = (Wg + tvs::kStripPx - 1) / tvs::kStripPx;
    CUtensorMap in_map[2], out_map[2];
    for (int i = 0; i < 2; ++i) {
      in_map[i] = make_act_map(act[i], B, Hg, Wg, tvs::kHaloPx);
      out_map[i] = make_act_map(act[i], B, Hg, Wg, 32);
    }
    auto geom = [&](int r0, int nrows) {
      tvs::ConvArgs a{};
      a.B = B; a.H = Hg; a.W = Wg; a.strips = strips;
      a.row0 = r0; a.rows = nrows;
      return a;
    };
    const bool fuse0 = !p->unfused_conv0;
    if (fuse0) cur = 1;  // the first hidden layer reads x and writes act[0]
    // fused layer pairs: strips form a cluster (<= 8 CTAs), enough rows per cluster
    const int S = strips;
    const bool pairs = p->pair_fuse && !fuse0 && S <= 8 &&
                       (long long)B * Hg >= 16LL * std::max(1, max_ctas / S);
    int l0 = 0;
    if (stack) {
      tvs::ConvArgs a = geom(0, Hg);
      a.wpack = p->wpack;
      a.shift = p->bhid;
      a.nshift = tvs::kC;
      a.nlayers = p->n_hidden();
      a.rowcnt = p->rowcnt;
      a.items = stack_items(p, B, strips, a.nlayers, st);
      if (const char* e = std::getenv("TVS_CONV_DBG")) a.dbg = std::atoi(e);
      tvs::StackMaps sm{};
      sm.in1 = in_map[1];
      sm.out0 = out_map[0];
      const long long items = (long long)B * strips * a.nlayers;
      const int grid = (int)std::min<long long>(p->num_sms, items);
      timed_launch(p, st, TVS_KIND_HIDDEN, a.nlayers * pxg * 2.0 * 9 * 64 * 64,
                   [&] { return tvs::launch_conv_stack(in_map[0], out_map[1], sm, a, grid, st); });
      l0 = a.nlayers;
      cur = l0 & 1;
    }
    if (pairs) {
      for (; l0 + 1 < p->n_hidden(); l0 += 2) {
        tvs::PairArgs pa{};
        pa.B = B; pa.H = Hg; pa.W = Wg; pa.S = S;
        pa.wpack0 = p->wpack + (size_t)l0 * tvs::conv_wpack_bytes(false);
        pa.wpack1 = p->wpack + (size_t)(l0 + 1) * tvs::conv_wpack_bytes(false);
        pa.shift0 = p->bhid + (size_t)l0 * tvs::kC;
        pa.shift1 = p->bhid + (size_t)(l0 + 1) * tvs::kC;
        pa.act_out = static_cast<uint8_t*>(act[cur ^ 1]);
        if (const char* e = std::getenv("TVS_PAIR_DBG")) pa.dbg = std::atoi(e);
        timed_launch(p, st, TVS_KIND_HIDDEN, 2 * pxg * 2.0 * 9 * 64 * 64,
                     [&] { return tvs::launch_conv_pair(in_map[cur], pa, max_ctas, st); });
        cur ^= 1;
      }
    }
    for (int l = l0; l < p->n_hidden(); ++l) {
      tvs::ConvArgs a = geom(0, Hg);
      a.wpack = p->wpack + (size_t)l * tvs::conv_wpack_bytes(false);
      a.shift = p->bhid + (size_t)l * tvs::kC;
      a.nshift = tvs::kC;
      a.x = x;
      const int grid = conv_grid(max_ctas, a);
      const bool first = fuse0 && l == 0;
      a.reverse = (p->l2_reverse_sub > 1) && (l & 1);
      a.nsub = p->l2_reverse_sub;
      a.l2_hints = p->l2_hints;
      if (const char* e = std::getenv("TVS_CONV_DBG")) a.dbg = std::atoi(e);
      const bool use_pair2 = p->pair2 && !first && strips % 2 == 0 && p->wpack2;
      if (use_pair2) {
        a.wpack = p->wpack2 + (size_t)l * tvs::conv_pair2_wpack_bytes();
        const long long tp = (long long)B * (strips / 2) * Hg;
        const int grid2 = 2 * (int)std::max(1LL, std::min<long long>(max_ctas / 2, (tp + 2) / 3));
        timed_launch(p, st, TVS_KIND_HIDDEN, pxg * 2.0 * 9 * 64 * 64,
                     [&] { return tvs::launch_conv_pair2(in_map[cur], out_map[cur ^ 1], a, grid2, st); });
      } else {
        timed_launch(p, st, TVS_KIND_HIDDEN, pxg * 2.0 * 9 * 64 * 64 + (first ? pxg * 2.0 * 9 * 64 : 0.0), [&] {
          return tvs::launch_conv_tc(first ? 2 : 0, in_map[cur], out_map[cur ^ 1], a, first ? &p->conv0 : nullptr,
                                     grid, st);
        });
      }
      cur ^= 1;
    }
    tvs::ConvArgs a = geom(row0 / us, rows / us);
    a.wpack = p->hpack;
    a.shift = p->bh;
    a.nshift = p->out_bands * us * us;
    a.x = x; a.bands = bands; a.closure = closure; a.K = p->out_bands;
    a.reverse = (p->l2_reverse_sub > 1) && (p->n_hidden() & 1);
    a.nsub = p->l2_reverse_sub;
    const int grid = conv_grid(max_ctas, a);
    timed_launch(p, st, TVS_KIND_HEAD, (double)B * rows * W * 2.0 * 9 * 64 * p->out_bands,
                 [&] { return tvs::launch_conv_tc(us == 2 ? 7 : 1, in_map[cur], in_map[cur], a, nullptr, grid, st); });
  } else {
    for (int l = 0; l < p->n_hidden(); ++l) {
      timed_launch(p, st, TVS_KIND_HIDDEN, px * 2.0 * 9 * C * C, [&] {
        return tvs::launch_hidden_f32(C, (const float*)act[cur], (float*)act[cur ^ 1],
                                      p->whid + (size_t)l * C * C * 9, p->shid + (size_t)l * C,
                                      p->bhid + (size_t)l * C, B, H, W, st);
      });
      cur ^= 1;
    }
    timed_launch(p, st, TVS_KIND_HEAD, (double)B * rows * W * 2.0 * 9 * C * p->out_bands, [&] {
      return tvs::launch_head_f32(C, (const float*)act[cur], x, p->wh, p->bh, bands, closure, B, H, W, p->out_bands,
                                  row0, rows, st);
    });
  }
}

void forward_impl(tvs_plan* p, const float* x, float* bands, float* closure, int B, int H, int W, int row0, int rows,
                  cudaStream_t st) {
  if (!p->weights_ready) throw TvsError(TVS_E_STATE, "tvs_forward before tvs_plan_set_weights");
  if (!x || !bands) throw TvsError(TVS_E_INVALID, "null x/bands pointer");
  if (B < 0 || H < 1 || W < 1) throw TvsError(TVS_E_INVALID, "bad shape B/H/W");
  if (rows < 0) { row0 = 0; rows = H; }
  if (row0 < 0 || rows < 1 || row0 + rows > H) throw TvsError(TVS_E_INVALID, "bad valid row window");
  if (p->unshuffle == 2 && (H % 2 || W % 2 || row0 % 2 || rows % 2))
    throw TvsError(TVS_E_INVALID, "unshuffle = 2 needs even H, W and an even row window");
  p->last_launches = 0;
  if (B == 0) return;
  ensure_device(p);
  const size_t per_img = (size_t)H * W * p->act_px_bytes() / ((size_t)p->unshuffle * p->unshuffle);
  const size_t in_img = (size_t)H * W, out_img = (size_t)rows * W;
  // concurrent L2-resident chunks: only when an image fits the chunk budget
  const int S = p->tc_path() ? std::min(p->n_streams, B) : 1;
  if (S > 1 && per_img <= p->l2_chunk_bytes) {
    const int cb = (int)std::min<size_t>((size_t)B, std::max<size_t>(1, p->l2_chunk_bytes / per_img));
    const int nchunks = (B + cb - 1) / cb;
    const int ns = std::min(S, nchunks);
    ensure_streams(p, ns, per_img * cb);
    TVS_CUDA(cudaEventRecord(p->fork_ev, st));
    for (int s = 0; s < ns; ++s) TVS_CUDA(cudaStreamWaitEvent(p->streams[s], p->fork_ev, 0));
    const int max_ctas = std::max(1, p->num_sms / ns);
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % ns, b0 = c * cb, nb = std::min(cb, B - b0);
      run_chunk(p, x + b0 * in_img, bands + (size_t)b0 * p->out_bands * out_img,
                closure ? closure + b0 * out_img : nullptr, nb, H, W, row0, rows, p->streams[s], &p->sact[2 * s],
                max_ctas);
    }
    for (int s = 0; s < ns; ++s) {
      TVS_CUDA(cudaEventRecord(p->join_ev[s], p->streams[s]));
      TVS_CUDA(cudaStreamWaitEvent(st, p->join_ev[s], 0));
    }
    return;
  }
  int cb = (int)std::max<size_t>(1, p->chunk_budget / std::max<size_t>(per_img, 1));
  cb = std::min(cb, B);
  ensure_act(p, per_img * cb);
  for (int b0 = 0; b0 < B; b0 += cb) {
    const int nb = std::min(cb, B - b0);
    run_chunk(p, x + b0 * in_img, bands + (size_t)b0 * p->out_bands * out_img,
              closure ? closure + b0 * out_img : nullptr, nb, H, W, row0, rows, st, p->act, p->num_sms);
  }
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return TVS_OK;
  } catch (const TvsError& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return TVS_E_CUDA;
  } catch (...) {
    g_last_error = "unknown error";
    return TVS_E_CUDA;
  }
}

}  // namespace

extern "C" {

int tvs_abi_version(void) { return TVS_ABI_VERSION; }

const char* tvs_last_error(void) { return g_last_error.c_str(); }

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
    TVS_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    TVS_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
      throw TvsError(TVS_E_UNSUPPORTED, "libtvsb200 is built for sm_100a (B200) only");
    auto* p = new tvs_plan();
    p->device = device; p->depth = depth; p->channels = channels; p->out_bands = out_bands; p->mode = mode;
    p->unshuffle = unshuffle;
    if (unshuffle == 2) p->unfused_conv0 = true;
    p->num_sms = prop.multiProcessorCount;
    if (const char* e = std::getenv("TVS_CHUNK_MB")) p->chunk_budget = (size_t)std::atoll(e) << 20;
    if (const char* e = std::getenv("TVS_STREAMS")) p->n_streams = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("TVS_REVERSE_SUB")) p->l2_reverse_sub = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("TVS_L2_CHUNK_MB")) p->l2_chunk_bytes = (size_t)std::atoll(e) << 20;
    if (const char* e = std::getenv("TVS_FUSE_CONV0")) p->unfused_conv0 = std::atoi(e) == 0;
    if (const char* e = std::getenv("TVS_FP32_CUDA")) p->fp32_split = std::atoi(e) == 0;
    if (const char* e = std::getenv("TVS_L2_HINTS")) p->l2_hints = std::atoi(e);
    if (const char* e = std::getenv("TVS_PAIR2")) p->pair2 = std::atoi(e) != 0;
    if (const char* e = std::getenv("TVS_CONV0_TC")) p->conv0_tc = std::atoi(e);
    if (const char* e = std::getenv("TVS_PAIR")) p->pair_fuse = std::atoi(e) != 0;
    if (const char* e = std::getenv("TVS_STACK")) p->stack = std::atoi(e);
    if (const char* e = std::getenv("TVS_WIDE_PAIR")) p->wide_pair_layers = std::atoi(e);
    if (const char* e = std::getenv("TVS_WIDE_HALVES")) p->wide_halves = std::atoi(e) != 0;
    if (const char* e = std::getenv("TVS_STACK_SKEW")) p->stack_skew = std::atoi(e);
    if (const char* e = std::getenv("TVS_WIDE_CUDA")) p->wide_cuda = std::atoi(e) != 0;
    try {
      TVS_CUDA(tvs::configure_kernels());
      const int nh = depth - 2;
      TVS_CUDA(cudaMalloc(&p->wh, (size_t)out_bands * channels * 9 * 4));
      TVS_CUDA(cudaMalloc(&p->bh, (size_t)out_bands * unshuffle * unshuffle * 4));  // head bias (4K if unshuffled)
      TVS_CUDA(cudaMalloc(&p->bhid, (size_t)nh * channels * 4));
      TVS_CUDA(cudaMalloc(&p->shid, (size_t)nh * channels * 4));
      if (p->tc_path()) {
        TVS_CUDA(cudaMalloc(&p->wpack, (size_t)nh * tvs::conv_wpack_bytes(false)));
        TVS_CUDA(cudaMalloc(&p->hpack, unshuffle == 2 ? tvs::conv_wpack_unshuf_head_bytes() : tvs::conv_wpack_bytes(true)));
        if (unshuffle == 2) {
          TVS_CUDA(cudaMalloc(&p->w0u, (size_t)channels * 36 * 4));
          TVS_CUDA(cudaMalloc(&p->b0u, (size_t)channels * 4));
        }
      } else if (p->split_path()) {
        TVS_CUDA(cudaMalloc(&p->wpack, (size_t)nh * tvs::conv_wpack_split_bytes()));
        TVS_CUDA(cudaMalloc(&p->hpack, tvs::conv_wpack_bytes(true)));
      } else if (p->wide_path()) {
        TVS_CUDA(cudaMalloc(&p->wpack, (size_t)nh * tvs::conv_wpack_wide_bytes(false)));
        TVS_CUDA(cudaMalloc(&p->hpack, tvs::conv_wpack_wide_bytes(true)));
      } else
        TVS_CUDA(cudaMalloc(&p->whid, (size_t)nh * channels * channels * 9 * 4));
    } catch (...) {
      free_all(p);
      delete p;
      throw;
    }
    *out_plan = p;
  });
}

int tvs_plan_set_weights(tvs_plan* p, const float* const* w_dev, const float* const* scale_dev,
                         const float* const* shift_dev, int n_layers, void* stream) {
  return guarded([&] {
    if (!p || !w_dev || !shift_dev) throw TvsError(TVS_E_INVALID, "null argument");
    if (n_layers != p->depth) throw TvsError(TVS_E_INVALID, "n_layers must equal depth");
    for (int i = 0; i < n_layers; ++i)
      if (!w_dev[i] || !shift_dev[i]) throw TvsError(TVS_E_INVALID, "null weight/shift pointer");
    ensure_device(p);
    cudaStream_t st = (cudaStream_t)stream;
    const int nh = p->n_hidden();
    auto scale_of = [&](int i) -> const float* { return scale_dev ? scale_dev[i] : nullptr; };
    if (scale_of(0) || scale_of(p->depth - 1))
      throw TvsError(TVS_E_UNSUPPORTED, "conv0/head take no BatchNorm scale (model.py:37,44)");
    const int C = p->channels;
    if (p->unshuffle == 2) {  // conv0 Conv2d(4, C) on the device; head Conv2d(C, 4K) packed below
      TVS_CUDA(cudaMemcpyAsync(p->w0u, w_dev[0], (size_t)C * 36 * 4, cudaMemcpyDeviceToDevice, st));
      TVS_CUDA(cudaMemcpyAsync(p->b0u, shift_dev[0], (size_t)C * 4, cudaMemcpyDeviceToDevice, st));
    } else {
      TVS_CUDA(cudaMemcpyAsync(p->conv0.w, w_dev[0], (size_t)C * 9 * 4, cudaMemcpyDeviceToHost, st));
      TVS_CUDA(cudaMemcpyAsync(p->conv0.b, shift_dev[0], (size_t)C * 4, cudaMemcpyDeviceToHost, st));
      TVS_CUDA(cudaStreamSynchronize(st));  // conv0 weights are kernel parameters (host side)
      TVS_CUDA(cudaMemcpyAsync(p->wh, w_dev[p->depth - 1], (size_t)p->out_bands * C * 9 * 4,
                               cudaMemcpyDeviceToDevice, st));
    }
    if (p->tc_path()) {  // K1 on tcgen05: TF32 hi/lo B pack + bias
      const int in_ch = p->unshuffle == 2 ? 4 : 1;
      if (!p->c0pack) TVS_CUDA(cudaMalloc(&p->c0pack, tvs::conv0_tc_pack_bytes(in_ch)));
      if (!p->c0bias) TVS_CUDA(cudaMalloc(&p->c0bias, 64 * sizeof(float)));
      TVS_CUDA(tvs::launch_pack_conv0_tc(w_dev[0], in_ch, p->c0pack, st));
      TVS_CUDA(cudaMemcpyAsync(p->c0bias, shift_dev[0], 64 * sizeof(float), cudaMemcpyDeviceToDevice, st));
    }
    TVS_CUDA(cudaMemcpyAsync(p->bh, shift_dev[p->depth - 1], (size_t)p->out_bands * p->unshuffle * p->unshuffle * 4,
                             cudaMemcpyDeviceToDevice, st));
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
        if (p->pair2 && p->unshuffle == 1) {
          if (!p->wpack2) TVS_CUDA(cudaMalloc(&p->wpack2, (size_t)nh * tvs::conv_pair2_wpack_bytes()));
          TVS_CUDA(tvs::launch_pack_hidden_pair2(w_dev[l + 1], dst_scale,
                                                 p->wpack2 + (size_t)l * tvs::conv_pair2_wpack_bytes(), st));
        }
      } else if (p->split_path()) {
        TVS_CUDA(tvs::launch_pack_hidden_split(w_dev[l + 1], dst_scale,
                                               p->wpack + (size_t)l * tvs::conv_wpack_split_bytes(), st));
      } else if (p->wide_path()) {  // pair-input layers: quarters (mode 5); single-input: halves (mode 11)
        const int P = std::max(0, std::min(p->wide_pair_layers, nh));
        const bool pair_in = l < P || P >= nh;
        TVS_CUDA(tvs::launch_pack_hidden_wide(w_dev[l + 1], dst_scale,
                                              p->wpack + (size_t)l * tvs::conv_wpack_wide_bytes(false), st,
                                              pair_in || !p->wide_halves ? 4 : 2));
      } else {
        TVS_CUDA(cudaMemcpyAsync(p->whid + (size_t)l * C * C * 9, w_dev[l + 1], (size_t)C * C * 9 * 4,
                                 cudaMemcpyDeviceToDevice, st));
      }
    }
    if (p->unshuffle == 2) {
      TVS_CUDA(tvs::launch_pack_head_unshuf(w_dev[p->depth - 1], 4 * p->out_bands, p->hpack, st));
    } else if (p->tc_path() || p->split_path()) {
      TVS_CUDA(tvs::launch_pack_head_f16(w_dev[p->depth - 1], p->out_bands, p->hpack, st));
    }
    if (p->wide_path()) TVS_CUDA(tvs::launch_pack_head_wide(w_dev[p->depth - 1], p->out_bands, p->hpack, st));
    p->weights_ready = true;
  });
}

int tvs_forward(tvs_plan* p, const float* x, float* bands, float* closure_or_null, int B, int H, int W,
                int valid_row0, int valid_rows, void* stream) {
  return guarded([&] {
    if (!p) throw TvsError(TVS_E_INVALID, "null plan");
    forward_impl(p, x, bands, closure_or_null, B, H, W, valid_row0, valid_rows, (cudaStream_t)stream);
  });
}

int tvs_forward_host(tvs_plan* p, const float* x_host, float* bands_host, float* closure_host_or_null, int B, int H,
                     int W, void* stream) {
  return guarded([&] {
    if (!p || !x_host || !bands_host) throw TvsError(TVS_E_INVALID, "null argument");
    if (B < 0 || H < 1 || W < 1) throw TvsError(TVS_E_INVALID, "bad shape B/H/W");
    ensure_device(p);
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
  });
}

int tvs_last_launch_count(const tvs_plan* p) { return p ? p->last_launches : 0; }

int tvs_profile_enable(tvs_plan* p, int on) {
  return guarded([&] {
    if (!p) throw TvsError(TVS_E_INVALID, "null plan");
    ensure_device(p);
    drain_profile(p);
    for (int k = 0; k < 3; ++k) { p->prof_ms[k] = 0; p->prof_n[k] = 0; p->prof_flops[k] = 0; }
    p->profiling = on != 0;
  });
}

int tvs_profile_read(tvs_plan* p, int kind, double* total_ms, long long* launches, double* flops) {
  return guarded([&] {
    if (!p || kind < 0 || kind > 2) throw TvsError(TVS_E_INVALID, "bad plan/kind");
    ensure_device(p);
    drain_profile(p);
    if (total_ms) *total_ms = p->prof_ms[kind];
    if (launches) *launches = p->prof_n[kind];
    if (flops) *flops = p->prof_flops[kind];
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

// diagnostics of the layer-stack kernel (not part of the public ABI): 1 if a
// row-flag wait timed out since the last reset (that forward's output is invalid)
int tvs_debug_stack(int reset) { return tvs::conv_stack_error(reset); }
int tvs_debug_cycles(unsigned long long* out, int reset) { return tvs::debug_cycles(out, reset); }

int tvs_plan_destroy(tvs_plan* p) {
  return guarded([&] {
    if (!p) return;
    cudaSetDevice(p->device);
    free_all(p);
    delete p;
  });
}

}  // extern "C"
