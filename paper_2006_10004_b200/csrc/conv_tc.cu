// conv_tc.cu — tcgen05 implicit-GEMM 3x3 convolutions over fp16 NHWC
// activations (sm_100a).  One kernel template, two epilogues:
//
//  K2 hidden layer  (Conv2d(64,64,3,p=1,no bias) -> BatchNorm2d(eval) -> ReLU,
//     /root/reference/pkg/trainer/src/tvsurrogate/model.py:40-43)
//     N block = 64 output channels, epilogue +shift, ReLU, fp16 -> TMA store.
//  K3 head          (Conv2d(64,K,3,p=1,bias), model.py:44, + closure plane
//     image - sum(bands), inference.py:34-42)
//     N block = 16 per dy = [8 cols W_hi | 8 cols W_lo] with W = W_hi + W_lo both
//     fp16 (exact split of the fp32 weight to ~2^-22), so the head stays
//     fp32-accurate on fp16 activations; epilogue sums hi+lo+bias and writes
//     fp32 NCHW bands (+ closure) for a row window.
//
// GEMM mapping (persistent CTAs, each owning an equal contiguous range of
// 128-px strip-rows, see SegIter):
//   * M = 128 output pixels of one row (TMEM lanes);
//   * the three dy taps are stacked along N: B = [W(dy=+1) | W(0) | W(-1)],
//     so one input row r updates the accumulators of output rows r-1, r, r+1,
//     which live in consecutive TMEM slots (slot = output-row sequence mod 8);
//     N = 3*NB >= 96 keeps the MMA off the shared-memory operand limit
//     (N=64 SS MMAs run at 2/3 rate on B200: tools/ubench_tcgen05.cu);
//   * K = 64 input channels x 3 dx taps; a dx tap is a 128 B shift of the A
//     descriptor start inside the SW128 input-row buffer (one 130-px halo
//     row loaded by TMA; OOB zero fill = Conv2d zero padding).
//   * The slot an input row touches for the first time is written with
//     accumulate=0 in that row's first K step (split into its own MMA), so
//     slots never need zeroing.
//
// Warp roles: w0 TMA producer, w1 TMEM alloc + single-thread MMA issuer,
// then kEpiGroups groups of 4 epilogue warps (output rows round-robin over the
// groups); every epilogue warp owns one TMEM lane quarter (32 pixels) and
// stores independently.
#include <algorithm>
#include <type_traits>

#include <cuda_fp8.h>

#include "common.cuh"
#include "sm100.cuh"

namespace tvs {

// Work partition: the output is a list of strip-rows ordered (image, strip,
// row) with rows restricted to the window [row0, row0+rows).  CTA i owns the
// contiguous range [i*T/G, (i+1)*T/G) of the T = B*strips*rows strip-rows, so
// every CTA gets the same number of output rows (+-1).  A range is walked as
// segments: maximal runs of consecutive rows inside one (image, strip) column.
struct Segment {
  int b, x0, ya, yb;
  int h;      // output-channel half (split hidden layer visits every segment twice)
  int layer;  // hidden layer of a layer-stack item (mode 8)
};
struct SegIter {
  long long cur, end;  // [cur, end): this CTA's strip-rows
  int nh = 1;          // visits per segment (2: once per output-channel half)
  bool pend = false;   // second visit of `last` outstanding
  Segment last;
  // `parts` = 4: the grid is split into groups of 4 CTAs (one per output-channel
  // quarter) that walk the same strip-row range
  TVS_DEV SegIter(const ConvArgs& a, int halves = 1, int parts = 1) : nh(halves) {
    const long long T = (long long)a.B * a.strips * a.rows;
    const long long part = blockIdx.x / parts, nparts = gridDim.x / parts;
    cur = T * part / nparts;
    end = T * (part + 1) / nparts;
  }
  TVS_DEV int first_layer_or0(const ConvArgs&) const { return 0; }
  TVS_DEV bool next(const ConvArgs& a, Segment& g) {
    if (pend) {
      g = last;
      g.h = 1;
      pend = false;
      return true;
    }
    if (cur >= end) return false;
    const long long col = cur / a.rows;
    const int y0 = (int)(cur - col * a.rows);
    const int n = (int)min((long long)(a.rows - y0), end - cur);
    g.b = (int)(col / a.strips);
    g.x0 = (int)(col % a.strips) * kStripPx;
    g.ya = a.row0 + y0;
    g.yb = g.ya + n;
    g.h = 0;
    g.layer = 0;
    cur += n;
    if (nh == 2) {
      last = g;
      pend = true;
    }
    return true;
  }
};

// Layer-stack work items (mode 8): item = output rows [ya, yb) of one strip of
// one hidden layer of one image (whole columns for big batches, row bands for
// small ones).  An item depends only on layer j-1 rows ya-1..yb of its image
// (strips s-1..s+1), so any order listing an image's layer j-1 items before
// its layer j items is topological.  CTA i walks entries i, i+G, i+2G, ... of
// the host-built table (stack_items in tvs_api.cu), which keeps every CTA's
// own sequence topologically sorted; then the minimal unfinished item is
// always the one its CTA is working on and has its inputs, so the persistent
// grid cannot deadlock while all G CTAs are co-resident (cooperative launch,
// 1 CTA/SM).  Entries with image -1 pad the table.
struct ItemIter {
  long long k, n;
  TVS_DEV ItemIter(const ConvArgs& a, int = 1, int = 1) {
    k = blockIdx.x;
    n = a.nitems;
    while (k < n && a.items[k].x < 0) k += gridDim.x;
  }
  TVS_DEV int first_layer_or0(const ConvArgs& a) const { return first_layer(a); }
  TVS_DEV int first_layer(const ConvArgs& a) const { return k < n ? a.items[k].y >> 16 : 0; }
  TVS_DEV bool next(const ConvArgs& a, Segment& g) {
    while (k < n && a.items[k].x < 0) k += gridDim.x;
    if (k >= n) return false;
    const int4 it = a.items[k];
    g.b = it.x;
    g.layer = it.y >> 16;
    g.x0 = (it.y & 0xffff) * kStripPx;
    g.ya = it.z;
    g.yb = it.w;
    g.h = 0;
    k += gridDim.x;
    return true;
  }
};

// TVS_CONV_DBG bit 15 (layer stack): MMA-issuer cycle accounting (sum over CTAs): [0] total,
// [1] waiting for a free accumulator slot, [2] waiting for the input row,
// [3] waiting for a layer's weights, [4] general-path rows, [5] fast-path rows,
// [6] elapsed ns (globaltimer), so [0] / [6] is the mean SM clock in GHz
__device__ unsigned long long g_dbg_cycles[8];
// kDbgTrace (layer stack, image 0, strip 0, rows < kTraceRows): [0][layer][row]
// gate passed (producer), [1][layer][row] input row landed (MMA issuer),
// [2][layer][row] output row published (epilogue), [3] accumulator ready
// (epilogue warp quarter 0), [4] TMA store issued; globaltimer ns
constexpr int kTraceKinds = 5, kTraceRows = 1024, kTraceLayers = 32;
__device__ unsigned long long g_trace[kTraceKinds][kTraceLayers][kTraceRows];
// Compiled in only by the diagnostics build (build.py --trace: -DTVS_STACK_TRACE,
// libtvsb200_trace.so): even untaken, the checks cost the issue-bound MMA
// thread ~2% of the config-2 stack (3.31 vs 3.25 ms, same box).
TVS_DEV void trace_mark(const ConvArgs& a, int kind, const Segment& g, int row) {
#ifdef TVS_STACK_TRACE
  if ((a.dbg & kDbgTrace) && g.b == 0 && g.x0 == 0 && row >= 0 && row < kTraceRows && g.layer < kTraceLayers)
    g_trace[kind][g.layer][row] = globaltimer_ns();
#endif
}
TVS_DEV void trace_cta(const ConvArgs& a, int kind) {
#ifdef TVS_STACK_TRACE
  if ((a.dbg & kDbgTrace) && threadIdx.x == 0 && blockIdx.x < kTraceRows)
    g_trace[kind][kTraceLayers - 1][blockIdx.x] = globaltimer_ns();
#endif
}

// Producer side of the layer stack: input row r of a layer-j item (j >= 1) is
// layer j-1's output row r of strips s-1..s+1 (the 130-px halo box reaches one
// pixel into each neighbour); it may be loaded once their 4 epilogue warps have
// stored it (count >= 4j).  A refresh reads kAhead consecutive row counters of
// every neighbour strip at once (independent loads, one L2 round trip) and
// remembers how far each is complete, so most rows need no memory access.
struct StackGate {
  static constexpr int kAhead = 8;
  int ready[3];  // last row known complete in strips s-1, s, s+1
  TVS_DEV void reset() { ready[0] = ready[1] = ready[2] = -1; }
  TVS_DEV void wait(const ConvArgs& a, const Segment& g, int r) { wait(a, g, r, 4 * g.layer); }
  TVS_DEV void wait(const ConvArgs& a, const Segment& g, int r, const int target) {
    const int s = g.x0 / kStripPx;
    const int* base = a.rowcnt + (long long)g.b * a.strips * a.H;
    bool refreshed = false;
    unsigned long long t0 = 0;
    for (uint32_t spins = 0;; ++spins) {
      int v[3][kAhead];
      bool need[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const int ss = s - 1 + d;
        need[d] = ss >= 0 && ss < a.strips && ready[d] < r;
        if (need[d]) {
          const int* f = base + (long long)ss * a.H + r;
#pragma unroll
          for (int i = 0; i < kAhead; ++i) v[d][i] = (r + i < a.H) ? ld_relaxed_gpu(f + i) : target;
        }
      }
      bool ok = true;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        if (!need[d]) continue;
        refreshed = true;
        int c = 0;
#pragma unroll
        for (int i = 0; i < kAhead; ++i)
          if (c == i && v[d][i] >= target) c = i + 1;
        ready[d] = r - 1 + c;
        ok = ok && c > 0;
      }
      if (ok) break;
      // watchdog: never hang.  Once any wait of this launch has expired the
      // output is invalid (the host reports it), so every later wait gives up
      // at once and the launch drains.
      if (ld_relaxed_gpu(a.abort)) return;
      if (!(a.dbg & kDbgSpinGate)) __nanosleep(32);
      if ((spins & 63u) == 63u) {
        const unsigned long long now = globaltimer_ns();
        if (t0 == 0) {
          t0 = now;
        } else if (now - t0 > a.watchdog_ns) {
          atomicExch(a.abort, 1);
          if (a.status) flag_set(a.status + kStatWatchdog);
          return;
        }
      }
    }
    if (refreshed) {  // acquire what the counters published, then hand it to the TMA (async) proxy
      fence_acq_rel_gpu();
      fence_proxy_async_global();
    }
  }
};

// Flag watcher of the layer stack (plan option stack_watcher, default on): a
// dedicated warp walks the CTA's items like the producer and keeps polling
// the row flags of the rows the producer will load next (StackGate's refresh,
// 8 rows x 3 strips per round trip), publishing progress in shared memory as
// (item ordinal << 32 | last ready row + 1) with a CTA-scope release after its
// gpu-scope acquire.  The TMA producer then only spins on shared memory, so a
// flag round trip is no longer serialised with every row it issues: when a
// layer runs right behind the one before it (batch 1, row bands) the
// producer's row rate was bounded by the poll latency and each layer trailed
// the previous one a little more (tools/stack_trace.py).
struct StackWatcher {
  TVS_DEV static void run(const ConvArgs& a, unsigned long long* ready) {
    ItemIter it(a);
    Segment g;
    StackGate gate;
    unsigned long long ord = 0;
    bool gave_up = false;
    while (it.next(a, g)) {
      const int r0 = max(g.ya - 1, 0), r1 = min(g.yb, a.H - 1);
      if (g.layer > 0 && !(a.dbg & 1) && !gave_up) {
        gate.reset();
        for (int r = r0; r <= r1;) {
          gate.wait(a, g, r);  // gpu-scope acquire: row r (and what the refresh saw after it) is ready
          if (ld_relaxed_gpu(a.abort)) { gave_up = true; break; }
          const int s = g.x0 / kStripPx;
          int last = r1;
#pragma unroll
          for (int d = 0; d < 3; ++d)
            if (s - 1 + d >= 0 && s - 1 + d < a.strips) last = min(last, gate.ready[d]);
          last = max(last, r);
          st_release_cta_shared(ready, (ord << 32) | (unsigned long long)(last + 1));
          r = last + 1;
        }
      }
      // item done (or ungated): everything of it is ready
      ++ord;
      st_release_cta_shared(ready, ord << 32);
    }
  }
};

// kMode: 0 = hidden layer, 1 = head,
// 3 / 4 = fp32-accurate hidden layer / head on split operands: activations
// are stored as an fp16 pair (hi = RN(a), lo = RN(a - hi): channels 0-63 and
// 64-127 of a 256 B/px NHWC row), weights as hi/lo fp16 packs scaled by 2^8
// (keeps lo normal), and every tap runs three products hi*hi + lo*hi + hi*lo
// (head: two, its B pack already carries hi|lo columns) into the same fp32
// TMEM accumulators; the epilogue unscales and re-splits.
// 5 / 6 = the wide variant (128 channels, fast mode) hidden layer / head on
// split activations (hi/lo fp16 pairs) and single fp16 weights: fp16 rounding
// of the activations alone would cost 1.06e-2 over 26 layers (gate 1e-2).
// Mode 5 CTAs come in groups of 4, one 32-output-channel quarter each (its
// 72 KB weight slice stays resident; the 4 CTAs share input rows via L2).
// 7 = head of the opt-in unshuffle = 2 variant (fast mode): Conv2d(C, 4K)
// with N block 64 = [32 hi | 32 lo] columns and pixel_shuffle folded into the
// band stores (head channel k*4 + i*2 + j -> band k at (2y+i, 2x+j)).
// 9 / 10 = the wide variant's hidden layer / head on SINGLE fp16 input
// activations (one pass; mode 9's output is a pair or single per a.out_single):
// the fast wide stack stores the first layers' activations as pairs and the
// rest as single fp16 (tools/emulate_wide.py), trading MMA work for accuracy.
// 8 = the whole fast hidden stack in one persistent launch (mode 0's pipeline
// over ItemIter work items): the weights are reloaded when a CTA moves to an
// item of another layer, and layer j's input rows are gated on row flags of
// layer j-1 (stack_wait_row), so consecutive layers run concurrently a few
// rows apart and the activations pass between them through L2.
template <int kMode>
struct ConvCfg {
  static constexpr bool kStack = kMode == 8;
  static constexpr bool kSplit = (kMode >= 3 && kMode <= 6) || kMode == 12 || kMode == 13;
  // 12 = the fp32-accurate hidden layer on CTA PAIRS (a cluster of 2): each CTA
  // computes one 32-channel half of the same strip-rows, the input rows are
  // TMA-multicast to both (each CTA loads one of the hi / lo boxes), and each
  // CTA keeps only its half's weights, so the ring is 4 deep instead of 2 and no
  // row is read twice (mode 3 visits every segment once per half)
  static constexpr bool kPairH = kMode == 12 || kMode == 13;
  // 13 = mode 12 with the auxiliary epilogue paths compiled in (raw fp32 output,
  // a second input block's partial sums added: the wide fp32 mode's 2 x 2 blocks).
  // Carrying them as run-time branches cost the plain mode 12 epilogue 11%
  // (825 vs 742 us per config-2 layer), so the plain mode compiles them out.
  static constexpr bool kAux = kMode != 12;
  // CTAs per cluster: mode 12 pairs; the wide pair-input layer (mode 5) runs
  // its 4 output-channel quarters of a strip-row range as one cluster, each
  // input row TMA-multicast to all four (CTAs 0-2 load one of its 3 boxes)
  // instead of each CTA fetching it from L2 (build knob TVS_WIDE_MCAST, off:
  // the cluster runs the four CTAs in lockstep per input row, config 5-wide
  // 91 vs 119 MP/s)
  static constexpr int kCluster = kPairH ? 2 : ((kMode == 5 && TVS_WIDE_MCAST) ? 4 : 1);
  static constexpr bool kUnshuf = kMode == 7;
  static constexpr bool kHead = kMode == 1 || kMode == 4 || kMode == 6 || kMode == 7 || kMode == 10;
  static constexpr bool kWide = kMode == 5 || kMode == 6 || kMode == 9 || kMode == 10 || kMode == 11;
  static constexpr bool kQuarters = kMode == 5 || kMode == 9;
  // mode 11: wide single-input layer split into output-channel HALVES (pairs of
  // CTAs, 64 channels each, N = 192 dy-stacked MMAs at full rate) instead of
  // quarters (N = 96, shared-memory-operand bound)
  static constexpr bool kWideHalves = kMode == 11;
  static constexpr bool kPartsW = kQuarters || kWideHalves;  // wide output-channel partition
  static constexpr int kCin = kWide ? 128 : 64;
  static constexpr int kKBlk = kCin / 64;        // 64-channel K blocks (one SW128 row buffer each)
  static constexpr int kKSteps = 4 * kKBlk;      // K16 steps per tap
  static constexpr int kMmaWarp = 1;  // warp 0: TMA producer
  static constexpr int kEpiWarp0 = 2;
  // plain fp16 hidden layer (modes 0 / 8): epilogue groups and ring depth are
  // build-time knobs (4 groups on a 5-deep ring measured no faster than 3 / 6)
  static constexpr bool kPlain = kMode == 0 || kMode == 8;
  static constexpr int kGroups = kPlain ? kEpiGroupsPlain : kEpiGroups;
  // layer stack: one more warp watches the row flags (StackWatcher)
  static constexpr int kWatchWarp = kEpiWarp0 + 4 * kGroups;
  static constexpr int kThreads = 32 * (kEpiWarp0 + 4 * kGroups + (kStack ? 1 : 0));
  // split hidden layer: two passes of 32 output channels (TMEM room for three rings)
  static constexpr bool kHalves = kMode == 3 || kPairH;
  // TMEM cols per row; the 64-channel heads (modes 1 / 4) use 8 hi + 8 lo
  // weight columns per dy (K <= kMaxBands = 8): N = 48 per MMA instead of 96
  static constexpr int NB = kUnshuf ? 64 : ((kMode == 1 || kMode == 4) ? 16 : ((kHead || kHalves || kQuarters) ? 32 : 64));
  static constexpr int kWdxBlk = 3 * NB * 128;        // B bytes per dx and K block (3 dy x NB rows x 128 B)
  static constexpr int kWdx = kKBlk * kWdxBlk;        // B bytes per dx
  static constexpr int kWhalf = 3 * kWdx;             // one channel half (all dx)
  static constexpr int kW1 = kWhalf * (kHalves ? 2 : 1);  // one weight pack
  // wide pair-input layer (mode 5): the activation pair is [hi fp16 | lo e4m3
  // x 2^kLo8ActExp] (384 B/px) and the lo pass runs on kind::f8f6f4 against an
  // e4m3 copy of the weights x 2^kLo8WExp (36 KB per quarter after the fp16
  // pack), accumulating into its own ring (kCorrCol); the epilogue adds it back
  // scaled by 2^-(kLo8ActExp + kLo8WExp).  A K=32 e4m3 MMA costs an N=96 K=16 f16
  // one (tools/ubench_tcgen05.cu), so the lo pass takes half the MMAs.
  static constexpr bool kLo8 = kMode == 5;
  static constexpr int kWdxLo = 3 * NB * 128;         // e4m3 B bytes per dx (3 dy x NB rows x 128 ci)
  static constexpr int kW = kPairH ? 2 * kWhalf : (kHalves ? 2 * kW1 : (kLo8 ? kW1 + 3 * kWdxLo : kW1));  // fp32: hi | lo
  static constexpr int kWChunk = kLo8 ? kWdxLo : kWdx;  // bulk-load granularity of the pack
  static constexpr int kPasses = kHalves ? 3 : (kSplit ? 2 : 1);
  // K steps of pass p (the e4m3 lo pass: K = 32 per MMA over the 128-byte lo row)
  static constexpr int ksteps(int p) { return (kLo8 && p == 1) ? 4 : kKSteps; }
  static constexpr bool f8(int p) { return kLo8 && p == 1; }
  static constexpr int kNStages =
      kSplit ? ((kMode == 4) ? 5 : (kPairH ? 4 : 2))
             : (kPlain ? kStagesPlain : (kWideHalves ? 2 : (kWide ? 4 : kStages)));  // input-row ring depth
  // one stage: [hi K blocks][lo K blocks], one 17 KB SW128 row buffer each
  static constexpr int kStageBytes = (kLo8 ? 3 : (kSplit ? 2 : 1) * kKBlk) * kInRowStride;
  static constexpr int kStageOut = (kHead || kSplit || kWide) ? 0 : 32 * 128;  // per-warp TMA-store staging
  static constexpr size_t kSmem = 1024 + kW + kNStages * kStageBytes + 4 * kGroups * kStageOut + 1024;
  // A / B descriptor offsets (bytes) of pass p, K step k (within-block k%4 added by the caller)
  static constexpr uint32_t a_off(int p, int k) {
    return ((kSplit && p == 1) ? kKBlk * kInRowStride : 0) + (k / 4) * kInRowStride;
  }
  static constexpr uint32_t b_off(int p) {
    return (kHalves && p == 2) ? (kPairH ? kWhalf : kW1) : ((kLo8 && p == 1) ? kW1 : 0);
  }
  static constexpr uint32_t b_koff(int k) { return (k / 4) * kWdxBlk + (k % 4) * 32; }
  // B byte offset of (pass p, dx tap, K step k) inside the pack (dy block 0)
  static constexpr uint32_t b_at(int p, int dx, int k) {
    return f8(p) ? kW1 + dx * kWdxLo + k * 32 : b_off(p) + dx * kWdx + b_koff(k);
  }
  // TMEM accumulator rings.  tcgen05 f16 MMAs add their products exactly and
  // truncate the fp32 accumulator toward zero once per MMA
  // (tools/probe_mma_rounding.cu), so every MMA into an accumulator costs it
  // ~0.5 ulp.  The split hidden layer therefore keeps the hi*hi products (36
  // MMAs per output) in a main ring and the two small correction products (72
  // MMAs) in a separate correction ring (4 slots each); the epilogue adds the
  // expected truncation loss of the main ring back (kMainDebias) and sums.
  // (the split head likewise: hi*[W_hi|W_lo] in the main ring, lo*[W_hi|W_lo]
  // in the correction ring, 8 slots x 32 columns each)
  // The split hidden layer goes one step further: its 32-channel passes leave
  // room for the hi*hi products of input channels 0-31 and 32-63 in two
  // separate rings (18 MMAs each: half the accumulated magnitude, half the
  // truncations), plus the correction ring.
  static constexpr bool kTwoRings = kMode == 3 || kMode == 4 || kPairH;  // the fp32-accurate modes
  static constexpr int kRing = kTwoRings ? (kHead ? 8 : 4) : kSlots;
  static constexpr int kTmemCols = (kTwoRings || kLo8) ? 512 : kSlots * NB;  // 512 / 256
  static constexpr uint32_t kRingMask = kRing - 1;
  static constexpr int kRingLog = kRing == 4 ? 2 : 3;
  static constexpr uint32_t kOddCol = kRing * NB;                      // split hidden: 2nd main ring
  static constexpr uint32_t kCorrCol = kHalves ? 2 * kRing * NB : kRing * NB;
  // TMEM ring of pass p, K step k; whether (p, k) (at dx 0) is the first MMA into that ring
  static constexpr uint32_t ring_col(int p, int k) {
    return !(kTwoRings || kLo8) ? 0 : (kHalves ? (p == 0 ? (k < 2 ? 0 : kOddCol) : kCorrCol) : (p > 0 ? kCorrCol : 0));
  }
  static constexpr bool enters(int p, int k) {
    return kHalves ? ((p == 0 && (k == 0 || k == 2)) || (p == 1 && k == 0))
                   : (k == 0 && (p == 0 || ((kTwoRings || kLo8) && p == 1)));
  }
  static constexpr int kParts = kQuarters ? 4 : ((kWideHalves || kPairH) ? 2 : 1);  // SegIter grid partition
  static constexpr int kVisits = (kHalves && !kPairH) ? 2 : 1;    // SegIter visits per segment
  static constexpr int kPxBytes = kSplit ? 4 * kCin : 2 * kCin;  // activation bytes per pixel
};
static_assert(ConvCfg<5>::kSmem <= 232448 && ConvCfg<9>::kSmem <= 232448 && ConvCfg<10>::kSmem <= 232448 &&
                  ConvCfg<11>::kSmem <= 232448,
              "wide single-input smem");
constexpr float kSplitWScale = 256.0f;  // split hidden weights are packed x 2^8
constexpr int kLo8ActExp = 11, kLo8WExp = 10;  // wide pair layers: lo activations x 2^11, e4m3 weights x 2^10
// 1 + E[truncation loss] of the main accumulator: 36 MMAs, each losing 0.5 ulp of
// a partial sum that grows ~linearly to the result, E[ulp(x)/|x|] = 0.7213 * 2^-23
// over a binade (tools/emulate_split_accum.py: 1.2e-5 -> 5.1e-6 worst band)
constexpr float kMainDebias = 1.0f + 0.5f * 0.7213f * 18.0f * 1.1920929e-7f;
constexpr float kMainDebias18 = 1.0f + 0.5f * 0.7213f * 9.0f * 1.1920929e-7f;  // a ring of 18 MMAs

// an f16 or (the wide pair layers' lo pass) e4m3 MMA; `f8` is a compile-time
// constant at every call site once the pass loop is unrolled
__device__ __forceinline__ void mma_any(bool f8, uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  if (f8) mma_f8_ss(d, a, b, id, acc); else mma_f16_ss(d, a, b, id, acc);
}
__device__ __forceinline__ void mma_any_fill(bool f8, uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  if (f8) mma_f8_ss_fill(d, a, b, id, acc); else mma_f16_ss_fill(d, a, b, id, acc);
}
__device__ __forceinline__ void mma_any_use(bool f8, uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  if (f8) mma_f8_ss_use(d, a, b, id, acc); else mma_f16_ss_use(d, a, b, id, acc);
}
__device__ __forceinline__ void mma_any_lastuse(bool f8, uint32_t d, uint64_t a, uint64_t b, uint32_t id,
                                                uint32_t acc) {
  if (f8) mma_f8_ss_lastuse(d, a, b, id, acc); else mma_f16_ss_lastuse(d, a, b, id, acc);
}

template <int kMode>
__global__ void __launch_bounds__(ConvCfg<kMode>::kThreads, 1)
conv3x3_tc_kernel(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_out,
                  const ConvArgs a, const __grid_constant__ StackMaps smaps) {
  using Cfg = ConvCfg<kMode>;
  using Iter = std::conditional_t<Cfg::kStack, ItemIter, SegIter>;
  constexpr bool kHead = Cfg::kHead;
  constexpr int NB = Cfg::NB;
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t full[kStages], empty[kStages], slot_full[kSlots], slot_empty[kSlots], wbar, wfree;
  __shared__ uint32_t tmem_base_smem;
  __shared__ unsigned long long sFlagsReady;  // layer stack: StackWatcher progress (item ordinal << 32 | row + 1)
  __shared__ __align__(16) float sShift[kMaxC];
  // layer stack: each epilogue group's copy of its current layer's BN shift
  // (a per-row __ldg of the shift missed L1 every row: the store-completion
  // wait cp.async.bulk.wait_group invalidates L1)
  __shared__ __align__(16) float sShiftG[Cfg::kStack ? Cfg::kGroups : 1][kC];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;
  uint8_t* sIn = sW + Cfg::kW;
  uint8_t* sOut = sIn + Cfg::kNStages * Cfg::kStageBytes;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    sFlagsReady = 0;
    // (CTA pairs: a stage is free once BOTH CTAs' MMAs read it - the rows are
    // multicast into both - so each empty barrier takes two commits)
    for (int i = 0; i < Cfg::kNStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], Cfg::kCluster); }
    for (int i = 0; i < kSlots; ++i) { mbar_init(&slot_full[i], 1); mbar_init(&slot_empty[i], 4); }
    mbar_init(&wbar, 1);
    mbar_init(&wfree, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < kMaxC) sShift[threadIdx.x] = (threadIdx.x < a.nshift) ? a.shift[threadIdx.x] : 0.0f;
  if (warp == Cfg::kMmaWarp) tmem_alloc<Cfg::kTmemCols>(&tmem_base_smem);
  // weights do not depend on the previous layer: start their load before the
  // PDL wait so it overlaps the previous kernel's tail
  // CTA pairs (mode 12): this CTA's output-channel half
  const uint32_t pair_rank = Cfg::kCluster > 1 ? cluster_ctarank() : 0u;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&wbar, Cfg::kW);
    if constexpr (Cfg::kPairH) {  // its half of the split pack: [W_hi half | W_lo half]
      bulk_load(sW, a.wpack + pair_rank * Cfg::kWhalf, Cfg::kWhalf, &wbar);
      bulk_load(sW + Cfg::kWhalf, a.wpack + Cfg::kW1 + pair_rank * Cfg::kWhalf, Cfg::kWhalf, &wbar);
    } else {
      const uint8_t* wsrc = a.wpack + (Cfg::kPartsW ? (blockIdx.x % Cfg::kParts) * Cfg::kW : 0) +
                            (size_t)Iter(a).first_layer_or0(a) * Cfg::kW;
      for (int i = 0; i < Cfg::kW / Cfg::kWChunk; ++i)
        bulk_load(sW + i * Cfg::kWChunk, wsrc + i * Cfg::kWChunk, Cfg::kWChunk, &wbar);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if constexpr (Cfg::kCluster > 1) cluster_sync_all();  // the peers' barriers exist before any multicast lands
  const uint32_t tmem = tmem_base_smem;
  pdl_launch_dependents();  // the next layer may start its prologue on free SMs
  // previous layer's activations are complete and visible (a head gated on
  // the stack's row flags acquires them row by row instead)
  if (!(kMode == 1 && a.gate_target)) pdl_wait();
  if (a.span && threadIdx.x == 0) span_open(a.span);
  // kDbgTrace: per-CTA start / end stamps in the unused layer slot 31
  if constexpr (Cfg::kStack) trace_cta(a, 0);

  if (warp == 0) {
    // ------------------------------------------------ TMA producer ----
    if (elect_one()) {
      prefetch_tmap(&tm_in);
      int stage = 0;
      uint32_t phase = 0;
      Iter it(a, Cfg::kVisits, Cfg::kParts);
      int cur_layer = it.first_layer_or0(a);
      uint32_t nreload = 0;
      const CUtensorMap* tmi = &tm_in;
      StackGate gate;
      Segment g;
      unsigned long long item_ord = ~0ull, seen = 0;  // stack: this item's ordinal; watcher progress seen
      while (it.next(a, g)) {
        ++item_ord;
        if constexpr (Cfg::kStack) {
          if (g.layer != cur_layer) {  // MMAs of the previous item done -> load this layer's weights
            mbar_wait(&wfree, nreload & 1);
            ++nreload;
            mbar_arrive_expect_tx(&wbar, Cfg::kW);
            const uint8_t* wsrc = a.wpack + (size_t)g.layer * Cfg::kW;
            for (int i = 0; i < Cfg::kW / Cfg::kWChunk; ++i)
              bulk_load(sW + i * Cfg::kWChunk, wsrc + i * Cfg::kWChunk, Cfg::kWChunk, &wbar);
            cur_layer = g.layer;
          }
          tmi = (g.layer & 1) ? &smaps.in1 : &tm_in;
          gate.reset();
        }
        if constexpr (kMode == 1) gate.reset();
        const int r0 = max(g.ya - 1, 0), r1 = min(g.yb, a.H - 1);
        for (int r = r0; r <= r1; ++r) {
          mbar_wait(&empty[stage], phase ^ 1);
          if constexpr (Cfg::kStack) {
            if (g.layer > 0 && !(a.dbg & 1)) {
              if (a.watcher) {  // the watcher warp acquired the flags; acquire its progress (CTA scope)
                const unsigned long long want = (item_ord << 32) | (unsigned long long)(r + 1);
                if (seen < want) {
                  while ((seen = ld_acquire_cta_shared(&sFlagsReady)) < want) __nanosleep(20);
                  fence_proxy_async_global();  // generic-proxy view -> this thread's TMA loads
                }
              } else {
                gate.wait(a, g, r);
              }
            }
          }
          if constexpr (kMode == 1)
            if (a.gate_target) gate.wait(a, g, r, a.gate_target);
          if constexpr (Cfg::kStack) trace_mark(a, 0, g, r);
          // [hi blocks][lo blocks]; the wide pair layer's lo half is one 128-byte e4m3 block
          constexpr int nbuf = Cfg::kLo8 ? 3 : (Cfg::kSplit ? 2 : 1) * Cfg::kKBlk;
          if (a.dbg & 32) {  // ablation (TVS_CONV_DBG): no input loads
            mbar_arrive(&full[stage]);
            if (++stage == Cfg::kNStages) { stage = 0; phase ^= 1; }
            continue;
          }
          mbar_arrive_expect_tx(&full[stage], nbuf * kInRowBytes);
          if constexpr (Cfg::kCluster > 1) {  // this CTA's box (if any) to every CTA of the cluster
            if ((int)pair_rank < nbuf)
              tma_load_4d_mc(sIn + stage * Cfg::kStageBytes + pair_rank * kInRowStride, tmi, &full[stage],
                             64 * (int)pair_rank, g.x0 - 1, r, g.b, (uint16_t)((1u << Cfg::kCluster) - 1u));
            if (++stage == Cfg::kNStages) { stage = 0; phase ^= 1; }
            continue;
          }
#pragma unroll
          for (int i = 0; i < nbuf; ++i) {  // buffer i = channels 64i..64i+63 of the pixel row
            tma_load_4d(sIn + stage * Cfg::kStageBytes + i * kInRowStride, tmi, &full[stage], 64 * i, g.x0 - 1, r,
                        g.b);
          }
          if (++stage == Cfg::kNStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == Cfg::kMmaWarp) {
    // ------------------------------------------------ MMA issuer ----
    // The whole warp walks the schedule (warp-uniform values stay in uniform
    // registers); one elected lane issues.  Per input row the MMA budget is
    // ~12 x 96 cycles, so the issue path is kept to a few instructions per MMA:
    // descriptors are a per-row base plus compile-time offsets.
    const uint32_t idesc1 = make_idesc(128, NB, kFmtF16, kFmtF16);
    const uint32_t idesc2 = make_idesc(128, 2 * NB, kFmtF16, kFmtF16);
    const uint32_t idesc3 = make_idesc(128, 3 * NB, kFmtF16, kFmtF16);
    const uint64_t adesc0 = make_smem_desc(smem_u32(sIn), 0, 1024, kLayoutSW128);
    const uint64_t bdesc0 = make_smem_desc(smem_u32(sW), 0, 1024, kLayoutSW128);
    const bool leader = elect_one();
    const bool domma = !(a.dbg & 64);  // ablation (TVS_CONV_DBG): no MMAs
    unsigned long long cyc[7] = {0, 0, 0, 0, 0, 0, 0};
    const long long tstart = clock64();
    unsigned long long gstart = 0;
    if (Cfg::kStack && (a.dbg & 32768)) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gstart));
    mbar_wait(&wbar, 0);
    int stage = 0;
    uint32_t phase = 0;
    uint32_t seq = 0;  // output-row sequence number: slot = seq % kRing, use = seq / kRing
    bool prewaited = false;  // this row's barriers were already awaited by the previous row
    Iter it(a, Cfg::kVisits, Cfg::kParts);
    int cur_layer = it.first_layer_or0(a);
    uint32_t wphase = 0;
    Segment g;
    while (it.next(a, g)) {
      if constexpr (Cfg::kStack) {
        if (g.layer != cur_layer) {  // release the weights once the issued MMAs complete, await the next layer's
          if (leader) mma_commit(&wfree);
          __syncwarp();
          wphase ^= 1;
          long long tw = (a.dbg & 32768) ? clock64() : 0;
          mbar_wait(&wbar, wphase);
          if (a.dbg & 32768) cyc[3] += clock64() - tw;
          cur_layer = g.layer;
        }
      }
      const int r0 = max(g.ya - 1, 0), r1 = min(g.yb, a.H - 1);
      for (int r = r0; r <= r1; ++r) {
        // ---- fast path: interior input row (targets r-1, r, r+1 inside the
        // segment; r+1 is the only new slot; r-1 completes after this row).
        // The barriers of the NEXT row are awaited (by the issuing lane) in
        // the middle of this row's MMA stream, while the tensor-core queue
        // (~5 MMAs deep) still holds work, so row transitions do not drain it.
        if (r >= 1 && r - 1 >= g.ya && r + 1 <= g.yb - 1) {
          const uint32_t sq = seq + (uint32_t)(r - 1 - g.ya);  // sequence of output row r-1
          const uint32_t s = sq & Cfg::kRingMask;
          const bool next_fast = (r + 2 <= g.yb - 1);  // row r+1 is interior too
          const int nstage = (stage + 1 == Cfg::kNStages) ? 0 : stage + 1;
          const uint32_t nphase = (stage + 1 == Cfg::kNStages) ? (phase ^ 1) : phase;
          const uint32_t sq2 = sq + 3;  // output row r+2, entered by input row r+1
          bool pre_ok = false;  // (issuing lane) the next row's barriers have completed
          if (leader) {
            if (Cfg::kStack && (a.dbg & 32768)) {
              ++cyc[5];
              if (!prewaited) {
                long long t0 = clock64();
                mbar_wait(&slot_empty[(sq + 2) & Cfg::kRingMask], (((sq + 2) >> Cfg::kRingLog) & 1) ^ 1);
                long long t1 = clock64();
                mbar_wait(&full[stage], phase);
                cyc[1] += t1 - t0;
                cyc[2] += clock64() - t1;
              }
            } else if (!prewaited)
              mbar_wait2(&slot_empty[(sq + 2) & Cfg::kRingMask], (((sq + 2) >> Cfg::kRingLog) & 1) ^ 1, &full[stage],
                         phase);
            if constexpr (Cfg::kStack) trace_mark(a, 1, g, r);
            tc_fence_after();
            const uint64_t ad_row = adesc0 + (uint64_t)((stage * Cfg::kStageBytes) >> 4);
            const uint32_t t0s = s * NB;  // slot column offset inside a ring
            const uint32_t hoff = Cfg::kPairH ? 0u : (uint32_t)g.h * Cfg::kWhalf;  // B offset of the channel half
            constexpr uint32_t b1 = NB * 128 / 16, b2 = 2 * NB * 128 / 16;  // W(dy=0), W(dy=-1) blocks
            // Non-blocking probes (mid-row and near the row's end): a blocking
            // wait here would hold back the rest of this row's MMAs whenever
            // the next input row is late, draining the tensor-core queue.
            auto prewait = [&](int p, int dx, int k) {
              if (((p == Cfg::kPasses / 2 && dx == 1 && k == 1) ||
                   (p == Cfg::kPasses - 1 && dx == 2 && k == Cfg::ksteps(p) - 2)) &&
                  next_fast && !pre_ok && !(a.dbg & 2048))
                pre_ok = mbar_test(&slot_empty[sq2 & Cfg::kRingMask], ((sq2 >> Cfg::kRingLog) & 1) ^ 1) &&
                         mbar_test(&full[nstage], nphase);
            };
            // Split pieces share A through the collector: the N=NB piece is
            // issued first (fill), the N=2NB piece second (lastuse) -> full rate.
            // ablation (TVS_CONV_DBG): 512 = wrap rows issue the unsplit pattern at
            // slot 0, 1024 = no first-step split (results invalid)
            const bool nowrap = (a.dbg & 512) && s + 3 > (uint32_t)Cfg::kRing;
            const bool nosplit = (a.dbg & 1024);
            if (s + 3 <= (uint32_t)Cfg::kRing || nowrap) {
#pragma unroll
              for (int p = 0; p < Cfg::kPasses; ++p)
#pragma unroll
              for (int dx = 0; dx < 3; ++dx)
#pragma unroll
                for (int k = 0; k < Cfg::kKSteps; ++k) {
                  if (k >= Cfg::ksteps(p)) continue;  // (the e4m3 lo pass has 4)
                  const bool f8p = Cfg::f8(p);
                  const uint64_t ad = ad_row + (uint64_t)((Cfg::a_off(p, k) + dx * 128 + (k % 4) * 32) >> 4);
                  const uint64_t bd = bdesc0 + (uint64_t)((Cfg::b_at(p, dx, k) + hoff) >> 4);
                  const bool first_k = Cfg::enters(p, k) && dx == 0 && !nosplit;
                  const uint32_t rb = tmem + Cfg::ring_col(p, k), t0 = rb + (nowrap ? 0u : t0s);
                  if (first_k) {  // enter row r+1 (acc=0), keep r-1, r
                    if (domma) mma_any_fill(f8p, t0 + 2 * NB, ad, bd + b2, idesc1, 0u);
                    if (domma) mma_any_lastuse(f8p, t0, ad, bd, idesc2, 1u);
                  } else {
                    if (domma) mma_any(f8p, t0, ad, bd, idesc3, 1u);
                  }
                  prewait(p, dx, k);
                }
            } else if (s + 2 == (uint32_t)Cfg::kRing) {  // slots R-2, R-1 | wrap | 0
#pragma unroll
              for (int p = 0; p < Cfg::kPasses; ++p)
#pragma unroll
              for (int dx = 0; dx < 3; ++dx)
#pragma unroll
                for (int k = 0; k < Cfg::kKSteps; ++k) {
                  if (k >= Cfg::ksteps(p)) continue;  // (the e4m3 lo pass has 4)
                  const bool f8p = Cfg::f8(p);
                  const uint64_t ad = ad_row + (uint64_t)((Cfg::a_off(p, k) + dx * 128 + (k % 4) * 32) >> 4);
                  const uint64_t bd = bdesc0 + (uint64_t)((Cfg::b_at(p, dx, k) + hoff) >> 4);
                  const bool first_k = Cfg::enters(p, k) && dx == 0;
                  const uint32_t rb = tmem + Cfg::ring_col(p, k), t0 = rb + t0s;
                  if (domma) mma_any_fill(f8p, rb, ad, bd + b2, idesc1, first_k ? 0u : 1u);
                  if (domma) mma_any_lastuse(f8p, t0, ad, bd, idesc2, 1u);
                  prewait(p, dx, k);
                }
            } else {  // slot R-1 | wrap | 0, 1
#pragma unroll
              for (int p = 0; p < Cfg::kPasses; ++p)
#pragma unroll
              for (int dx = 0; dx < 3; ++dx)
#pragma unroll
                for (int k = 0; k < Cfg::kKSteps; ++k) {
                  if (k >= Cfg::ksteps(p)) continue;  // (the e4m3 lo pass has 4)
                  const bool f8p = Cfg::f8(p);
                  const uint64_t ad = ad_row + (uint64_t)((Cfg::a_off(p, k) + dx * 128 + (k % 4) * 32) >> 4);
                  const uint64_t bd = bdesc0 + (uint64_t)((Cfg::b_at(p, dx, k) + hoff) >> 4);
                  const bool first_k = Cfg::enters(p, k) && dx == 0;
                  const uint32_t rb = tmem + Cfg::ring_col(p, k), t0 = rb + t0s;
                  if (domma) mma_any_fill(f8p, t0, ad, bd, idesc1, 1u);
                  if (first_k) {
                    if (domma) mma_any_use(f8p, rb, ad, bd + b1, idesc1, 1u);
                    if (domma) mma_any_lastuse(f8p, rb + NB, ad, bd + b2, idesc1, 0u);
                  } else {
                    if (domma) mma_any_lastuse(f8p, rb, ad, bd + b1, idesc2, 1u);
                  }
                  prewait(p, dx, k);
                }
            }
            if constexpr (Cfg::kCluster > 1) mma_commit_mc(&empty[stage], (uint16_t)((1u << Cfg::kCluster) - 1u)); else mma_commit(&empty[stage]);
            mma_commit(&slot_full[s]);
          }
          __syncwarp();
          prewaited = next_fast && pre_ok;
          stage = nstage;
          phase = nphase;
          continue;
        }
        prewaited = false;
        // ---- general path (segment edges, image top/bottom)
        const int q_lo = max(r - 1, g.ya), q_hi = min(r + 1, g.yb - 1);
        // output rows whose first contributing input row is r: first(q) = max(q-1, 0)
        const int q_new = (r == 0) ? q_lo : r + 1;
        long long tg0 = (Cfg::kStack && (a.dbg & 32768)) ? clock64() : 0;
        for (int q = max(q_new, q_lo); q <= q_hi; ++q) {
          const uint32_t sq = seq + (uint32_t)(q - g.ya);
          mbar_wait(&slot_empty[sq & Cfg::kRingMask], ((sq >> Cfg::kRingLog) & 1) ^ 1);
        }
        long long tg1 = (Cfg::kStack && (a.dbg & 32768)) ? clock64() : 0;
        // Target rows [q_lo, q_hi] -> consecutive slots, split at the ring wrap
        // (regular ops R0, R1); the first K step also splits off the
        // newly-entered suffix [q_new, q_hi] with accumulate = 0 (ops F0..F2).
        // An op = (TMEM column, B row offset in 16-byte units, idesc, acc).
        const uint32_t s_lo = (seq + (uint32_t)(q_lo - g.ya)) & Cfg::kRingMask;
        const int cnt = q_hi - q_lo + 1;
        const int c0 = min(cnt, Cfg::kRing - (int)s_lo), c1 = cnt - c0;
        auto idesc_of = [&](int c) { return c == 3 ? idesc3 : (c == 2 ? idesc2 : idesc1); };
        auto brow16 = [&](int q) { return (uint32_t)(q - (r - 1)) * (uint32_t)(NB * 128 / 16); };
        // column offsets inside a ring (the ring base is added per pass)
        const uint32_t R0t = s_lo * NB, R0b = brow16(q_lo), R0i = idesc_of(c0);
        const uint32_t R1t = 0, R1b = brow16(q_lo + c0), R1i = idesc_of(c1);
        // first-K-step ops: old / new part of segment 0 and of segment 1
        const int s0e = q_lo + c0 - 1, s1b = q_lo + c0;
        const int A_e = min(s0e, q_new - 1), B_b = max(q_lo, q_new);
        const int C_e = min(q_hi, q_new - 1), D_b = max(s1b, q_new);
        const bool vA = q_lo <= A_e, vB = B_b <= s0e, vC = c1 > 0 && s1b <= C_e, vD = c1 > 0 && D_b <= q_hi;
        const uint32_t At = R0t, Ab = R0b, Ai = idesc_of(A_e - q_lo + 1);
        const uint32_t Bt = R0t + (uint32_t)(B_b - q_lo) * NB, Bb = brow16(B_b), Bi = idesc_of(s0e - B_b + 1);
        const uint32_t Ct = R1t, Cb = R1b, Ci = idesc_of(C_e - s1b + 1);
        const uint32_t Dt = R1t + (uint32_t)(D_b - s1b) * NB, Db = brow16(D_b), Di = idesc_of(q_hi - D_b + 1);
        mbar_wait(&full[stage], phase);
        if constexpr (Cfg::kStack) if (leader) trace_mark(a, 1, g, r);
        if (Cfg::kStack && (a.dbg & 32768)) { cyc[1] += tg1 - tg0; cyc[2] += clock64() - tg1; ++cyc[4]; }
        tc_fence_after();
        if (leader) {
          const uint64_t ad_row = adesc0 + (uint64_t)((stage * Cfg::kStageBytes) >> 4);
#pragma unroll
          for (int p = 0; p < Cfg::kPasses; ++p)
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) {
#pragma unroll
            for (int k = 0; k < Cfg::kKSteps; ++k) {
                  if (k >= Cfg::ksteps(p)) continue;  // (the e4m3 lo pass has 4)
                  const bool f8p = Cfg::f8(p);
              const uint64_t ad = ad_row + (uint64_t)((Cfg::a_off(p, k) + dx * 128 + (k % 4) * 32) >> 4);
              const uint64_t bd = bdesc0 + (uint64_t)((Cfg::b_at(p, dx, k) +
                                                       (Cfg::kPairH ? 0u : (uint32_t)g.h * Cfg::kWhalf)) >> 4);
              const uint32_t rb = tmem + Cfg::ring_col(p, k);
              if (Cfg::enters(p, k) && dx == 0) {
                if (vA) if (domma) mma_any(f8p, rb + At, ad, bd + Ab, Ai, 1u);
                if (vB) if (domma) mma_any(f8p, rb + Bt, ad, bd + Bb, Bi, 0u);
                if (vC) if (domma) mma_any(f8p, rb + Ct, ad, bd + Cb, Ci, 1u);
                if (vD) if (domma) mma_any(f8p, rb + Dt, ad, bd + Db, Di, 0u);
              } else {
                if (domma) mma_any(f8p, rb + R0t, ad, bd + R0b, R0i, 1u);
                if (c1 > 0) if (domma) mma_any(f8p, rb + R1t, ad, bd + R1b, R1i, 1u);
              }
            }
          }
          if constexpr (Cfg::kCluster > 1) mma_commit_mc(&empty[stage], (uint16_t)((1u << Cfg::kCluster) - 1u)); else mma_commit(&empty[stage]);
          for (int q = q_lo; q <= q_hi; ++q)
            if (min(q + 1, a.H - 1) == r) mma_commit(&slot_full[(seq + (uint32_t)(q - g.ya)) & Cfg::kRingMask]);
        }
        __syncwarp();
        if (++stage == Cfg::kNStages) { stage = 0; phase ^= 1; }
      }
      seq += (uint32_t)(g.yb - g.ya);
    }
    if (Cfg::kStack && (a.dbg & 32768) && leader) {
      cyc[0] = clock64() - tstart;
      unsigned long long gend;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gend));
      cyc[6] = gend - gstart;  // ns: cyc[0] / cyc[6] = the SM clock in GHz
      for (int i = 0; i < 7; ++i) atomicAdd(&g_dbg_cycles[i], cyc[i]);
    }
  } else if (Cfg::kStack && warp == Cfg::kWatchWarp) {
    // ------------------------------------------------ flag watcher ----
    if (a.watcher && lane == 0) StackWatcher::run(a, &sFlagsReady);
  } else {
    // ------------------------------------------------ epilogue ----
    const int ew = warp - Cfg::kEpiWarp0;     // 0 .. 4*kEpiGroups-1
    const uint32_t grp = (uint32_t)(ew >> 2); // output rows with seq % kGroups == grp
    const int quarter = warp & 3;             // TMEM lane quarter this warp may access
    const int px = quarter * 32 + lane;       // pixel within the strip == TMEM lane
    const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
    const uint32_t stage_out = smem_u32(sOut + ew * Cfg::kStageOut);
    const uint32_t shift_u = smem_u32(sShift);
    if (!kHead && !Cfg::kSplit && !Cfg::kWide && lane == 0) prefetch_tmap(&tm_out);
    uint32_t seq = 0, gsel = 0;  // gsel = seq % kGroups
    double bn_s1 = 0.0, bn_s2 = 0.0;  // training forward (mode 13): this lane's channel, sum y and sum y^2
    int grp_key = -1;            // layer stack: (image, layer) whose scaled shift sShiftG[grp] holds
    const uint32_t shift_g = smem_u32(&sShiftG[Cfg::kStack ? grp : 0][0]);
    Iter it(a, Cfg::kVisits, Cfg::kParts);
    Segment g;
    while (it.next(a, g)) {
      // layer-stack: this item's BN shift and output buffer
      const float4* shg = reinterpret_cast<const float4*>(a.shift + (size_t)g.layer * kC);
      const CUtensorMap* tmo = (Cfg::kStack && (g.layer & 1)) ? &smaps.out0 : &tm_out;
      // 2^-e_b of this segment's image (exact; 1 for in-range inputs)
      const float sc = image_scale(a.escale, g.b);
      if constexpr (Cfg::kStack) {
        const int key = g.b * 4096 + g.layer;
        if (key != grp_key && !(a.dbg & 16384)) {
          // every warp of the group is past the previous item's last per-row
          // barrier, so nobody still reads the old shift
          const int t = quarter * 32 + lane;
          if (t < kC) sShiftG[grp][t] = a.shift[(size_t)g.layer * kC + t] * sc;
          named_bar_sync(1 + grp, 128);
          grp_key = key;
        }
      }
      for (int q = g.ya; q < g.yb; ++q, ++seq, gsel = (gsel + 1 == Cfg::kGroups) ? 0 : gsel + 1) {
        if (gsel != grp) continue;
        const uint32_t slot = seq & Cfg::kRingMask;
        const int xg = g.x0 + px;
        // heads: the input pixel of the closure plane is loaded before the
        // accumulator wait (its global-load latency stalled the epilogue on the
        // closure subtraction: 21% of the head's warp samples)
        float xpre = 0.0f;
        if constexpr (kHead && !Cfg::kUnshuf)
          if (a.closure && xg < a.W) xpre = __ldg(a.x + ((long long)g.b * a.H + q) * a.W + xg);
        mbar_wait(&slot_full[slot], (seq >> Cfg::kRingLog) & 1);
        if constexpr (Cfg::kStack) if (quarter == 0 && lane == 0) trace_mark(a, 3, g, q);
        tc_fence_after();
        if constexpr (Cfg::kPartsW) {
          // wide hidden: channels NB*part..+NB-1 of this CTA's part (quarter: 32,
          // half: 64), + shift, ReLU, re-split into an fp16 pair: 2*NB B hi +
          // 2*NB B lo per pixel straight to global (single output: hi only)
          const int qtr = blockIdx.x % Cfg::kParts;
          uint32_t v[NB / 16][16];
#pragma unroll
          for (int j = 0; j < NB / 16; ++j) tmem_ld16(tmem + lane_addr + slot * NB + j * 16, v[j]);
          if constexpr (Cfg::kLo8) {  // + the e4m3 lo pass's ring, unscaled (exact: a power of two)
            uint32_t w[NB / 16][16];
#pragma unroll
            for (int j = 0; j < NB / 16; ++j) tmem_ld16(tmem + lane_addr + Cfg::kCorrCol + slot * NB + j * 16, w[j]);
            tmem_ld_wait();
            constexpr float kUn = 1.0f / (float)(1 << (kLo8ActExp + kLo8WExp));
#pragma unroll
            for (int j = 0; j < NB / 16; ++j) {
              reg_fence16(v[j]);
              reg_fence16(w[j]);
#pragma unroll
              for (int i = 0; i < 16; ++i)
                v[j][i] = __float_as_uint(fmaf(__uint_as_float(w[j][i]), kUn, __uint_as_float(v[j][i])));
            }
          } else {
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < NB / 16; ++j) reg_fence16(v[j]);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&slot_empty[slot]);
          if (xg < a.W) {
            // output pixel stride: pair 3*C bytes (hi C fp16 | lo C e4m3), single 2*C
            const int opx = a.out_single ? 2 * Cfg::kCin : 3 * Cfg::kCin;
            uint8_t* dst = a.act_out + (((long long)g.b * a.H + q) * a.W + xg) * opx + qtr * NB * 2;
            uint8_t* dst_lo = a.act_out + (((long long)g.b * a.H + q) * a.W + xg) * opx + 2 * Cfg::kCin + qtr * NB;
#pragma unroll
            for (int chunk = 0; chunk < NB / 8; ++chunk) {
              const uint32_t sh_u = shift_u + (uint32_t)(qtr * NB + chunk * 8) * 4;
              const float4 s0 = ld_shared_f4(sh_u);
              const float4 s1 = ld_shared_f4(sh_u + 16);
              const float sh[8] = {s0.x * sc, s0.y * sc, s0.z * sc, s0.w * sc, s1.x * sc, s1.y * sc, s1.z * sc,
                                   s1.w * sc};
              uint32_t hi[4];
              uint16_t lo8[4];
#pragma unroll
              for (int t2 = 0; t2 < 4; ++t2) {
                const int ch = chunk * 8 + t2 * 2;
                const float f0 = fmaxf(__uint_as_float(v[ch >> 4][ch & 15]) + sh[t2 * 2], 0.0f);
                const float f1 = fmaxf(__uint_as_float(v[ch >> 4][(ch & 15) + 1]) + sh[t2 * 2 + 1], 0.0f);
                const __half2 hh = __floats2half2_rn(f0, f1);
                const float2 hf = __half22float2(hh);
                hi[t2] = *reinterpret_cast<const uint32_t*>(&hh);
                // lo = (f - hi) x 2^11 as e4m3 (the pair format of the next pair layer)
                lo8[t2] = __nv_cvt_float2_to_fp8x2(make_float2((f0 - hf.x) * (float)(1 << kLo8ActExp),
                                                               (f1 - hf.y) * (float)(1 << kLo8ActExp)),
                                                   __NV_SATFINITE, __NV_E4M3);
              }
              *reinterpret_cast<uint4*>(dst + chunk * 16) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
              if (!a.out_single)
                *reinterpret_cast<uint2*>(dst_lo + chunk * 8) =
                    make_uint2((uint32_t)lo8[0] | ((uint32_t)lo8[1] << 16), (uint32_t)lo8[2] | ((uint32_t)lo8[3] << 16));
            }
          }
        } else if constexpr (Cfg::kHalves) {
          const int hh = Cfg::kPairH ? (int)pair_rank : g.h;  // this output-channel half
          // channels 32h..32h+31: z = (E + O) debiased + corrections (x 2^-8) +
          // shift, ReLU, re-split into an fp16 pair; one pixel per lane, 64 B hi
          // + 64 B lo straight to global
          uint32_t e[2][16], o[2][16], c[2][16];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            tmem_ld16(tmem + lane_addr + slot * NB + j * 16, e[j]);
            tmem_ld16(tmem + lane_addr + Cfg::kOddCol + slot * NB + j * 16, o[j]);
            tmem_ld16(tmem + lane_addr + Cfg::kCorrCol + slot * NB + j * 16, c[j]);
          }
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 2; ++j) { reg_fence16(e[j]); reg_fence16(o[j]); reg_fence16(c[j]); }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&slot_empty[slot]);
          // rows at the image's top / bottom edge have 2 (or 1) dy taps inside the
          // image: 12 (6) MMAs per main ring instead of 18, so less truncation to undo
          const int ndy = (q > 0 ? 1 : 0) + 1 + (q + 1 < a.H ? 1 : 0);
          const float kDb = 1.0f + 0.5f * 0.7213f * 3.0f * 1.1920929e-7f * (float)ndy;
          if (Cfg::kAux && a.raw_f32) {  // training forward: pre-BatchNorm conv output, fp32
            const bool inside = xg < a.W;
            float* dst = reinterpret_cast<float*>(a.act_out) + (((long long)g.b * a.H + q) * a.W + xg) * 64 + hh * 32;
#pragma unroll
            for (int c8 = 0; c8 < 4; ++c8) {
              float f[8];
#pragma unroll
              for (int t = 0; t < 8; ++t) {
                const int ch = c8 * 8 + t;
                const float z = fmaf(__uint_as_float(e[ch >> 4][ch & 15]), kDb,
                                     fmaf(__uint_as_float(o[ch >> 4][ch & 15]), kDb,
                                          __uint_as_float(c[ch >> 4][ch & 15])));
                f[t] = z * (1.0f / kSplitWScale);
              }
              if (inside) {
                *reinterpret_cast<float4*>(dst + c8 * 8) = make_float4(f[0], f[1], f[2], f[3]);
                *reinterpret_cast<float4*>(dst + c8 * 8 + 4) = make_float4(f[4], f[5], f[6], f[7]);
              }
              if (Cfg::kPairH && a.bn_sums) {
                // batch statistics: sum and sum of squares of these 8 channels over
                // the warp's 32 pixels.  A transposing butterfly (4 + 2 + 1 exchanges
                // inside groups of 8 lanes, then two across the groups) leaves the
                // 32-pixel sums of channel 8*c8 + lane % 8 in every lane; the lanes
                // of group c8 add them to their fp64 accumulator (lane = channel).
                float s1[8], s2[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                  s1[t] = inside ? f[t] : 0.0f;
                  s2[t] = s1[t] * s1[t];
                }
#pragma unroll
                for (int off = 4; off >= 1; off >>= 1) {
                  const bool up = lane & off;
#pragma unroll
                  for (int i = 0; i < off; ++i) {
                    const float k1 = up ? s1[i + off] : s1[i], g1 = up ? s1[i] : s1[i + off];
                    const float k2 = up ? s2[i + off] : s2[i], g2 = up ? s2[i] : s2[i + off];
                    s1[i] = k1 + __shfl_xor_sync(0xffffffffu, g1, off);
                    s2[i] = k2 + __shfl_xor_sync(0xffffffffu, g2, off);
                  }
                }
                s1[0] += __shfl_xor_sync(0xffffffffu, s1[0], 8);
                s2[0] += __shfl_xor_sync(0xffffffffu, s2[0], 8);
                s1[0] += __shfl_xor_sync(0xffffffffu, s1[0], 16);
                s2[0] += __shfl_xor_sync(0xffffffffu, s2[0], 16);
                if ((lane >> 3) == c8) {
                  bn_s1 += (double)s1[0];
                  bn_s2 += (double)s2[0];
                }
              }
            }
            continue;
          }
          if (xg < a.W) {
            uint8_t* dst = a.act_out + (((long long)g.b * a.H + q) * a.W + xg) * 256 + hh * 64;
            // wide fp32 mode: the other input block's raw partial sums of this pixel
            const float* accp =
                (Cfg::kAux && a.acc_in) ? a.acc_in + (((long long)g.b * a.H + q) * a.W + xg) * 64 + hh * 32 : nullptr;
#pragma unroll
            for (int chunk = 0; chunk < 4; ++chunk) {
              const uint32_t sh_u = shift_u + (uint32_t)(hh * 32 + chunk * 8) * 4;
              const float4 s0 = ld_shared_f4(sh_u);
              const float4 s1 = ld_shared_f4(sh_u + 16);
              float sh[8] = {s0.x * sc, s0.y * sc, s0.z * sc, s0.w * sc, s1.x * sc, s1.y * sc, s1.z * sc, s1.w * sc};
              if (Cfg::kAux && accp) {
                const float4 a0 = *reinterpret_cast<const float4*>(accp + chunk * 8);
                const float4 a1 = *reinterpret_cast<const float4*>(accp + chunk * 8 + 4);
                sh[0] += a0.x; sh[1] += a0.y; sh[2] += a0.z; sh[3] += a0.w;
                sh[4] += a1.x; sh[5] += a1.y; sh[6] += a1.z; sh[7] += a1.w;
              }
              uint32_t hi[4], lo[4];
#pragma unroll
              for (int t2 = 0; t2 < 4; ++t2) {
                float f[2];
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                  const int ch = chunk * 8 + t2 * 2 + t;  // channel within the half
                  const float z = fmaf(__uint_as_float(e[ch >> 4][ch & 15]), kDb,
                                       fmaf(__uint_as_float(o[ch >> 4][ch & 15]), kDb,
                                            __uint_as_float(c[ch >> 4][ch & 15])));
                  f[t] = fmaxf(fmaf(z, 1.0f / kSplitWScale, sh[t2 * 2 + t]), 0.0f);
                }
                const __half2 hh = __floats2half2_rn(f[0], f[1]);
                const float2 hf = __half22float2(hh);
                const __half2 ll = __floats2half2_rn(f[0] - hf.x, f[1] - hf.y);
                hi[t2] = *reinterpret_cast<const uint32_t*>(&hh);
                lo[t2] = *reinterpret_cast<const uint32_t*>(&ll);
              }
              *reinterpret_cast<uint4*>(dst + chunk * 16) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
              *reinterpret_cast<uint4*>(dst + 128 + chunk * 16) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
            }
          }
        } else if constexpr (!kHead) {
          if (a.dbg & 16) {  // ablation (TVS_CONV_DBG): drain the slot without reading it
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&slot_empty[slot]);
            continue;
          }
          uint32_t v[4][16];
#pragma unroll
          for (int j = 0; j < 4; ++j) tmem_ld16(tmem + lane_addr + slot * NB + j * 16, v[j]);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 4; ++j) reg_fence16(v[j]);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&slot_empty[slot]);
          if (!Cfg::kStack && a.raw_f32) {  // training dgrad: raw fp32 accumulator, unscaled
            // The lane's 64 fp32 channels go out through the warp's 4 KB staging
            // tile in two halves of 32 channels, transposed so that every store
            // instruction writes whole 128-byte lines (4 pixels x 32 channels);
            // per-lane 256 B rows cost 32 partial sectors per instruction and made
            // this epilogue 2.6x slower per pixel than the inference layer's TMA store.
            const float m = a.out_exp ? pow2i(-__ldg(a.out_exp)) : 1.0f;
            float* row = reinterpret_cast<float*>(a.act_out) +
                         (((long long)g.b * a.H + q) * a.W + g.x0 + quarter * 32) * 64;  // pixel 0 of this warp
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
              for (int c = 0; c < 8; ++c) {  // 16-byte chunk c of the lane's 128-byte half row, XOR-swizzled
                const int j = hf * 2 + (c >> 2), i0 = (c & 3) * 4;
                st_shared_v4(stage_out + lane * 128 + ((c ^ (lane & 7)) << 4),
                             __float_as_uint(__uint_as_float(v[j][i0]) * m),
                             __float_as_uint(__uint_as_float(v[j][i0 + 1]) * m),
                             __float_as_uint(__uint_as_float(v[j][i0 + 2]) * m),
                             __float_as_uint(__uint_as_float(v[j][i0 + 3]) * m));
              }
              __syncwarp();
#pragma unroll
              for (int i = 0; i < 8; ++i) {  // 4 pixels x 128 B per instruction
                const int pp = i * 4 + (lane >> 3), c = lane & 7;
                const float4 t = ld_shared_f4(stage_out + pp * 128 + ((c ^ (pp & 7)) << 4));
                if (g.x0 + quarter * 32 + pp < a.W)
                  *reinterpret_cast<float4*>(row + (long long)pp * 64 + hf * 32 + c * 4) = t;
              }
              __syncwarp();
            }
            continue;
          }
          if (a.dbg & 128) {  // ablation: TMEM read only (keep the values alive)
            uint32_t acc = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
              for (int i = 0; i < 16; ++i) acc ^= v[j][i];
            if (acc == 0x7fc00123u) a.rowcnt[0] = 1;
            continue;
          }
          // this warp's staging buffer: its previous TMA store must have read it
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
          const uint32_t rowp = stage_out + lane * 128;
#pragma unroll
          for (int chunk = 0; chunk < 8; ++chunk) {  // 16-byte chunk = 8 channels
            const bool gl = Cfg::kStack && (a.dbg & 16384);  // A/B: the per-row global loads
            const float4 s0 = gl ? __ldg(shg + 2 * chunk) : ld_shared_f4((Cfg::kStack ? shift_g : shift_u) + chunk * 32);
            const float4 s1 = gl ? __ldg(shg + 2 * chunk + 1)
                                 : ld_shared_f4((Cfg::kStack ? shift_g : shift_u) + chunk * 32 + 16);
            float sh[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
            if (!Cfg::kStack && sc != 1.0f) {
#pragma unroll
              for (int i = 0; i < 8; ++i) sh[i] *= sc;
            }
            uint32_t packed[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int c = chunk * 8 + e * 2;
              // packed fp32x2 add (FADD2): channel pair (c, c+1) in one instruction
              // (measured neutral against scalar adds; fewer issue slots)
              const float2 fs = __fadd2_rn(make_float2(__uint_as_float(v[c >> 4][c & 15]),
                                                       __uint_as_float(v[c >> 4][(c & 15) + 1])),
                                           make_float2(sh[2 * e], sh[2 * e + 1]));
              const float f0 = fs.x, f1 = fs.y;
              if (a.dbg & 65536) {  // A/B: separate ReLU and conversion
                __half2 hv = __floats2half2_rn(fmaxf(f0, 0.0f), fmaxf(f1, 0.0f));
                packed[e] = *reinterpret_cast<uint32_t*>(&hv);
              } else {
                // ReLU fused into the fp16 rounding (fewer epilogue instructions
                // competing with the MMA warp for issue slots)
                asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(packed[e]) : "f"(f1), "f"(f0));
              }
            }
            st_shared_v4(rowp + ((chunk ^ (lane & 7)) << 4), packed[0], packed[1], packed[2], packed[3]);
          }
          fence_async_smem();
          __syncwarp();
          if (a.dbg & 256) continue;  // ablation: no TMA store
          if (lane == 0) {
            tma_store_4d(tmo, sOut + ew * Cfg::kStageOut, 0, g.x0 + quarter * 32, q, g.b);
            bulk_commit();
            if constexpr (Cfg::kStack) {
              if (quarter == 0) trace_mark(a, 4, g, q);
              // this warp's quarter row has landed (async proxy); order it
              // before the generic-proxy release below (the reader acquires,
              // then fences into the async proxy before its TMA load)
              if (!(a.dbg & kDbgNoStoreWait)) {
                bulk_wait<0>();
                fence_proxy_async_global();
              }
            }
          }
          if constexpr (Cfg::kStack) {
            // publish the row to the next layer's items: the group's 4 warps
            // meet on a named barrier, one thread releases the row counter (+4)
            __syncwarp();
            named_bar_sync(1 + grp, 128);
            const bool withhold = (a.dbg & kDbgWithholdFlag) && g.b == 0 && g.x0 == 0 && q == 1 && g.layer == 2;
            if (quarter == 0 && lane == 0 && !withhold) {
              red_release_gpu_add(a.rowcnt + ((long long)g.b * a.strips + g.x0 / kStripPx) * a.H + q, 4);
              trace_mark(a, 2, g, q);
            }
          }
        } else if constexpr (Cfg::kUnshuf) {
          uint32_t v[4][16];
#pragma unroll
          for (int j = 0; j < 4; ++j) tmem_ld16(tmem + lane_addr + slot * NB + j * 16, v[j]);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 4; ++j) reg_fence16(v[j]);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&slot_empty[slot]);
          double rr2 = 0.0, rx2 = 0.0;  // reconstruction check (recon_accumulate, pre-squared)
          if (xg < a.W) {
            // half-res pixel (q, xg) -> full-res 2x2 block at rows 2q+i, cols 2xg+j
            const int Wf = 2 * a.W;
            const long long planef = (long long)(2 * a.rows) * Wf;
            const long long r0f = 2LL * (q - a.row0);
            float sum[4] = {0.f, 0.f, 0.f, 0.f};
            const float inv = 1.0f / sc;  // undo the image's 2^-e activation scale (exact)
            bool bad = false;
#pragma unroll
            for (int k = 0; k < kMaxBands; ++k) {
              if (k < a.K) {
                float* ob = a.bands + ((long long)g.b * a.K + k) * planef;
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                  float f[2];
#pragma unroll
                  for (int jj = 0; jj < 2; ++jj) {
                    const int o = k * 4 + i * 2 + jj;  // head channel (pixel_shuffle order)
                    f[jj] = (__uint_as_float(v[o >> 4][o & 15]) + __uint_as_float(v[(32 + o) >> 4][(32 + o) & 15])) *
                                inv + sShift[o];
                    sum[i * 2 + jj] += f[jj];
                    bad |= !isfinite(f[jj]);
                  }
                  *reinterpret_cast<float2*>(ob + (r0f + i) * Wf + 2 * xg) = make_float2(f[0], f[1]);
                }
              }
            }
            if (bad && a.status) flag_set(a.status + kStatNonFiniteOut);
            if (a.closure) {
#pragma unroll
              for (int i = 0; i < 2; ++i) {
                const float2 xi =
                    *reinterpret_cast<const float2*>(a.x + ((long long)g.b * 2 * a.H + 2 * q + i) * Wf + 2 * xg);
                const float2 c = make_float2(xi.x - sum[i * 2], xi.y - sum[i * 2 + 1]);
                *reinterpret_cast<float2*>(a.closure + (long long)g.b * planef + (r0f + i) * Wf + 2 * xg) = c;
                const float r0 = xi.x - (sum[i * 2] + c.x), r1 = xi.y - (sum[i * 2 + 1] + c.y);
                rr2 += (double)r0 * r0 + (double)r1 * r1;
                rx2 += (double)xi.x * xi.x + (double)xi.y * xi.y;
              }
            }
          }
          if (a.recon) {  // four full-res pixels per lane: pre-squared sums
#pragma unroll
            for (int o = 16; o; o >>= 1) {
              rr2 += __shfl_xor_sync(0xffffffffu, rr2, o);
              rx2 += __shfl_xor_sync(0xffffffffu, rx2, o);
            }
            if (lane == 0) {
              atomicAdd(a.recon + 2 * g.b, rr2);
              atomicAdd(a.recon + 2 * g.b + 1, rx2);
            }
          }
        } else {
          // v[0][k] = [x * W_hi]_k, v[1][k] = [x * W_lo]_k (w: the correction ring)
          uint32_t v[2][16], w[2][16];
          if constexpr (NB == 16) {  // one load: cols 0-7 hi, 8-15 lo
            uint32_t t[16], c[16];
            tmem_ld16(tmem + lane_addr + slot * NB, t);
            if constexpr (Cfg::kTwoRings) tmem_ld16(tmem + lane_addr + Cfg::kCorrCol + slot * NB, c);
            tmem_ld_wait();
            reg_fence16(t);
            if constexpr (Cfg::kTwoRings) reg_fence16(c);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              v[0][k] = t[k];
              v[1][k] = t[8 + k];
              if constexpr (Cfg::kTwoRings) { w[0][k] = c[k]; w[1][k] = c[8 + k]; }
            }
          } else {
            tmem_ld16(tmem + lane_addr + slot * NB, v[0]);
            tmem_ld16(tmem + lane_addr + slot * NB + 16, v[1]);
            if constexpr (Cfg::kTwoRings) {
              tmem_ld16(tmem + lane_addr + Cfg::kCorrCol + slot * NB, w[0]);
              tmem_ld16(tmem + lane_addr + Cfg::kCorrCol + slot * NB + 16, w[1]);
            }
            tmem_ld_wait();
            reg_fence16(v[0]);
            reg_fence16(v[1]);
            if constexpr (Cfg::kTwoRings) { reg_fence16(w[0]); reg_fence16(w[1]); }
          }
          if constexpr (Cfg::kTwoRings) {
#pragma unroll
            for (int k = 0; k < kMaxBands; ++k)  // main hi*W_hi (debiased) + the three correction products
              v[0][k] = __float_as_uint(fmaf(__uint_as_float(v[0][k]), kMainDebias,
                                             (__uint_as_float(v[1][k]) + __uint_as_float(w[0][k])) +
                                                 __uint_as_float(w[1][k])));
#pragma unroll
            for (int k = 0; k < kMaxBands; ++k) v[1][k] = 0u;
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&slot_empty[slot]);
          float rr = 0.0f, rx = 0.0f;  // reconstruction-check residual and input of this lane's pixel
          if (xg < a.W) {
            const long long plane = (long long)a.rows * a.W;
            const long long pix = (long long)(q - a.row0) * a.W + xg;
            float* ob = a.bands + (long long)g.b * a.K * plane + pix;
            float sum = 0.0f;
            const float inv = 1.0f / sc;  // undo the image's 2^-e activation scale (exact)
            bool bad = false;
#pragma unroll
            for (int k = 0; k < kMaxBands; ++k) {
              if (k < a.K) {
                float o = (__uint_as_float(v[0][k]) + __uint_as_float(v[1][k])) * inv + sShift[k];
                if (a.acc_bands) o += ob[k * plane];  // wide fp32 mode: + the first input block's partial
                ob[k * plane] = o;
                sum += o;
                bad |= !isfinite(o);
              }
            }
            if (bad && a.status) flag_set(a.status + kStatNonFiniteOut);
            if (a.closure) {
              const float xv = xpre;
              const float c = xv - sum;
              a.closure[(long long)g.b * plane + pix] = c;
              rr = xv - (sum + c);
              rx = xv;
            }
          }
          if (a.recon) recon_accumulate(a.recon, g.b, rr, rx);  // warp-uniform; every lane arrives
        }
      }
    }
    if (!kHead && !Cfg::kSplit && !Cfg::kWide && lane == 0) bulk_wait<0>();
    if constexpr (Cfg::kAux && Cfg::kPairH) {
      if (a.raw_f32 && a.bn_sums) {  // lane = channel 32 * half + lane of this CTA's output-channel half
        atomicAdd(a.bn_sums + pair_rank * 32 + lane, bn_s1);
        atomicAdd(a.bn_sums + 64 + pair_rank * 32 + lane, bn_s2);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == Cfg::kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem);
  }
  // CTA pairs: no CTA leaves while its peer may still multicast into it or
  // commit to its barriers
  if constexpr (Cfg::kCluster > 1) cluster_sync_all();
  if (a.span && threadIdx.x == 0) span_close(a.span);
  if constexpr (Cfg::kStack) trace_cta(a, 1);
}

// --------------------------------------------------------------------------
// Weight packs.
//
// Hidden: BN-folded W*s rounded to fp16 with tap-sum compensation: round to
// nearest, then per (co, ci) flip the rounding direction of individual taps
// (cheapest first) while that brings the sum of rounding residuals over the 9
// taps closer to zero.  Each filter's response to locally-constant input (the
// DC term that dominates with non-negative ReLU activations) is then exact to
// fp32 precision; this halves the fp16 error of the 17-layer stack
// (tools/emulate_precision.py: 1.04e-2 -> 6.1e-3 worst band on config 1).
//
// Head: W = W_hi + W_lo, both fp16 round-to-nearest (exact split to ~2^-22).
// --------------------------------------------------------------------------
__device__ __forceinline__ float half_other_side(float w, __half rn) {
  const float r = __half2float(rn);
  if (r == w) return r;
  unsigned short bits = __half_as_ushort(rn);
  const bool toward_up = (r < w);
  const bool neg = (bits & 0x8000u) != 0;
  if (r == 0.0f) {
    bits = toward_up ? 0x0001u : 0x8001u;
  } else {
    const bool grow = (toward_up != neg);  // magnitude grows when moving away from zero
    bits = grow ? (unsigned short)(bits + 1) : (unsigned short)(bits - 1);
  }
  return __half2float(__ushort_as_half(bits));
}

// B row n (0..3*NB) of dx block kx: 128 B = 64 ci fp16, SW128 chunk swizzle
__device__ __forceinline__ void put_b(uint8_t* out, int wdx, int kx, int n, int ci, __half v) {
  const uint32_t off = (uint32_t)kx * wdx + (uint32_t)n * 128u + (uint32_t)(((ci >> 3) ^ (n & 7)) << 4) +
                       (uint32_t)((ci & 7) << 1);
  *reinterpret_cast<__half*>(out + off) = v;
}

// Tap-sum compensated fp16 rounding of one (co, ci) filter's 9 taps (see above).
__device__ __forceinline__ void dc_round9(const float* wv, float* rn) {
  float alt[9], cost[9];
  float s = 0.0f;
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    const __half h = __float2half_rn(wv[t]);
    rn[t] = __half2float(h);
    alt[t] = half_other_side(wv[t], h);
    cost[t] = fabsf(alt[t] - wv[t]) - fabsf(rn[t] - wv[t]);
    s += rn[t] - wv[t];
  }
  uint32_t used = 0;
  for (int it = 0; it < 9; ++it) {
    int best = 0;
    float bc = 3.4e38f;
#pragma unroll
    for (int t = 0; t < 9; ++t)
      if (!(used >> t & 1u) && cost[t] < bc) { bc = cost[t]; best = t; }
    used |= 1u << best;
    const float d = (alt[best] - wv[best]) - (rn[best] - wv[best]);
    if (fabsf(s + d) < fabsf(s)) { s += d; rn[best] = alt[best]; }
  }
}

__global__ void pack_hidden_f16_kernel(const float* __restrict__ w, const float* __restrict__ scale,
                                       uint8_t* __restrict__ out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // co*64 + ci
  if (idx >= kC * kC) return;
  const int co = idx / kC, ci = idx % kC;
  float wv[9], rn[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) wv[t] = w[idx * 9 + t] * scale[co];  // BatchNorm fold W' = W*s (fp32)
  dc_round9(wv, rn);
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    const int ky = t / 3, kx = t % 3;
    put_b(out, ConvCfg<0>::kWdx, kx, (2 - ky) * 64 + co, ci, __float2half_rn(rn[t]));
  }
}

// Training dgrad (mode 0 on gradients): the transposed, flipped filter
// W'[ci][co][2-ky][2-kx] = W[co][ci][ky][kx] as a mode-0 B pack, plain fp16
// rounding (the backward tolerates fp16 operands).
__device__ __forceinline__ void pack_f16_t_elem(const float* __restrict__ w, uint8_t* __restrict__ out, int idx) {
  const int co = idx / kC, ci = idx % kC;  // co*64 + ci of the forward filter
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    const int ky = t / 3, kx = t % 3;
    // output channel ci of the dgrad conv at tap (2-ky, 2-kx): B row (2 - (2-ky))*64 + ci = ky*64 + ci
    put_b(out, ConvCfg<0>::kWdx, 2 - kx, ky * 64 + ci, co, __float2half_rn(w[idx * 9 + t]));
  }
}
__global__ void pack_hidden_f16_t_kernel(const float* __restrict__ w, uint8_t* __restrict__ out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < kC * kC) pack_f16_t_elem(w, out, idx);
}

// Training head dgrad: the head filter W_h[k][ci][3][3] (k < K bands) as a
// 64 x 64 transposed pack with zero rows for k >= K, so the head's input
// gradient runs on the same tcgen05 dgrad kernel as the hidden layers (the
// gradient operand holds the bands in channels 0..K-1 of a 64-channel buffer)
__global__ void pack_head_f16_t_kernel(const float* __restrict__ w, int K, uint8_t* __restrict__ out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // co*64 + ci, co = band
  if (idx >= kC * kC) return;
  const int co = idx / kC, ci = idx % kC;
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    const int ky = t / 3, kx = t % 3;
    const float v = co < K ? w[idx * 9 + t] : 0.0f;
    put_b(out, ConvCfg<0>::kWdx, 2 - kx, ky * 64 + ci, co, __float2half_rn(v));
  }
}
cudaError_t launch_pack_head_f16_t(const float* w, int K, uint8_t* out, cudaStream_t st) {
  pack_head_f16_t_kernel<<<(kC * kC + 127) / 128, 128, 0, st>>>(w, K, out);
  return cudaGetLastError();
}

cudaError_t launch_pack_hidden_f16_t(const float* w, uint8_t* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, ConvCfg<0>::kW, st);
  if (e != cudaSuccess) return e;
  pack_hidden_f16_t_kernel<<<(kC * kC + 127) / 128, 128, 0, st>>>(w, out);
  return cudaGetLastError();
}

// Wide hidden (mode 5): 128x128 filters, DC-compensated fp16, packed per output
// quarter qtr = co/32: [qtr][dx][K block ci/64][3 dy x 32 rows x 128 B]
__global__ void pack_hidden_wide_kernel(const float* __restrict__ w, const float* __restrict__ scale,
                                        uint8_t* __restrict__ out, int parts, int lo8) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // co*128 + ci
  if (idx >= 128 * 128) return;
  const int co = idx / 128, ci = idx % 128;
  float wv[9], rn[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) wv[t] = w[idx * 9 + t] * scale[co];
  dc_round9(wv, rn);
  // quarters (modes 5 / 9): 4 packs of 32 output channels; halves (mode 11): 2 of 64
  const int nbp = 128 / parts;
  // per-part stride: quarters of a pair-input layer (mode 5) carry the e4m3
  // copy after the fp16 pack; single-input quarters (mode 9) / halves (mode 11) do not
  const size_t wpart = parts == 4 ? (lo8 ? ConvCfg<5>::kW : ConvCfg<9>::kW) : ConvCfg<11>::kW;
  const int wdxblk = 3 * nbp * 128, wdx = 2 * wdxblk;
  uint8_t* base = out + (co / nbp) * wpart + (ci >> 6) * wdxblk;
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    const int ky = t / 3, kx = t % 3;
    put_b(base, wdx, kx, (2 - ky) * nbp + (co % nbp), ci & 63, __float2half_rn(rn[t]));
  }
  if (lo8) {  // mode 5 lo pass: e4m3(W s 2^kLo8WExp), [dx][3 dy x 32 rows x 128 ci bytes], SW128
    uint8_t* lob = out + (co / nbp) * wpart + ConvCfg<5>::kW1;
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      const int ky = t / 3, kx = t % 3;
      const int n = (2 - ky) * nbp + (co % nbp);
      const uint32_t off = (uint32_t)kx * ConvCfg<5>::kWdxLo + (uint32_t)n * 128u +
                           (uint32_t)(((ci >> 4) ^ (n & 7)) << 4) + (uint32_t)(ci & 15);
      lob[off] = (uint8_t)__nv_cvt_float_to_fp8(wv[t] * (float)(1 << kLo8WExp), __NV_SATFINITE, __NV_E4M3);
    }
  }
}

// Wide head (mode 10): W = W_hi + W_lo over 128 input channels, [dx][K block][96 rows]
__global__ void pack_head_wide_kernel(const float* __restrict__ w, int K, uint8_t* __restrict__ out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // k*128 + ci
  if (idx >= K * 128) return;
  const int k = idx / 128, ci = idx % 128;
  using C6 = ConvCfg<10>;
  uint8_t* base = out + (ci >> 6) * C6::kWdxBlk;
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    const int ky = t / 3, kx = t % 3;
    const float wf = w[idx * 9 + t];
    const __half hi = __float2half_rn(wf);
    const __half lo = __float2half_rn(wf - __half2float(hi));
    const int nb = (2 - ky) * 32;
    put_b(base, C6::kWdx, kx, nb + k, ci & 63, hi);
    put_b(base, C6::kWdx, kx, nb + 16 + k, ci & 63, lo);
  }
}

// fp32-accurate hidden pack: W' = W*s (BatchNorm fold, fp32) x 2^8 split into
// hi = RN16(W'), lo = RN16(W' - hi); pack 0 = hi, pack 1 = lo.
__device__ __forceinline__ void pack_split_elem(const float* __restrict__ w, const float* __restrict__ scale,
                                                uint8_t* __restrict__ out, int idx, int cin, int co0, int ci0) {
  const int co = idx / kC, ci = idx % kC;
  const float* wsrc = w + ((size_t)(co0 + co) * cin + ci0 + ci) * 9;
  const float sc = scale ? scale[co0 + co] : 1.0f;
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    const int ky = t / 3, kx = t % 3;
    const float wv = (wsrc[t] * sc) * kSplitWScale;
    const __half hi = __float2half_rn(wv);
    const __half lo = __float2half_rn(wv - __half2float(hi));
    // channel half h = co / 32: rows (2-ky)*32 + co%32 of that half's dx block
    uint8_t* base = out + (co >> 5) * ConvCfg<3>::kWhalf;
    put_b(base, ConvCfg<3>::kWdx, kx, (2 - ky) * 32 + (co & 31), ci, hi);
    put_b(base + ConvCfg<3>::kW1, ConvCfg<3>::kWdx, kx, (2 - ky) * 32 + (co & 31), ci, lo);
  }
}
__global__ void pack_hidden_split_kernel(const float* __restrict__ w, const float* __restrict__ scale,
                                         uint8_t* __restrict__ out, int cin, int co0, int ci0) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // co*64 + ci
  if (idx < kC * kC) pack_split_elem(w, scale, out, idx, cin, co0, ci0);
}

// Training step: the split (forward) and transposed fp16 (dgrad) packs of up
// to kTrainPackLayers hidden layers in ONE launch (blockIdx.y = layer): 60
// launches per step became 1 (the step is host-bound at small batches).
__global__ void train_pack_hidden_kernel(TrainPackPtrs ptrs, uint8_t* __restrict__ wsplit,
                                         uint8_t* __restrict__ wt) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= kC * kC) return;
  const float* w = ptrs.w[blockIdx.y];
  pack_split_elem(w, nullptr, wsplit + (size_t)blockIdx.y * ConvCfg<3>::kW, idx, kC, 0, 0);
  pack_f16_t_elem(w, wt + (size_t)blockIdx.y * ConvCfg<0>::kW, idx);
}

cudaError_t launch_train_pack_hidden(const float* const* w_dev, int n, uint8_t* wsplit, uint8_t* wt, cudaStream_t st) {
  // both packs are written completely (every (co, ci, tap) has its own slot)
  for (int l0 = 0; l0 < n; l0 += kTrainPackLayers) {
    TrainPackPtrs ptrs{};
    const int cnt = std::min(kTrainPackLayers, n - l0);
    for (int i = 0; i < cnt; ++i) ptrs.w[i] = w_dev[l0 + i];
    train_pack_hidden_kernel<<<dim3((kC * kC + 127) / 128, cnt), 128, 0, st>>>(
        ptrs, wsplit + (size_t)l0 * ConvCfg<3>::kW, wt + (size_t)l0 * ConvCfg<0>::kW);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

__global__ void pack_head_f16_kernel(const float* __restrict__ w, int K, uint8_t* __restrict__ out, int cin,
                                     int ci0) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // k*64 + ci
  if (idx >= K * kC) return;
  const int k = idx / kC, ci = idx % kC;
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    const int ky = t / 3, kx = t % 3;
    const float wf = w[((size_t)k * cin + ci0 + ci) * 9 + t];
    const __half hi = __float2half_rn(wf);
    const __half lo = __float2half_rn(wf - __half2float(hi));
    const int nb = (2 - ky) * ConvCfg<1>::NB;  // per dy: 8 hi rows, then 8 lo rows
    put_b(out, ConvCfg<1>::kWdx, kx, nb + k, ci, hi);
    put_b(out, ConvCfg<1>::kWdx, kx, nb + ConvCfg<1>::NB / 2 + k, ci, lo);
  }
}

// Unshuffled head (mode 7): Conv2d(64, K4) weights, hi rows (2-ky)*64 + o,
// lo rows (2-ky)*64 + 32 + o
__global__ void pack_head_unshuf_kernel(const float* __restrict__ w, int K4, uint8_t* __restrict__ out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // o*64 + ci
  if (idx >= K4 * kC) return;
  const int o = idx / kC, ci = idx % kC;
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    const int ky = t / 3, kx = t % 3;
    const float wf = w[idx * 9 + t];
    const __half hi = __float2half_rn(wf);
    const __half lo = __float2half_rn(wf - __half2float(hi));
    put_b(out, ConvCfg<7>::kWdx, kx, (2 - ky) * 64 + o, ci, hi);
    put_b(out, ConvCfg<7>::kWdx, kx, (2 - ky) * 64 + 32 + o, ci, lo);
  }
}

__global__ void fill_kernel(float* dst, float v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = v;
}

// ------------------------------------------------------------ launchers ----

size_t conv_wpack_bytes(bool head) { return head ? ConvCfg<1>::kW : ConvCfg<0>::kW; }
size_t conv_wpack_split_bytes() { return ConvCfg<3>::kW; }
size_t conv_wpack_wide_bytes(bool head) { return head ? ConvCfg<10>::kW : 4 * ConvCfg<5>::kW; }
size_t conv_wpack_unshuf_head_bytes() { return ConvCfg<7>::kW; }

// Launched with programmatic stream serialization (PDL): the kernel's
// prologue overlaps the previous kernel; griddepcontrol.wait guards all
// activation reads and writes.
cudaError_t launch_conv_tc(int mode, const CUtensorMap& tm_in, const CUtensorMap& tm_out, const ConvArgs& a,
                           int grid, cudaStream_t st) {
  static const StackMaps zs{};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  switch (mode) {
    case 12:  // fp32-accurate hidden layer on CTA pairs: clusters of 2 (one output-channel half each)
      attr[1].id = cudaLaunchAttributeClusterDimension;
      attr[1].val.clusterDim.x = 2;
      attr[1].val.clusterDim.y = 1;
      attr[1].val.clusterDim.z = 1;
      cfg.numAttrs = 2;
      cfg.gridDim = dim3(std::max(2, grid & ~1));
      cfg.blockDim = dim3(ConvCfg<12>::kThreads);
      cfg.dynamicSmemBytes = ConvCfg<12>::kSmem;
      if (a.raw_f32 || a.acc_in)  // auxiliary epilogue paths: their own instantiation
        return cudaLaunchKernelEx(&cfg, conv3x3_tc_kernel<13>, tm_in, tm_out, a, zs);
      return cudaLaunchKernelEx(&cfg, conv3x3_tc_kernel<12>, tm_in, tm_out, a, zs);
    case 0:
      cfg.blockDim = dim3(ConvCfg<0>::kThreads);
      cfg.dynamicSmemBytes = ConvCfg<0>::kSmem;
      return cudaLaunchKernelEx(&cfg, conv3x3_tc_kernel<0>, tm_in, tm_out, a, zs);
    case 1:
      cfg.blockDim = dim3(ConvCfg<1>::kThreads);
      cfg.dynamicSmemBytes = ConvCfg<1>::kSmem;
      return cudaLaunchKernelEx(&cfg, conv3x3_tc_kernel<1>, tm_in, tm_out, a, zs);
    case 3:
      cfg.blockDim = dim3(ConvCfg<3>::kThreads);
      cfg.dynamicSmemBytes = ConvCfg<3>::kSmem;
      return cudaLaunchKernelEx(&cfg, conv3x3_tc_kernel<3>, tm_in, tm_out, a, zs);
    case 4:
      cfg.blockDim = dim3(ConvCfg<4>::kThreads);
      cfg.dynamicSmemBytes = ConvCfg<4>::kSmem;
      return cudaLaunchKernelEx(&cfg, conv3x3_tc_kernel<4>, tm_in, tm_out, a, zs);
    case 5:
      cfg.gridDim = dim3(std::max(4, grid & ~3));  // groups of 4 CTAs (output-channel quarters)
      if (ConvCfg<5>::kCluster > 1) {  // ... as clusters (input rows multicast)
        attr[1].id = cudaLaunchAttributeClusterDimension;
        attr[1].val.clusterDim.x = ConvCfg<5>::kCluster;
        attr[1].val.clusterDim.y = 1;
        attr[1].val.clusterDim.z = 1;
        cfg.numAttrs = 2;
      }
      cfg.blockDim = dim3(ConvCfg<5>::kThreads);
      cfg.dynamicSmemBytes = ConvCfg<5>::kSmem;
      return cudaLaunchKernelEx(&cfg, conv3x3_tc_kernel<5>, tm_in, tm_out, a, zs);
    case 7:
      cfg.blockDim = dim3(ConvCfg<7>::kThreads);
      cfg.dynamicSmemBytes = ConvCfg<7>::kSmem;
      return cudaLaunchKernelEx(&cfg, conv3x3_tc_kernel<7>, tm_in, tm_out, a, zs);
    case 9:
      cfg.gridDim = dim3(std::max(4, grid & ~3));  // groups of 4 CTAs (output-channel quarters)
      cfg.blockDim = dim3(ConvCfg<9>::kThreads);
      cfg.dynamicSmemBytes = ConvCfg<9>::kSmem;
      return cudaLaunchKernelEx(&cfg, conv3x3_tc_kernel<9>, tm_in, tm_out, a, zs);
    case 11:
      cfg.gridDim = dim3(std::max(2, grid & ~1));  // pairs of CTAs (output-channel halves)
      cfg.blockDim = dim3(ConvCfg<11>::kThreads);
      cfg.dynamicSmemBytes = ConvCfg<11>::kSmem;
      return cudaLaunchKernelEx(&cfg, conv3x3_tc_kernel<11>, tm_in, tm_out, a, zs);
    case 10:
      cfg.blockDim = dim3(ConvCfg<10>::kThreads);
      cfg.dynamicSmemBytes = ConvCfg<10>::kSmem;
      return cudaLaunchKernelEx(&cfg, conv3x3_tc_kernel<10>, tm_in, tm_out, a, zs);
  }
  return cudaErrorInvalidValue;
}

// Layer stack (mode 8): a cooperative launch, so the driver guarantees that
// all `grid` CTAs are co-resident (the deadlock-freedom argument of ItemIter
// needs it) or fails the launch (cudaErrorCooperativeLaunchTooLarge, e.g.
// under MPS SM limits), in which case the host falls back to the per-layer
// kernels.  rowcnt and the abort word must be zero on entry.
cudaError_t launch_conv_stack(const CUtensorMap& tm_in0, const CUtensorMap& tm_out1, const StackMaps& sm,
                              const ConvArgs& a, int grid, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(ConvCfg<8>::kThreads);
  cfg.dynamicSmemBytes = ConvCfg<8>::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (a.dbg & kDbgNoPdlStack) ? 1 : 2;
  return cudaLaunchKernelEx(&cfg, conv3x3_tc_kernel<8>, tm_in0, tm_out1, a, sm);
}

int debug_trace(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace)) != cudaSuccess) return -1;
  if (reset) {
    static unsigned long long z[kTraceKinds * kTraceLayers * kTraceRows];
    cudaMemcpyToSymbol(g_trace, z, sizeof(z));
  }
  return 0;
}

int debug_cycles(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_dbg_cycles, sizeof(unsigned long long) * 8) != cudaSuccess) return -1;
  if (reset) {
    const unsigned long long z[8] = {};
    cudaMemcpyToSymbol(g_dbg_cycles, z, sizeof(z));
  }
  return 0;
}

bool conv_stack_fits(int num_sms, int grid) {
  int dev = 0, coop = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  if (cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev) != cudaSuccess || !coop) return false;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, conv3x3_tc_kernel<8>, ConvCfg<8>::kThreads,
                                                    ConvCfg<8>::kSmem) != cudaSuccess)
    return false;
  return (long long)per_sm * num_sms >= grid;
}

cudaError_t launch_pack_hidden_f16(const float* w, const float* scale, uint8_t* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, ConvCfg<0>::kW, st);
  if (e != cudaSuccess) return e;
  pack_hidden_f16_kernel<<<(kC * kC + 127) / 128, 128, 0, st>>>(w, scale, out);
  return cudaGetLastError();
}

cudaError_t launch_pack_hidden_split(const float* w, const float* scale, uint8_t* out, cudaStream_t st, int cin,
                                     int co0, int ci0) {
  cudaError_t e = cudaMemsetAsync(out, 0, ConvCfg<3>::kW, st);
  if (e != cudaSuccess) return e;
  pack_hidden_split_kernel<<<(kC * kC + 127) / 128, 128, 0, st>>>(w, scale, out, cin, co0, ci0);
  return cudaGetLastError();
}

// one wide hidden layer's pack inside its conv_wpack_wide_bytes(false) slot:
// quarters of a pair-input layer (mode 5, lo8: fp16 + e4m3 copies), or
// single-input quarters (mode 9) / halves (mode 11)
cudaError_t launch_pack_hidden_wide(const float* w, const float* scale, uint8_t* out, cudaStream_t st, int parts,
                                    bool lo8) {
  static_assert(4 * ConvCfg<9>::kW == 2 * ConvCfg<11>::kW && 4 * ConvCfg<5>::kW >= 2 * ConvCfg<11>::kW,
                "every wide pack fits the layer stride");
  cudaError_t e = cudaMemsetAsync(out, 0, 4 * ConvCfg<5>::kW, st);
  if (e != cudaSuccess) return e;
  pack_hidden_wide_kernel<<<(128 * 128 + 127) / 128, 128, 0, st>>>(w, scale, out, parts, lo8 ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_pack_head_wide(const float* w, int K, uint8_t* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, ConvCfg<10>::kW, st);
  if (e != cudaSuccess) return e;
  pack_head_wide_kernel<<<(K * 128 + 127) / 128, 128, 0, st>>>(w, K, out);
  return cudaGetLastError();
}

cudaError_t launch_pack_head_unshuf(const float* w, int K4, uint8_t* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, ConvCfg<7>::kW, st);
  if (e != cudaSuccess) return e;
  pack_head_unshuf_kernel<<<(K4 * kC + 127) / 128, 128, 0, st>>>(w, K4, out);
  return cudaGetLastError();
}

cudaError_t launch_pack_head_f16(const float* w, int K, uint8_t* out, cudaStream_t st, int cin, int ci0) {
  cudaError_t e = cudaMemsetAsync(out, 0, ConvCfg<1>::kW, st);
  if (e != cudaSuccess) return e;
  pack_head_f16_kernel<<<(K * kC + 127) / 128, 128, 0, st>>>(w, K, out, cin, ci0);
  return cudaGetLastError();
}

cudaError_t launch_fill(float* dst, float v, int n, cudaStream_t st) {
  fill_kernel<<<(n + 255) / 256, 256, 0, st>>>(dst, v, n);
  return cudaGetLastError();
}

cudaError_t configure_edge_kernels();
cudaError_t configure_kernels() {
  cudaError_t e = cudaFuncSetAttribute(conv3x3_tc_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)ConvCfg<0>::kSmem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(conv3x3_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)ConvCfg<1>::kSmem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(conv3x3_tc_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)ConvCfg<3>::kSmem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(conv3x3_tc_kernel<12>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)ConvCfg<12>::kSmem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(conv3x3_tc_kernel<13>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)ConvCfg<13>::kSmem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(conv3x3_tc_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)ConvCfg<4>::kSmem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(conv3x3_tc_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)ConvCfg<5>::kSmem);
  if (e != cudaSuccess) return e;
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(conv3x3_tc_kernel<7>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)ConvCfg<7>::kSmem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(conv3x3_tc_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)ConvCfg<8>::kSmem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(conv3x3_tc_kernel<9>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)ConvCfg<9>::kSmem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(conv3x3_tc_kernel<11>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)ConvCfg<11>::kSmem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(conv3x3_tc_kernel<10>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)ConvCfg<10>::kSmem);
  if (e != cudaSuccess) return e;
  return configure_edge_kernels();
}

}  // namespace tvs
