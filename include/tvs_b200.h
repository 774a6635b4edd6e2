/* tvs_b200.h — C ABI of the B200-native TVSpecNET forward (libtvsb200.so).
 *
 * This is the drop-in boundary for the reference's model module
 * /root/reference/pkg/trainer/src/tvsurrogate/model.py:29-56.  The reference
 * has no FFI (pure PyTorch CPU); every entry point below replaces a piece of
 * the in-process call the reference makes:
 *
 *   tvs_plan_create       <- TVSpecNet.__init__(depth, channels, out_bands)   model.py:32-47
 *   tvs_plan_set_weights  <- load_state_dict + eval() (BN running stats)       training.py:163-172
 *   tvs_forward           <- TVSpecNet.forward(x) -> (B, out_bands, H, W)      model.py:49-52
 *                            (+ optional closure plane image - sum(bands),     inference.py:34-42)
 *   tvs_forward_host      <- predict_bands(model, image) with CPU in/out       inference.py:25-32
 *   tvs_plan_sync         <- the point where the reference's synchronous forward has returned
 *   tvs_plan_destroy      <- module teardown
 *
 * Conventions: every function returns 0 on success or a negative TVS_E_*
 * code; no C++ exception crosses the boundary; tvs_last_error() returns the
 * calling thread's last message.  All device pointers are caller-owned; the
 * plan owns packed weights, TMA descriptors and activation scratch.  Calls
 * on one plan must be serialised by the caller (one plan per device; plans on
 * different devices are independent).  `stream` is a cudaStream_t (NULL =
 * legacy default stream).
 */
#ifndef TVS_B200_H_
#define TVS_B200_H_

#ifdef __cplusplus
extern "C" {
#endif

#define TVS_ABI_VERSION 2

/* status codes */
#define TVS_OK 0
#define TVS_E_INVALID (-1)     /* bad argument (shape, depth, null pointer) -> ValueError */
#define TVS_E_UNSUPPORTED (-2) /* valid model, configuration not built (e.g. channels != 64) */
#define TVS_E_CUDA (-3)        /* CUDA runtime/driver failure */
#define TVS_E_STATE (-4)       /* forward before set_weights, etc. */
#define TVS_E_NUMERIC (-5)     /* a finite input produced non-finite bands (fp16-range overflow) */

/* numerics modes */
#define TVS_MODE_FP32 0 /* fp32-accurate (<= 1e-5): split fp16 hi/lo operands on tcgen05 */
#define TVS_MODE_FAST 1 /* fp16 tcgen05 hidden layers, exact fp32 conv0 + head (<= 1e-2) */

typedef struct tvs_plan tvs_plan;

int tvs_abi_version(void);
const char* tvs_last_error(void);

/* depth >= 3 (model.py:34-35); channels 64 or 128 (the wide variant: FAST on tcgen05,
 * FP32 on CUDA cores); 1 <= out_bands <= 8 */
int tvs_plan_create(int device, int depth, int channels, int out_bands, int mode, tvs_plan** out_plan);

/* As tvs_plan_create, plus unshuffle in {1, 2}.  unshuffle = 2 is the opt-in
 * F-TVSpecNET-style variant (not the reference architecture):
 * pixel_unshuffle(x, 2) -> Conv2d(4, C) ... Conv2d(C, 4K) -> pixel_shuffle(., 2),
 * with the unshuffle folded into conv0's loads and the shuffle into the head's
 * stores; the hidden stack runs on the (H/2, W/2) grid.  Weights:
 * conv0 (C, 4, 3, 3), head (4K, C, 3, 3), 4K <= 32.  H, W and the row window
 * must be even.  FAST mode, channels 64 only. */
int tvs_plan_create_ex(int device, int depth, int channels, int out_bands, int mode, int unshuffle,
                       tvs_plan** out_plan);

/* n_layers == depth.  Layer i computes  y[co] = scale[co] * conv(W_i, a)[co] + shift[co]
 * (then ReLU for all but the head).  w_dev[i]: DEVICE pointer to the conv
 * weights [cout][cin][3][3] fp32; scale_dev[i]: DEVICE pointer to [cout]
 * fp32, or NULL for 1 (scale_dev itself may be NULL); shift_dev[i]: DEVICE
 * pointer to [cout] fp32.  For the reference module: conv0/head have scale
 * NULL and shift = conv bias; hidden layer j has the eval-BatchNorm fold
 * scale = gamma/sqrt(var+eps), shift = beta - mean*scale (model.py:40-43).
 * The plan repacks on `stream` (FAST: W*scale rounded to fp16 with tap-sum
 * compensation); the sources may be freed once the stream passes this call. */
int tvs_plan_set_weights(tvs_plan* plan, const float* const* w_dev, const float* const* scale_dev,
                         const float* const* shift_dev, int n_layers, void* stream);

/* Plan options; unknown names or bad values -> TVS_E_INVALID.
 *   "check"        1 (default): tvs_forward verifies the forward's status words
 *                  before returning (it synchronises `stream`) and returns
 *                  TVS_E_CUDA / TVS_E_NUMERIC instead of invalid output.
 *                  2: deferred - the status is evaluated by a later tvs_forward
 *                  or tvs_plan_sync (async callers).  0: unchecked.
 *   "stack"        -1 auto / 0 / 1: the all-hidden-layers-in-one-launch kernel
 *   "watchdog_ms"  layer-stack row-flag wait limit (default 2000)
 *   "input_scale"  1 (default): per-image power-of-two activation scale that
 *                  keeps the fp16-range formats finite for any input magnitude
 *   "span" (see tvs_profile_span), "conv0_tc", "chunk_mb", "debug"; and, applied by the next
 *   tvs_plan_set_weights: "fp32_cuda", "wide_cuda", "wide_pair_layers",
 *   "wide_halves". */
int tvs_plan_set_option(tvs_plan* plan, const char* name, long long value);

/* Synchronise `stream` and evaluate every outstanding (deferred) status:
 * returns the first failure of a forward since the last sync. */
int tvs_plan_sync(tvs_plan* plan, void* stream);

/* x: (B,1,H,W) fp32 NCHW; bands: (B,out_bands,valid_rows,W) fp32 receiving
 * rows [valid_row0, valid_row0+valid_rows) of the full forward; closure (may
 * be NULL): (B,1,valid_rows,W) = x - sum_k bands_k.  valid_rows < 0 means all
 * H rows.  All device pointers, 16-byte aligned.  With the default "check"
 * option the call returns once the forward has completed and either the
 * output is valid (TVS_OK) or an error is returned: a layer-stack watchdog
 * expiry (TVS_E_CUDA; the next forward is unaffected) or non-finite bands from
 * a finite input (TVS_E_NUMERIC).  Non-finite inputs propagate as in the
 * reference's fp32 forward. */
int tvs_forward(tvs_plan* plan, const float* x, float* bands, float* closure_or_null, int B, int H, int W,
                int valid_row0, int valid_rows, void* stream);

/* tvs_forward with the fused band-sum reconstruction check (north_star item 3;
 * the closure identity of inference.py:34-42, tested by the reference at
 * pkg/trainer/tests/test_inference.py:31-38).  `closure` is required.  The
 * head kernel's epilogue evaluates r = x - (sum_k bands_k + closure) from the
 * fp32 values it stores and accumulates, per image b over the row window,
 *   recon[2b]   = sum r^2,   recon[2b+1] = sum x^2     (fp64)
 * into `recon`, a caller-owned DEVICE buffer of 2*B doubles (zeroed by the
 * call, stream-ordered).  sqrt(recon[2b] / recon[2b+1]) is the image's
 * relative reconstruction error. */
int tvs_forward_checked(tvs_plan* plan, const float* x, float* bands, float* closure, double* recon, int B, int H,
                        int W, int valid_row0, int valid_rows, void* stream);

/* Same contract with HOST buffers: copies in, runs, copies out, and
 * synchronises `stream` before returning. */
int tvs_forward_host(tvs_plan* plan, const float* x_host, float* bands_host, float* closure_host_or_null, int B,
                     int H, int W, void* stream);

/* Number of kernels the last tvs_forward launched (for launch accounting),
 * and whether it ran the layer-stack kernel. */
int tvs_last_launch_count(const tvs_plan* plan);
int tvs_last_used_stack(const tvs_plan* plan);

/* Per-kernel CUDA-event timing on the forward's stream (off by default).
 * kind: 0 = conv0 (K1), 1 = hidden conv (K2), 2 = head + closure (K3).
 * tvs_profile_read synchronises the recorded events and returns, since the
 * last enable/reset, the summed device milliseconds, the launch count and the
 * algorithmic FLOPs of those launches. */
#define TVS_KIND_CONV0 0
#define TVS_KIND_HIDDEN 1
#define TVS_KIND_HEAD 2
int tvs_profile_enable(tvs_plan* plan, int on);
int tvs_profile_read(tvs_plan* plan, int kind, double* total_ms, long long* launches, double* flops);

/* With plan option "span" = 1, every hidden-layer kernel launch (the layer
 * stack, or each per-layer conv) records its device duration from inside the
 * kernel: globaltimer from the first CTA past its PDL wait to the last CTA's
 * exit, so measuring does not perturb the launch overlap.  Returns the summed
 * milliseconds and launch count since the last reset (synchronises the device). */
int tvs_profile_span(tvs_plan* plan, double* total_ms, long long* launches, int reset);

int tvs_plan_destroy(tvs_plan* plan);

/* ---- Training step: replaces the train-mode forward and
 * the autograd backward of TVSpecNet (model.py:29-52, BatchNorm2d with batch
 * statistics) inside _epoch_pass (training.py:45-61).  64 channels.
 *
 *   tvs_train_create   <- TVSpecNet(depth, out_bands) in train() mode
 *   tvs_train_forward  <- model(img) with model.training == True
 *   tvs_train_backward <- loss.backward() through the model
 *
 * Forward: w_dev[i] conv weights [cout][cin][3][3] fp32 (i = 0..depth-1),
 * bias_dev[0] / bias_dev[depth-1] the conv0 / head biases (others ignored),
 * gamma_dev[j] / beta_dev[j] the BatchNorm affine parameters of hidden layer j
 * (j = 0..depth-3), all DEVICE pointers that must stay valid until the
 * matching backward returns.  out: (B,out_bands,H,W) fp32.  mean_out /
 * var_out: (depth-2) x 64 batch mean and UNBIASED variance per hidden layer
 * (the caller updates running_mean / running_var with its momentum, as
 * BatchNorm2d does).  Activations for the backward stay in the train plan: one
 * forward/backward pair at a time per plan.
 * Backward: g_out = dL/d(out) (B,out_bands,H,W) fp32; writes dw[i] (conv
 * weight layout), dbias[0], dbias[depth-1], dgamma[j], dbeta[j], fp32 DEVICE. */
typedef struct tvs_train tvs_train;
int tvs_train_create(int device, int depth, int out_bands, tvs_train** out_plan);
int tvs_train_forward(tvs_train* plan, const float* const* w_dev, const float* const* bias_dev,
                      const float* const* gamma_dev, const float* const* beta_dev, float eps, const float* x,
                      float* out, float* mean_out, float* var_out, int B, int H, int W, void* stream);
int tvs_train_backward(tvs_train* plan, const float* g_out, float* const* dw, float* const* dbias,
                       float* const* dgamma, float* const* dbeta, void* stream);
/* Training options (the train-plan counterpart of tvs_plan_set_option):
 *   "wgrad_tc"  1 (default) weight gradients on the tcgen05 kernel (wgrad_tc.cu),
 *               0 one cuBLAS split-K GEMM per filter tap.
 *   "head_dgrad_tc" 1 (default) the head's input gradient on the hidden layers'
 *               tcgen05 dgrad kernel (fp16 operands), 0 the fp32 CUDA-core kernel.
 *   "bn_bwd_fused" 1 (default) BatchNorm backward's reduction and apply passes in
 *               one cooperative launch, 0 two kernels.
 *   "bn_fused"  1 (default) BatchNorm's batch sums come from the forward conv's
 *               epilogue, 0 from a separate pass over the conv output. */
int tvs_train_set_option(tvs_train* plan, const char* name, int value);
int tvs_train_destroy(tvs_train* plan);

/* Training losses: replaces compute_loss (tvsurrogate
 * losses.py:54-129) and its autograd graph inside _epoch_pass (training.py:51-53).
 * pred, gt: DEVICE (B,K,H,W) fp32; image, residual: DEVICE (B,1,H,W) fp32 (only
 * read for the sum constraint).  terms: bit 0 = sum constraint (selectors L1 /
 * L3), bit 1 = gradient Huber (L2 / L3); huber_delta = losses.HUBER_DELTA.
 * tvs_loss_sums writes
 *   sums   DEVICE B*K*4 + B*2 doubles: per (b,k) [gt energy, residual energy,
 *          Huber numerator, Huber denominator], then per b [reconstruction
 *          error, image energy]
 *   values DEVICE 8 floats: [0] total [1] mse [2] sum term [3] gradient term
 *          [4] zero-energy bands skipped [5] zero-gradient bands skipped
 *          [6] bands with energy (0 -> the reference raises ValueError)
 * tvs_loss_grad writes grad_pred = *g_total (DEVICE scalar) * d total / d pred
 * from the same sums.  Both run on the caller's current device. */
int tvs_loss_sums(const float* pred, const float* gt, const float* image, const float* residual, int B, int K, int H,
                  int W, int terms, float huber_delta, double* sums, float* values, void* stream);
int tvs_loss_grad(const float* pred, const float* gt, const float* image, const float* residual, int B, int K, int H,
                  int W, int terms, float huber_delta, const double* sums, const float* g_total, float* grad_pred,
                  void* stream);

/* Band scoring statistics (spectv metrics.py:28-237), fp64.
 * gt, pred: DEVICE (planes, H, W) fp32.  stats: DEVICE planes x 8 doubles:
 *   [0] sum (gt - pred)^2           -> PSNR / MSE   (metrics.py:28-37)
 *   [1] sLMSE numerator, [2] denominator: sums over 16x16 patches at stride 8
 *       (+ clipped tail patch) of (gt-pred)^2 and pred^2   (metrics.py:126-150)
 *   [3] gt max, [4] gt min           -> data range      (metrics.py:222-225)
 *   [5] sum of the 11x11 Gaussian SSIM map over the interior, [6] interior
 *       pixel count                  -> windowed SSIM   (metrics.py:61-112)
 *   [7] unused
 * range_or_null: DEVICE planes doubles = SSIM data range per plane (ssim(...,
 * data_range), metrics.py:61); NULL = each gt plane's own floored range
 * (band_metrics convention).  Replaces the per-plane numpy loop of
 * band_metrics (metrics.py:211-237). */
int tvs_band_stats(const float* gt, const float* pred, int planes, int H, int W, const double* range_or_null,
                   double* stats, void* stream);

/* Model-driven TV-flow decomposition: the ground-truth producer (SURVEY §8(f)
 * row 3).  Replaces ModelDrivenDecomposer.analyze (spectv pipeline.py:105-145)
 * with rof_prox's accelerated primal-dual solver (solver.py:242-372): fp64,
 * reference operation order, one persistent CTA per image.
 *   f          DEVICE (N, H, W) fp64 finite images, W <= 2048
 *   schedule   HOST n_bands (<= 16) inclusive band end indices on the fine grid
 *              1..n_steps-1, strictly increasing, last == n_steps-1
 *              (transform.py:131-144, dyadic_schedule :186-207)
 *   solver     max_iters >= 1, gap_tol > 0, pd_tau*pd_sigma*8 <= 1, pd_accel
 *              0/1 (SolverConfig, solver.py:54-90; method primal-dual only)
 *   workspace  DEVICE, >= tvs_tvflow_workspace_bytes(N, H, W)
 *   bands      DEVICE (N, n_bands, H, W) fp64, last band includes the residual
 *   spectrum   DEVICE (N, n_steps-1) fp64: S(t_i) = sum |phi_i|
 *   residual   DEVICE (N, H, W) fp64: f_r = u_N - N (u_N - u_{N-1})
 *   iters      DEVICE (N, n_steps) int32: prox iterations of each flow step,
 *              stored as -(iters+1) when the gap tolerance was not certified
 *              (the reference's `warnings` list, pipeline.py:116-127). */
size_t tvs_tvflow_workspace_bytes(int N, int H, int W);
int tvs_tvflow_analyze(const double* f, int N, int H, int W, double dt, int n_steps, const int* schedule,
                       int n_bands, int max_iters, double gap_tol, double pd_tau, double pd_sigma, int pd_accel,
                       void* workspace, double* bands, double* spectrum, double* residual, int* iters,
                       void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TVS_B200_H_ */
