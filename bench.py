#!/usr/bin/env python
"""TVSpecNET K-band decomposition throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

One step = one forward of the config's whole batch through the drop-in
``TVSpecNet`` (conv0 -> 15 tcgen05 hidden convs -> head + closure), inputs
resident in HBM.  Default workload: BASELINE.json configs[1] = config 2,
64 x 1 x 256 x 256, fast (fp16 tcgen05) mode; the fp32-accurate mode is
measured on the same workload and reported alongside.  Multi-GPU (torchrun):
every rank processes its own config-2 batch (weak scaling, no collective on
the data path); value = all ranks' megapixels / max-over-ranks time.

``--impl reference`` times the reference's CPU forward (the oracle port of
/root/reference/pkg/trainer/src/tvsurrogate/model.py, identical torch CPU ops)
on the host cores, rank 0 only, on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2006_10004_b200.workloads import CONFIGS, flop_per_px, make_image  # noqa: E402

METRIC = "TVSpecNET megapixels/sec (K-band decomposition)"
UNIT = "MP/s"


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["bf16_tflops"], d.get("bf16_tflops_sustained"), d["hbm_gbs"], "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi-equivalent clock/throttle sampling (NVML) during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x20: "sync_boost", 0x40: "sw_thermal_slowdown", 0x80: "hw_thermal_slowdown",
        0x100: "hw_power_brake_slowdown", 0x200: "display_clock_setting",
    }

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                mask = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        if self.nvml:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nvml:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def _kernel_name(tc, used_stack, depth):
    """The dominant kernel: the layer-stack launch (all hidden layers, conv_tc.cu
    mode 8) when the forward ran it, else the per-layer hidden conv; the
    128-channel wide variant runs conv_tc.cu modes 5 (pair input) / 11 (single)."""
    if tc == "wide":
        return "conv3x3_tc_kernel<5>/<11> (wide hidden layers, 128 ch: pair input on quarters, single on halves)"
    if not tc:
        return "hidden_f32_kernel"
    if used_stack:
        return f"conv3x3_tc_kernel<8> (layer stack: {depth - 2} hidden layers per launch)"
    return "conv3x3_tc_kernel<0> (hidden layer)"


def _traffic(spec, kernel):
    """dram read+write bytes per launch of the dominant kernel from the committed
    ncu capture (profiles/traffic.json), when it was taken on this workload."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text()).get(kernel.split(" ")[0], {})
    if d.get("config") != spec.name:
        return None
    return d["dram_bytes_read"] + d["dram_bytes_write"]


def tc_stack_probe(plan, step):
    """Run one forward with the stack kernel's cycle accounting on; sets
    tc_stack_probe.mhz (None when the forward did not use the layer stack)."""
    import ctypes

    from paper_2006_10004_b200 import _native

    tc_stack_probe.mhz = None
    lib = _native.load()
    if not hasattr(lib, "tvs_debug_cycles"):
        return False
    lib.tvs_debug_cycles.restype = ctypes.c_int
    lib.tvs_debug_cycles.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    buf = (ctypes.c_ulonglong * 8)()
    torch.cuda.synchronize()
    lib.tvs_debug_cycles(buf, 1)
    plan.set_option("debug", 32768)  # MMA-issuer cycle accounting (conv_tc.cu)
    try:
        step()
        torch.cuda.synchronize()
    finally:
        plan.set_option("debug", 0)
    lib.tvs_debug_cycles(buf, 1)
    if buf[6] == 0:
        return False
    tc_stack_probe.mhz = round(buf[0] / buf[6] * 1e3, 1)
    return True


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _batch(spec, count=None):
    n = spec.batch if count is None else count
    return np.stack([make_image(spec, i) for i in range(n)])[:, None]


def _seeded_state(depth, channels):
    from oracle.tvspecnet_oracle import build_seeded_state  # checker-side weight recipe only

    return build_seeded_state(depth, channels, 5)


def cpu_reference(spec, steps, warmup, sample_images, threads, budget_s=None):
    """The reference CPU forward (oracle port), per image as predict_bands does
    (inference.py:25-32).  Each step runs `sample_images` images, or - with
    `budget_s` - as many images (>= 1) as fit in that many seconds."""
    from oracle.tvspecnet_oracle import oracle_from_state

    torch.set_num_threads(threads)
    model = oracle_from_state(_seeded_state(spec.depth, spec.channels), spec.depth, spec.channels, 5)
    n_max = min(spec.batch, sample_images)
    imgs = [torch.from_numpy(make_image(spec, j)[None, None]) for j in range(n_max)]
    rates, secs = [], []
    with torch.no_grad():
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            n = 0
            while n < n_max:
                model(imgs[n])
                n += 1
                if budget_s is not None and time.perf_counter() - t0 >= budget_s:
                    break
            dt = time.perf_counter() - t0
            if i >= warmup:
                rates.append(n * spec.height * spec.width / 1e6 / dt)
                secs.append((n, dt))
    return statistics.median(rates), secs


def run_reference(args, spec):
    world, rank, _ = _dist()
    if world > 1 and rank != 0:
        return
    threads = os.cpu_count() or 1
    budget = args.ref_step_seconds
    mp_s, secs = cpu_reference(spec, args.steps, args.warmup, spec.batch, threads, budget_s=budget)
    n_img = statistics.median([n for n, _ in secs])
    line = {
        "metric": METRIC, "value": round(mp_s, 5), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(statistics.median([d for _, d in secs]) * 1e3, 3),
        "higher_is_better": True, "scaling": _scaling(spec), "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (SURVEY §8(d) generator)", "impl": "reference",
        "config": {"workload": spec.name, "batch": spec.batch, "height": spec.height, "width": spec.width,
                   "depth": spec.depth, "channels": spec.channels},
        "cpu_baseline": {"value": round(mp_s, 5), "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"per step: images of this workload, one forward each (predict_bands style), "
                                   f"until {budget:g} s elapse (median {n_img:g} images), torch CPU (oneDNN) "
                                   f"fp32, {threads} threads"},
        "e2e": {"value": round(mp_s, 5), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _scaling(spec):
    # config 2: every rank its own batch (weak); single images are row-banded and
    # configs 4/5 batch-sharded across ranks (strong, fixed total work)
    return "weak" if spec.name.startswith("cfg2") else "strong"


def _flush_l2(buf):
    buf.add_(1.0)


def time_steps(fn, steps, warmup, flush, reset=None):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if reset is not None:
        reset()
    st = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in evs:
        _flush_l2(flush)
        a.record(st)
        fn()
        b.record(st)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def _rank_work(spec, world, rank):
    """This rank's images / rows.  Returns (image indices, row band or None)."""
    from paper_2006_10004_b200.shard import batch_shards, row_bands

    if spec.name.startswith("cfg2"):
        return list(range(spec.batch)), None  # weak scaling: each rank a full config-2 batch
    if spec.batch == 1:
        return [0], (row_bands(spec.height, world, spec.depth)[rank] if world > 1 else None)
    s, n = batch_shards(spec.batch, world)[rank]
    return list(range(s, s + n)), None


def run_ours(args, spec):
    world, rank, local = _dist()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2006_10004_b200 import TVSpecNet

    state = _seeded_state(spec.depth, spec.channels)
    idx, band = _rank_work(spec, world, rank)
    x_np = np.stack([make_image(spec, i) for i in idx])[:, None]
    if band is not None:  # row band with receptive-field halo (shard.row_bands)
        x_np = np.ascontiguousarray(x_np[:, :, band.src0 : band.src1])
        row0, nrows = band.valid_row0, band.rows
    else:
        row0, nrows = 0, x_np.shape[2]
    x_host = torch.from_numpy(x_np).pin_memory()
    x = x_host.to(dev)
    B, _, H, W = x.shape
    px_out = B * nrows * W  # output pixels this rank produces
    total_px = (spec.batch * spec.height * spec.width) if _scaling(spec) == "strong" else world * px_out
    flush = torch.empty(256 << 20 >> 2, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2

    precs = ["fast"] + (["fp32"] if args.fp32_fast_steps > 0 else [])
    if args.fp32_steps > 0 and spec.channels == 64:
        precs.append("fp32cuda")
    if args.unshuffle_steps > 0 and spec.channels == 64 and H % 2 == 0 and W % 2 == 0 \
            and row0 % 2 == 0 and nrows % 2 == 0:
        precs.append("fast_u2")  # opt-in unshuffle = 2 variant (not the reference architecture)
    results = {}
    for prec in precs:
        if prec == "fast_u2":
            from oracle.tvspecnet_oracle import build_seeded_state  # checker-side weight recipe only

            model = TVSpecNet(spec.depth, spec.channels, 5, unshuffle=2).eval()
            model.load_state_dict(build_seeded_state(spec.depth, spec.channels, 5, unshuffle=2))
        else:
            model = TVSpecNet(spec.depth, spec.channels, 5, precision="fp32" if prec == "fp32cuda" else prec,
                              options={"fp32_cuda": 1} if prec == "fp32cuda" else None).eval()
            model.load_state_dict(state)
        bands = torch.empty((B, 5, nrows, W), device=dev)
        clos = torch.empty((B, 1, nrows, W), device=dev)
        plan = model._plan_for(dev)
        # timed steps: status words checked once at the end (deferred) instead
        # of a host synchronisation per forward; hidden-layer kernels record
        # their own device spans (tvs_profile_span) for the roofline
        plan.set_option("check", 2)
        plan.set_option("span", 1)

        def step():
            plan.forward(x.data_ptr(), bands.data_ptr(), clos.data_ptr(), B, H, W, row0, nrows,
                         torch.cuda.current_stream().cuda_stream)

        steps = args.steps if prec == "fast" else max(1, min(args.steps, args.fp32_steps))
        if prec == "fp32":
            steps = max(1, min(args.steps, args.fp32_fast_steps))
        if prec == "fast_u2":
            steps = max(1, min(args.steps, args.unshuffle_steps))
        warm = args.warmup if prec == "fast" else max(1, min(args.warmup, 3))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            plan.profile_span(reset=True)  # drops the warm-up launches inside time_steps below
            ms = time_steps(step, steps, warm, flush, reset=lambda: plan.profile_span(reset=True))
        span_ms, span_n = plan.profile_span(reset=True)
        plan.sync(torch.cuda.current_stream().cuda_stream)  # raises if any timed forward failed
        plan.set_option("check", 1)
        plan.set_option("span", 0)
        launches = plan.last_launch_count()
        used_stack = plan.last_used_stack()
        tot_ms = sum(ms)
        if world > 1:
            t = torch.tensor([tot_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tot_ms = float(t.item())
        value = total_px * steps / 1e6 / (tot_ms / 1e3)

        # algorithmic FLOPs of one hidden-layer launch (per-kernel accounting of the plan)
        plan.profile_enable(True)
        step()
        torch.cuda.synchronize()
        _, hid_n1, hid_flops1 = plan.profile_read(1)
        plan.profile_enable(False)
        hid_flops = hid_flops1 / max(1, hid_n1) * span_n

        # the SM clock the layer-stack kernel actually ran at (clock64 cycles
        # over globaltimer ns in its MMA thread, TVS_CONV_DBG bit 15): the
        # nvidia-smi sampler sees the idle gaps between launches, while the
        # stack runs power-limited
        in_kernel_mhz = None
        if prec == "fast" and tc_stack_probe(plan, step):
            in_kernel_mhz = tc_stack_probe.mhz

        # end to end through the public API with host buffers (pinned input ->
        # CPU result: H2D + forward + D2H inside the timed region), on at most
        # `e2e_max_images` images of this rank's work
        ne = max(1, min(B, args.e2e_max_images, (1 << 30) // (5 * 4 * nrows * W)))  # <= 1 GiB of pinned results
        xe = x_host[:ne]
        e2e_steps = max(1, min(steps, args.e2e_steps))
        out_host = None
        for _ in range(3):  # same pattern as timed: keeps two pinned result blocks cached
            out_host = model.forward_planes(xe, rows=(row0, nrows))[0]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            _flush_l2(flush)
            out_host = model.forward_planes(xe, rows=(row0, nrows))[0]
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        if world > 1:
            t = torch.tensor([e2e_s], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e_px = ne * nrows * W * world  # every rank times its own share (max over ranks below)
        results[prec] = dict(value=value, ms=tot_ms / steps, ms_list=ms, launches=launches, steps=steps,
                             warmup=warm, clocks=clk.summary(), hid_ms=span_ms, hid_n=span_n, hid_flops=hid_flops,
                             e2e=e2e_px / 1e6 / e2e_s, hid_per_fwd=span_n / steps, used_stack=used_stack,
                             in_kernel_mhz=in_kernel_mhz,
                             e2e_bytes=(xe.numel() * 4, out_host.numel() * 4), e2e_images=ne)
        del model, plan, bands, clos

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    peak_tf, peak_sus, hbm, peak_kind = _peaks()
    f = results["fast"]
    fpx = flop_per_px(spec.depth, spec.channels)
    hid_avg_ms = f["hid_ms"] / max(1, f["hid_n"])
    hid_tflops = f["hid_flops"] / max(1, f["hid_n"]) / (hid_avg_ms / 1e3) / 1e12
    step_ms = f["ms"]
    tc = True if spec.channels == 64 else "wide"  # both fast paths run on tcgen05
    wide_pairs = min(12, spec.depth - 2)  # the plan's default pair-input layers (tvs_api.cu wide_pair_layers)
    nh = spec.depth - 2
    # algorithmic activation bytes per hidden launch (read + write one activation):
    # 64 ch fp16 = 128 B/px each way; wide pair = 512, single = 256 B/px
    if tc is True:
        alg_bytes_px = 2 * 128
    else:
        alg_bytes_px = sum((512 if j < wide_pairs else 256) + (512 if j + 1 < wide_pairs else 256)
                           for j in range(nh)) / nh
    parallelism = (f"row-bands x{world} (halo {spec.depth})" if band is not None else
                   ("batch per rank" if _scaling(spec) == "weak" else f"batch-shard x{world}"))
    line = {
        "metric": METRIC, "value": round(f["value"], 3), "unit": UNIT, "n_gpus": world, "steps": f["steps"],
        "warmup": f["warmup"], "ms_per_step": round(step_ms, 4), "higher_is_better": True,
        "scaling": _scaling(spec), "vs_baseline": None,
        "dtype": ("f16 operands / f32 accumulate (tcgen05 kind::f16); conv0+head f32" if tc is True
                  else f"f16 operands / f32 accumulate (tcgen05 kind::f16), first {wide_pairs} of {nh} hidden "
                       "layers on fp16 hi/lo activation pairs; conv0+head f32"),
        "data": f"synthetic (SURVEY §8(d) piecewise-constant generator, seed {spec.seed})",
        "config": {"workload": spec.name, "batch": spec.batch, "rank_images": B, "height": spec.height,
                   "width": spec.width, "depth": spec.depth, "channels": spec.channels, "out_bands": 5,
                   "precision": "fast", "parallelism": parallelism,
                   "l2": "256 MiB buffer written between timed steps", "inputs_resident": "HBM"},
        "latency_ms": round(step_ms, 4) if spec.batch == 1 else None,
        "tflops_algorithmic": round(f["value"] * 1e6 * fpx / 1e12 / world, 2),
        "frac_of_bf16_peak": round(f["value"] * 1e6 * fpx / 1e12 / world / peak_tf, 4),
        "roofline": {"bound": "tensor", "kernel": _kernel_name(tc, f["used_stack"], spec.depth),
                     "achieved": round(hid_tflops, 2), "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": round(hid_tflops / peak_tf, 4), "peak_kind": f"{peak_kind} bf16 burst",
                     "frac_of_sustained": round(hid_tflops / peak_sus, 4) if peak_sus else None,
                     "avg_launch_ms": round(hid_avg_ms, 5), "launches_timed": f["hid_n"],
                     "launch_timing": "in-kernel globaltimer span of each launch inside the timed steps "
                                      "(first CTA past its PDL wait to last CTA exit; tvs_profile_span)",
                     "flop_per_launch": f["hid_flops"] / max(1, f["hid_n"]),
                     "share_of_step": round(f["hid_ms"] / max(1e-9, step_ms * f["steps"]), 4),
                     "whole_forward_frac": round(f["value"] * 1e6 * fpx / 1e12 / world / peak_tf, 4),
                     "traffic": _traffic(spec, _kernel_name(tc, f["used_stack"], spec.depth)),
                     "traffic_unit": "bytes per launch (ncu dram read+write)",
                     "algorithmic_bytes_per_launch": int(B * H * W * alg_bytes_px)},
        "gpu_launches": f["launches"] * f["steps"],
        "e2e": {"value": round(f["e2e"], 3), "unit": UNIT, "h2d_bytes_per_step": f["e2e_bytes"][0],
                "d2h_bytes_per_step": f["e2e_bytes"][1], "images_per_rank": f["e2e_images"]},
        "clocks": dict(f["clocks"], **({"stack_kernel_sm_mhz": f["in_kernel_mhz"],
                                          "stack_kernel_sm_mhz_note": "clock64/globaltimer in the layer-stack "
                                          "kernel's MMA thread during one forward (nvidia-smi samples the gaps)"}
                                         if f.get("in_kernel_mhz") else {})),
    }
    if "fp32" in results:
        r32 = results["fp32"]
        line["fp32_mode"] = {"value": round(r32["value"], 3), "unit": UNIT, "ms_per_step": round(r32["ms"], 3),
                             "steps": r32["steps"], "e2e": round(r32["e2e"], 3)}
    if "fast_u2" in results:
        r = results["fast_u2"]
        line["unshuffle2_variant"] = {
            "value": round(r["value"], 3), "unit": UNIT, "ms_per_step": round(r["ms"], 3), "steps": r["steps"],
            "e2e": round(r["e2e"], 3),
            "note": "opt-in TVSpecNet(unshuffle=2): pixel_unshuffle folded into conv0 loads, pixel_shuffle into "
                    "the head stores, hidden stack on the (H/2, W/2) grid; NOT the reference architecture "
                    "(SURVEY F2), parity vs a torch composition oracle"}
    if "fp32cuda" in results:
        r = results["fp32cuda"]
        line["fp32_mode_cuda_cores"] = {"value": round(r["value"], 3), "unit": UNIT,
                                        "ms_per_step": round(r["ms"], 3), "steps": r["steps"],
                                        "note": "TVS_FP32_CUDA=1: fp32 FFMA + fp64 combine kernels"}
    if world == 1 and args.train_steps > 0 and str(args.config) == "2":
        try:
            line["train_step"] = train_step_leg(state, args.train_steps)
        except Exception as e:  # never lose the bench line to the extra leg
            line["train_step"] = {"error": f"{type(e).__name__}: {e}"[:200]}
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        mp_s, secs = cpu_reference(spec, 1, 0, spec.batch, threads, budget_s=args.cpu_seconds)
        n, dt = secs[0]
        line["cpu_baseline"] = {"value": round(mp_s, 5), "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": f"{n} of {spec.batch} images ({dt:.1f} s), one forward per image, "
                                          f"torch CPU fp32 oracle port, {threads} threads"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def train_step_leg(state, steps, B=8, S=128):
    """SURVEY §8(f) row 4 beside the inference line: one _epoch_pass iteration
    (training.py:45-61: zero_grad, model(img), compute_loss, backward, Adam step,
    loss read) through the drop-in's train() mode and fused losses, at the
    reference's batch size 8 on seeded synthetic 128 x 128 crops."""
    from paper_2006_10004_b200 import TVSpecNet
    from paper_2006_10004_b200.losses import compute_loss

    m = TVSpecNet()
    m.load_state_dict(state)
    m = m.cuda().train()
    opt = torch.optim.Adam(m.parameters(), lr=1e-3)
    g = torch.Generator().manual_seed(3)
    gt = torch.randn(B, 5, S, S, generator=g).cuda()
    res = (0.1 * torch.randn(B, 1, S, S, generator=g)).cuda()
    img = gt.sum(1, keepdim=True) + res
    warm = 3
    for it in range(warm + steps):
        if it == warm:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
        opt.zero_grad(set_to_none=True)
        v = compute_loss(m(img), gt, img, res, "L")
        v.total.backward()
        opt.step()
        loss = float(v.total.detach())
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    return {"value": round(1.0 / dt, 2), "unit": "steps/s", "ms_per_step": round(dt * 1e3, 3), "batch": B,
            "size": [S, S], "steps": steps, "selector": "L", "last_loss": round(loss, 6),
            "note": "forward (batch-stat BN, split tcgen05 convs) + fused loss + backward (tcgen05 dgrad/wgrad) + "
                    "Adam, wall clock incl. the per-step loss read; tools/bench_train.py times the CPU flow beside it"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="2")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU baseline sample budget (s)")
    ap.add_argument("--ref-step-seconds", type=float, default=4.0, help="--impl reference: seconds per step")
    ap.add_argument("--fp32-steps", type=int, default=None,
                    help="steps of the CUDA-core fp32 kernels (TVS_FP32_CUDA=1) (0 = skip)")
    ap.add_argument("--unshuffle-steps", type=int, default=10,
                    help="steps of the opt-in unshuffle=2 variant (0 = skip)")
    ap.add_argument("--fp32-fast-steps", type=int, default=10,
                    help="steps of the fp32-accurate mode (tcgen05 split operands) (0 = skip)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-max-images", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--train-steps", type=int, default=10, help="steps of the training-step leg (0 = skip)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    key = args.config if args.config == "5w" else int(args.config)
    spec = CONFIGS[key]
    if args.fp32_steps is None:  # the CUDA-core fp32 mode takes ~0.1 s/MP: only on the small configs
        args.fp32_steps = 3 if spec.batch * spec.height * spec.width <= (1 << 23) else 0
    if args.impl == "reference":
        run_reference(args, spec)
    else:
        run_ours(args, spec)


if __name__ == "__main__":
    main()
