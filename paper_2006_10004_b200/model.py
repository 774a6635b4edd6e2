"""Drop-in TVSpecNet whose forward runs on hand-written sm_100a kernels.

Mirrors /root/reference/pkg/trainer/src/tvsurrogate/model.py:

* ``ARCH_SPEC``            — model.py:19-26 (unchanged constants)
* ``TVSpecNet(depth=17, channels=64, out_bands=5)`` — model.py:29-47: the
  same ``nn.Sequential`` body, so ``state_dict`` keys/shapes, ``depth`` and
  ``out_bands`` attributes, module counts and ``load_state_dict`` (strict)
  behave exactly like the reference (training.py:163-172 loads into it).
* ``forward(x)``           — model.py:49-52: ValueError unless x is
  (B, 1, H, W); returns (B, out_bands, H, W) float32 on x's device.
* ``receptive_field``      — model.py:55-56.

What differs is where the arithmetic happens: ``forward`` turns eval-mode
BatchNorm into per-channel scale/shift (fp64 on the host side, cached by
parameter versions), hands them to a per-device C-ABI plan (libtvsb200.so), and runs
conv0 -> 15 tcgen05 hidden convs -> head on the GPU.  CPU tensors are copied
to the execution device and the result copied back, so the reference's CPU
callers (``predict_bands``, inference.py:25-32) work unchanged.  There is no
CPU fallback: ``forward`` raises when no CUDA device is present.  In
``train()`` mode it runs the B200 training step (train_step.py, csrc/train.cu):
batch-statistics BatchNorm, an autograd backward on the C ABI, and the
running-stat updates, so the reference's training loop (training.py:45-61)
drives the drop-in unchanged.

``precision`` selects the numerics: ``"fast"`` (default; fp16 tcgen05 hidden
layers, exact fp32 conv0/head; <= 1e-2 relative L2 per band vs the fp32
reference) or ``"fp32"`` (split fp16 hi/lo operands on tcgen05; <= 1e-5).

``unshuffle=2`` (keyword-only, default 1 = the reference architecture) builds
the opt-in F-TVSpecNET-style variant BASELINE.json's north_star describes but
the reference does not have: pixel_unshuffle(x, 2) -> Conv2d(4, C)
-> hidden stack on the (H/2, W/2) grid -> Conv2d(C, 4K) -> pixel_shuffle(., 2).
The unshuffle is folded into conv0's loads and the shuffle into the head's
stores (no separate passes).  Its parity reference is the torch composition in
oracle/tvspecnet_oracle.py (unpinned by the reference).  Fast mode only.
"""

from __future__ import annotations

import torch
from torch import nn

from . import _native

__all__ = ["ARCH_SPEC", "TVSpecNet", "receptive_field"]

ARCH_SPEC = {
    "depth": 17,
    "channels": 64,
    "kernel": 3,
    "out_bands": 5,
    "batch_norm": True,
    "receptive_field": 35,
}

_PRECISIONS = {"fp32": _native.MODE_FP32, "fast": _native.MODE_FAST}


class TVSpecNet(nn.Module):
    """DnCNN-shaped regressor from an image to its first ``out_bands`` bands."""

    def __init__(self, depth: int = 17, channels: int = 64, out_bands: int = 5, *, precision: str = "fast",
                 unshuffle: int = 1, options: dict | None = None):
        super().__init__()
        if depth < 3:
            raise ValueError("depth must be at least 3 (first, hidden, last)")
        if unshuffle not in (1, 2):
            raise ValueError("unshuffle must be 1 or 2")
        if unshuffle == 2 and precision != "fast":
            raise ValueError("unshuffle=2 is built for precision='fast'")
        u2 = unshuffle * unshuffle
        layers: list[nn.Module] = [nn.Conv2d(u2, channels, 3, padding=1, bias=True), nn.ReLU(inplace=True)]
        for _ in range(depth - 2):
            layers.append(nn.Conv2d(channels, channels, 3, padding=1, bias=False))
            layers.append(nn.BatchNorm2d(channels))
            layers.append(nn.ReLU(inplace=True))
        layers.append(nn.Conv2d(channels, out_bands * u2, 3, padding=1, bias=True))
        self.body = nn.Sequential(*layers)
        self.depth = depth
        self.out_bands = out_bands
        self.channels = channels
        self.unshuffle = unshuffle
        if precision not in _PRECISIONS:
            raise ValueError(f"precision must be one of {sorted(_PRECISIONS)}")
        self._precision = precision
        # C-ABI plan options (include/tvs_b200.h tvs_plan_set_option), applied
        # to every per-device plan this module creates
        self._options: dict[str, int] = dict(options or {})
        self._plans: dict[int, tuple[_native.Plan, tuple]] = {}

    # ------------------------------------------------------------ config ----
    @property
    def precision(self) -> str:
        return self._precision

    @precision.setter
    def precision(self, value: str) -> None:
        if value not in _PRECISIONS:
            raise ValueError(f"precision must be one of {sorted(_PRECISIONS)}")
        if getattr(self, "unshuffle", 1) == 2 and value != "fast":
            raise ValueError("unshuffle=2 is built for precision='fast'")
        if value != self._precision:
            self._precision = value
            self._drop_plans()

    @property
    def plan_options(self) -> dict:
        return dict(self._options)

    def set_plan_option(self, name: str, value: int) -> None:
        """Set a plan option (e.g. ``stack``, ``check``, ``watchdog_ms``); the
        per-device plans are rebuilt with it at the next forward."""
        self._options[name] = int(value)
        self._drop_plans()

    def _drop_plans(self) -> None:
        for plan, _ in self._plans.values():
            plan.close()
        self._plans.clear()

    def __getstate__(self):
        state = self.__dict__.copy()
        state["_plans"] = {}
        state["_train_plans"] = {}
        # per-process caches (device buffers, streams, events, module walks) never travel
        for k in ("_wk_cache", "_train_stage", "_train_layers", "_train_step_id", "_single_bufs", "_host_pipes",
                  "_row_pipes", "_sched_cache"):
            state.pop(k, None)
        return state

    def _train_plan(self, idx: int):
        from .train_step import new_train_plan

        plans = self.__dict__.setdefault("_train_plans", {})
        if idx not in plans:
            plans[idx] = new_train_plan(self, idx)
        return plans[idx]

    # ------------------------------------------------------ weight folding ----
    def _weight_key(self, device: torch.device) -> tuple:
        """Identity + version of every tensor the forward reads (checked on each
        call, so in-place updates such as load_state_dict repack the plan).
        Reads the body's parameter/buffer dicts directly (cached per module
        list; the dicts are iterated live, so replaced or newly set tensors
        are seen): list(self.parameters()) costs ~0.3 ms per call, this ~0.03."""
        mods = tuple(self.body._modules.values())
        cache = self.__dict__.get("_wk_cache")
        if cache is None or cache[0] != mods:  # (element-wise identity: nn.Module defines no __eq__)
            cache = (mods, [d for mod in mods for d in (mod._parameters, mod._buffers)])
            self.__dict__["_wk_cache"] = cache
        key = [(t.data_ptr(), t._version) for d in cache[1] if d for t in d.values() if t is not None]
        key.append((str(device), self._precision))
        return tuple(key)

    @torch.no_grad()
    def layer_params(self) -> list[tuple[torch.Tensor, torch.Tensor | None, torch.Tensor]]:
        """Per conv: (W, scale-or-None, shift) in fp64 with y = scale*conv(W, a) + shift.
        Eval BatchNorm2d (model.py:41): scale = gamma/sqrt(var+eps),
        shift = beta + (bias - mean)*scale; convs without BN: scale None, shift = bias."""
        mods = list(self.body)
        out = []
        for i, m in enumerate(mods):
            if not isinstance(m, nn.Conv2d):
                continue
            w = m.weight.detach().double()
            b = (m.bias.detach().double() if m.bias is not None
                 else torch.zeros(w.shape[0], dtype=torch.float64, device=w.device))
            nxt = mods[i + 1] if i + 1 < len(mods) else None
            if isinstance(nxt, nn.BatchNorm2d):
                s = nxt.weight.detach().double() / torch.sqrt(nxt.running_var.detach().double() + nxt.eps)
                out.append((w, s, nxt.bias.detach().double() + (b - nxt.running_mean.detach().double()) * s))
            else:
                out.append((w, None, b))
        return out

    def _plan_for(self, device: torch.device) -> _native.Plan:
        idx = device.index if device.index is not None else torch.cuda.current_device()
        key = self._weight_key(torch.device("cuda", idx))
        entry = self._plans.get(idx)
        if entry is not None and entry[1] == key:
            return entry[0]
        plan = entry[0] if entry is not None else self._new_plan(idx)
        self._load_plan(plan, idx)
        self._plans[idx] = (plan, key)
        return plan

    def _new_plan(self, idx: int) -> _native.Plan:
        """A fresh C-ABI plan on device `idx` with this module's options (no weights)."""
        plan = _native.Plan(idx, self.depth, self.channels, self.out_bands, _PRECISIONS[self._precision],
                            self.unshuffle)
        for name, value in self._options.items():
            plan.set_option(name, value)
        return plan

    @torch.no_grad()
    def _load_plan(self, plan: _native.Plan, idx: int) -> None:
        """Fold eval BatchNorm on the host side and hand the layers to `plan`."""
        with torch.cuda.device(idx):
            stream = torch.cuda.current_stream(idx)
            dev = torch.device("cuda", idx)
            staged = []
            for w, s, b in self.layer_params():
                staged.append((w.to(dev, torch.float32).contiguous(),
                               None if s is None else s.to(dev, torch.float32).contiguous(),
                               b.to(dev, torch.float32).contiguous()))
            plan.set_weights([w.data_ptr() for w, _, _ in staged],
                             [0 if s is None else s.data_ptr() for _, s, _ in staged],
                             [b.data_ptr() for _, _, b in staged], stream.cuda_stream)
            # keep the fp32 staging alive until the repack kernels have consumed it
            stream.synchronize()

    # ------------------------------------------------------------- forward ----
    def _exec_device(self, x: torch.Tensor) -> torch.device:
        if x.is_cuda:
            return x.device
        if not torch.cuda.is_available():
            raise RuntimeError("TVSpecNet (B200) needs a CUDA device; there is no CPU fallback")
        p = self.body._modules["0"]._parameters["weight"]  # (next(self.parameters()) walks named_modules: 12 us)
        if p.is_cuda:
            return p.device
        return torch.device("cuda", torch.cuda.current_device())

    def _check_input(self, x: torch.Tensor) -> None:
        if x.ndim != 4 or x.shape[1] != 1:
            raise ValueError(f"expected (batch, 1, h, w) input, got {tuple(x.shape)}")
        if x.dtype != torch.float32:
            raise RuntimeError(f"Input type ({x.dtype}) and weight type (torch.float32) should be the same")
        if self.unshuffle == 2 and (x.shape[2] % 2 or x.shape[3] % 2):
            raise ValueError(f"unshuffle=2 needs even height and width, got {tuple(x.shape[2:])}")

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if self.training:
            from .train_step import TrainForward, train_params

            self._check_input(x)
            return TrainForward.apply(self, x, *train_params(self))
        return self.forward_planes(x)[0]

    def forward_planes(self, x: torch.Tensor, closure: bool = False, rows: tuple[int, int] | None = None,
                       check_reconstruction: bool = False):
        """(bands, closure-or-None).  ``closure`` adds the band-sum
        reconstruction plane image - sum(bands) (inference.py:34-42) from the
        head kernel's epilogue; ``rows=(row0, nrows)`` returns only that row
        window of the full-image forward (row-band sharding).

        ``check_reconstruction`` (implies ``closure``; CUDA tensors) returns
        (bands, closure, rel) with rel[b] = ||x - sum(bands) - closure|| /
        ||x|| over the row window, evaluated by the head epilogue from the
        stored values (tvs_forward_checked) - the identity the reference tests
        at 1e-5 (pkg/trainer/tests/test_inference.py:31-38)."""
        self._check_input(x)
        if self.training:
            raise RuntimeError("forward_planes is the eval-mode (inference) forward; call .eval() first")
        dev = self._exec_device(x)
        plan = self._plan_for(dev)
        B, _, H, W = x.shape
        row0, nrows = (0, H) if rows is None else rows
        if not (0 <= row0 and nrows >= 1 and row0 + nrows <= H):
            raise ValueError(f"bad row window {rows} for height {H}")
        if self.unshuffle == 2 and (row0 % 2 or nrows % 2):
            raise ValueError(f"unshuffle=2 needs an even row window, got {rows}")
        if check_reconstruction and not x.is_cuda:
            raise ValueError("check_reconstruction needs a CUDA input (device-side check sums)")
        if B == 0:  # an empty batch is a valid forward (the reference returns (0, K, H, W)): nothing to launch
            bands = x.new_empty((0, self.out_bands, nrows, W))
            clos = x.new_empty((0, 1, nrows, W)) if (closure or check_reconstruction) else None
            if check_reconstruction:
                return bands, clos, x.new_empty((0,), dtype=torch.float64)
            return bands, clos
        if not x.is_cuda:
            return self._forward_host(plan, x, dev, closure, row0, nrows)
        closure = closure or check_reconstruction
        with torch.cuda.device(dev):
            stream = torch.cuda.current_stream(dev)
            xd = x.contiguous()
            bands = torch.empty((B, self.out_bands, nrows, W), device=dev, dtype=torch.float32)
            clos = torch.empty((B, 1, nrows, W), device=dev, dtype=torch.float32) if closure else None
            if check_reconstruction:
                recon = torch.empty((B, 2), device=dev, dtype=torch.float64)
                plan.forward_checked(xd.data_ptr(), bands.data_ptr(), clos.data_ptr(), recon.data_ptr(), B, H, W,
                                     row0, nrows, stream.cuda_stream)
                rel = torch.sqrt(recon[:, 0] / recon[:, 1].clamp_min(torch.finfo(torch.float64).tiny))
                return bands, clos, rel
            plan.forward(xd.data_ptr(), bands.data_ptr(), clos.data_ptr() if closure else 0, B, H, W, row0, nrows,
                         stream.cuda_stream)
        return bands, clos

    # host tensors: pipelined H2D -> forward -> D2H over sub-batches.
    # None = automatic schedule (_host_schedule); an int = that many equal
    # sub-batches; a sequence = relative sub-batch sizes.
    host_chunks = None
    # single-sub-batch host path: results up to this size are written by the head
    # kernel directly into the pinned host tensor (0 = always copy)
    zero_copy_out_bytes = 8 << 20

    def _host_schedule(self, B: int, H: int, W: int, nrows: int, closure: bool, sms: int) -> list[int]:
        """Sub-batch sizes for the host-tensor pipeline.  Sub-batch i's D2H
        overlaps the forward of sub-batch i+1, and the last D2H is exposed, so
        sizes shrink towards the end (ratio ~ D2H time / forward time per
        image); a tiny first sub-batch starts the GPU after a short H2D; the
        big one is sized so the layer-stack kernel is eligible (tvs_api.cu
        run_chunk: >= 6 items per SM and a last round >= 95% full).  Candidate
        schedules are scored with a three-stream timeline model."""
        if B <= 2:
            return [B]
        us = self.unshuffle
        strips = (W // us + 127) // 128
        cols = strips * (self.depth - 2)
        fast = self._precision == "fast" and self.channels == 64
        px = H * W
        rate = (1.1e9 if fast else 0.27e9) / (self.channels / 64) ** 2 * (17 - 2) / max(1, self.depth - 2)
        t_h = 4.0 * px / 50e9
        t_d = 4.0 * (self.out_bands + (1 if closure else 0)) * nrows * W / 54e9

        def stack_ok(n):
            items = n * cols
            rounds = -(-items // sms)
            return fast and items >= 6 * sms and items >= 0.95 * rounds * sms

        def t_c(n):
            return n * px / rate * (1.0 if stack_ok(n) else 1.06) + (0.0 if stack_ok(n) else 2e-5)

        def finish(ch):
            hd = cd = dd = 0.0
            C, D = [], []
            for i, n in enumerate(ch):
                hs = hd if i < 2 else max(hd, C[i - 2])
                hd = hs + n * t_h
                cs = max(hd, cd, D[i - 2] if i >= 2 else 0.0)
                cd = cs + t_c(n)
                C.append(cd)
                dd = max(cd, dd) + n * t_d
                D.append(dd)
            return dd

        best = (finish([B]), [B])
        r = max(0.1, min(0.9, t_d / max(t_c(1), 1e-12)))
        for head in range(0, min(4, B // 8) + 1):
            for tail in range(1, max(1, B // 16) + 1):
                rest, c = [], tail
                while head + sum(rest) + c < B:
                    rest.insert(0, c)
                    c = max(c + 1, int(round(c / r)))
                big = B - head - sum(rest)
                for cand in range(big, max(0, big - 12), -1):  # prefer a stack-eligible big chunk
                    ch = ([head] if head else []) + [cand] + rest
                    if cand < big:
                        ch[len(ch) - len(rest)] += big - cand if rest else 0
                        if not rest:
                            ch.append(big - cand)
                    ch = [n for n in ch if n > 0]
                    t = finish(ch)
                    if t < best[0] - 1e-9:
                        best = (t, ch)
                    if stack_ok(cand):
                        break
        return best[1]

    def _forward_host(self, plan, x: torch.Tensor, dev: torch.device, closure: bool, row0: int, nrows: int):
        """CPU in / CPU out (the reference calling convention, inference.py:25-32).
        Sub-batches flow through three streams so the PCIe copies of one
        sub-batch overlap the forward of another; results land in pinned
        host memory.  Streams and device staging buffers are cached per device."""
        B, _, H, W = x.shape
        K = self.out_bands
        x_pin = x.contiguous()
        if not x_pin.is_pinned():
            x_pin = x_pin.pin_memory()
        out = torch.empty((B, K, nrows, W), dtype=torch.float32, pin_memory=True)
        cout = torch.empty((B, 1, nrows, W), dtype=torch.float32, pin_memory=True) if closure else None
        idx = dev.index
        nb = self._host_row_bands(B, H, W, row0, nrows, closure)
        if nb > 1:
            sizes = [B]
        elif isinstance(self.host_chunks, (list, tuple)):
            w = [float(v) for v in self.host_chunks]
            cuts = [0] + [round(B * sum(w[:i + 1]) / sum(w)) for i in range(len(w))]
            sizes = [cuts[i + 1] - cuts[i] for i in range(len(w)) if cuts[i + 1] > cuts[i]]
        elif self.host_chunks:
            n = max(1, min(int(self.host_chunks), B))
            sizes = [B * (i + 1) // n - B * i // n for i in range(n)]
        else:
            skey = (B, H, W, nrows, closure)
            cache = self.__dict__.setdefault("_sched_cache", {})
            if skey not in cache:
                sms = torch.cuda.get_device_properties(idx).multi_processor_count
                cache[skey] = self._host_schedule(B, H, W, nrows, closure, sms)
            sizes = cache[skey]
        # sub-batch forwards report their status at the final plan.sync (one
        # synchronisation instead of one per sub-batch)
        if nb > 1:
            def run(plan, x_pin, out, cout, sizes, dev, closure, row0, nrows):
                return self._pipeline_rows(plan, x_pin, out, cout, dev, closure, nb)
        else:
            run = self._single if len(sizes) == 1 else self._pipeline
        if self._options.get("check", 1) == 1:
            plan.set_option("check", 2)
            try:
                return run(plan, x_pin, out, cout, sizes, dev, closure, row0, nrows)
            finally:
                plan.set_option("check", 1)
        return run(plan, x_pin, out, cout, sizes, dev, closure, row0, nrows)

    # single large image from the host: number of row bands of the band pipeline
    # (None = automatic, 0 / 1 = off)
    host_row_bands = None

    def _host_row_bands(self, B: int, H: int, W: int, row0: int, nrows: int, closure: bool) -> int:
        """Row bands for one large host image (config 3's shape): the D2H of a
        1024 x 1024 result (24 MB, 0.45 ms) is half of its forward, and a batch
        of one has no other sub-batch to hide it behind.  Two (four for >= 6 MP)
        bands with a `depth`-row halo (recomputed) flow through the
        same three streams as sub-batches do."""
        if B != 1 or row0 != 0 or nrows != H or self.unshuffle != 1:
            return 1
        if self.host_row_bands is not None:
            return max(1, min(int(self.host_row_bands), H))
        out_bytes = 4 * (self.out_bands + (1 if closure else 0)) * H * W
        if out_bytes <= (16 << 20) or H < 512:
            return 1
        # few, large bands: every band pays a forward's fixed costs (measured:
        # 1024^2 1.50 ms whole, 1.43 in 2 bands, 1.53 in 4; 2048^2 5.60 / 4.89 /
        # 4.97; one 2160 x 3840 frame 9.48 in 2, 9.25 in 4, 10.3 in 8)
        return 4 if H * W >= (6 << 20) else 2

    def _pipeline_rows(self, plan, x_pin, out, cout, dev, closure, nbands):
        """One image as `nbands` row bands: band i's input rows (with halo) go
        H2D while band i-1 computes and band i-2's result goes D2H.  Each band
        is the forward of the halo-extended slice with a valid-row window
        (shard.row_bands), bitwise equal to the rows of the whole-image
        forward for in-range inputs (the per-image power-of-two input scale is
        chosen per band for inputs outside [2^-6, 64])."""
        from .shard import row_bands

        _, _, H, W = x_pin.shape
        K = self.out_bands
        bands = row_bands(H, nbands, self.depth)
        hmax = max(b.src1 - b.src0 for b in bands)
        rmax = max(b.rows for b in bands)
        idx = dev.index
        with torch.cuda.device(dev):
            comp = torch.cuda.current_stream(dev)
            pipes = self.__dict__.setdefault("_row_pipes", {})
            pk = (hmax, rmax, K, W, closure)
            pipe = pipes.get(idx)
            if pipe is None or pipe["key"] != pk:
                old = pipe
                pipe = {"key": pk,
                        "h2d": old["h2d"] if old else torch.cuda.Stream(dev),
                        "d2h": old["d2h"] if old else torch.cuda.Stream(dev),
                        "xbuf": [torch.empty((hmax, W), device=dev) for _ in range(2)],
                        "bbuf": [torch.empty((K, rmax, W), device=dev) for _ in range(2)],
                        "cbuf": [torch.empty((rmax, W), device=dev) if closure else None for _ in range(2)],
                        "events": []}
                pipes[idx] = pipe
            h2d, d2h = pipe["h2d"], pipe["d2h"]
            evs = pipe["events"]
            while len(evs) < 4 + 2 * len(bands):
                evs.append(torch.cuda.Event())
            x_free, b_free = evs[0:2], evs[2:4]
            for ev in x_free + b_free:
                ev.record(comp)
            for i, b in enumerate(bands):
                j, hb = i % 2, b.src1 - b.src0
                xb = pipe["xbuf"][j].view(-1)[: hb * W].view(hb, W)
                ob = pipe["bbuf"][j].view(-1)[: K * b.rows * W].view(K, b.rows, W)
                cb = pipe["cbuf"][j].view(-1)[: b.rows * W].view(b.rows, W) if closure else None
                h2d.wait_event(x_free[j])
                with torch.cuda.stream(h2d):
                    xb.copy_(x_pin[0, 0, b.src0:b.src1], non_blocking=True)
                landed = evs[4 + 2 * i]
                landed.record(h2d)
                comp.wait_event(landed)
                comp.wait_event(b_free[j])
                plan.forward(xb.data_ptr(), ob.data_ptr(), cb.data_ptr() if closure else 0, 1, hb, W,
                             b.valid_row0, b.rows, comp.cuda_stream)
                done = evs[5 + 2 * i]
                done.record(comp)
                x_free[j].record(comp)
                d2h.wait_event(done)
                with torch.cuda.stream(d2h):
                    for k in range(K):  # contiguous row blocks of each band plane
                        out[0, k, b.out0:b.out1].copy_(ob[k], non_blocking=True)
                    if closure:
                        cout[0, 0, b.out0:b.out1].copy_(cb, non_blocking=True)
                b_free[j].record(d2h)
            d2h.synchronize()
            plan.sync(comp.cuda_stream)
        return out, cout

    def _single(self, plan, x_pin, out, cout, sizes, dev, closure, row0, nrows):
        """One sub-batch (batch 1, the reference's predict_bands pattern): H2D,
        forward and D2H in order on the current stream with cached device
        buffers, one synchronisation - no copy streams or events to order."""
        B, _, H, W = x_pin.shape
        K = self.out_bands
        with torch.cuda.device(dev):
            comp = torch.cuda.current_stream(dev)
            bufs = self.__dict__.setdefault("_single_bufs", {})
            bkey = (dev.index, B, H, W, nrows, closure)
            if bkey not in bufs:
                bufs.clear()  # one shape at a time (the host pipeline caches likewise)
                bufs[bkey] = (torch.empty((B, 1, H, W), device=dev), torch.empty((B, K, nrows, W), device=dev),
                              torch.empty((B, 1, nrows, W), device=dev) if closure else None)
            xd, bd, cd = bufs[bkey]
            # (the input is copied: kernels reading the pinned image over PCIe measured
            # slower, 0.305 vs 0.261 ms per batch-1 call - conv0's taps and the head's closure re-read it)
            xd.copy_(x_pin, non_blocking=True)
            if out.numel() * 4 <= self.zero_copy_out_bytes:
                # small results: the head's epilogue stores go straight to the pinned
                # (device-mapped) result over PCIe, no D2H copy behind the forward
                plan.forward(xd.data_ptr(), out.data_ptr(), cout.data_ptr() if closure else 0, B, H, W, row0, nrows,
                             comp.cuda_stream)
            else:
                plan.forward(xd.data_ptr(), bd.data_ptr(), cd.data_ptr() if closure else 0, B, H, W, row0, nrows,
                             comp.cuda_stream)
                out.copy_(bd, non_blocking=True)
                if closure:
                    cout.copy_(cd, non_blocking=True)
            plan.sync(comp.cuda_stream)  # synchronises the stream; raises a failed forward
        return out, cout

    def _pipeline(self, plan, x_pin, out, cout, sizes, dev, closure, row0, nrows):
        B, _, H, W = x_pin.shape
        K = self.out_bands
        idx = dev.index
        bounds, s0 = [], 0
        for n in sizes:
            bounds.append((s0, s0 + n))
            s0 += n
        per = max(sizes)
        with torch.cuda.device(dev):
            comp = torch.cuda.current_stream(dev)
            pipes = self.__dict__.setdefault("_host_pipes", {})
            pk = (per, K, nrows, H, W, closure)
            pipe = pipes.get(idx)
            if pipe is None or pipe["key"] != pk:
                old = pipe
                pipe = {"key": pk,
                        "h2d": old["h2d"] if old else torch.cuda.Stream(dev),
                        "d2h": old["d2h"] if old else torch.cuda.Stream(dev),
                        "xbuf": [torch.empty((per, 1, H, W), device=dev) for _ in range(2)],
                        "bbuf": [torch.empty((per, K, nrows, W), device=dev) for _ in range(2)],
                        "cbuf": [torch.empty((per, 1, nrows, W), device=dev) if closure else None
                                 for _ in range(2)]}
                pipes[idx] = pipe
            h2d, d2h = pipe["h2d"], pipe["d2h"]
            xbuf, bbuf, cbuf = pipe["xbuf"], pipe["bbuf"], pipe["cbuf"]
            # events are reused across calls (every call ends synchronized)
            evs = pipe.setdefault("events", [])
            need = 4 + 2 * len(bounds)
            while len(evs) < need:
                evs.append(torch.cuda.Event())
            x_free, b_free = evs[0:2], evs[2:4]
            for ev in x_free + b_free:
                ev.record(comp)
            for i, (s, e) in enumerate(bounds):
                j, nb = i % 2, e - s
                h2d.wait_event(x_free[j])
                with torch.cuda.stream(h2d):
                    xbuf[j][:nb].copy_(x_pin[s:e], non_blocking=True)
                landed = evs[4 + 2 * i]
                landed.record(h2d)
                comp.wait_event(landed)
                comp.wait_event(b_free[j])
                plan.forward(xbuf[j].data_ptr(), bbuf[j].data_ptr(), cbuf[j].data_ptr() if closure else 0,
                             nb, H, W, row0, nrows, comp.cuda_stream)
                done = evs[5 + 2 * i]
                done.record(comp)
                x_free[j].record(comp)
                d2h.wait_event(done)
                with torch.cuda.stream(d2h):
                    out[s:e].copy_(bbuf[j][:nb], non_blocking=True)
                    if closure:
                        cout[s:e].copy_(cbuf[j][:nb], non_blocking=True)
                b_free[j].record(d2h)
            d2h.synchronize()
            plan.sync(comp.cuda_stream)  # raises a deferred failure of any sub-batch
        return out, cout

    def last_used_stack(self, device: int | None = None) -> bool:
        """Whether the last forward on that device ran the layer-stack kernel."""
        idx = torch.cuda.current_device() if device is None else device
        return self._plans[idx][0].last_used_stack() if idx in self._plans else False

    def last_launch_count(self, device: int | None = None) -> int:
        idx = torch.cuda.current_device() if device is None else device
        return self._plans[idx][0].last_launch_count() if idx in self._plans else 0


def receptive_field(depth: int = 17, kernel: int = 3) -> int:
    return depth * (kernel - 1) + 1
