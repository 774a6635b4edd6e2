"""Emulate the fp32-accurate split-operand tcgen05 layer bit-for-bit on the CPU
and compare accumulation schemes against the reference fp32 outputs.

tcgen05.mma kind::f16 with fp32 accumulators (measured by
tools/probe_mma_rounding.cu on B200): each MMA adds its K=16 products to the
accumulator exactly and truncates the result toward zero once.  With split
operands (a = a_hi + a_lo, w = w_hi + w_lo, all fp16) an output receives

    main : 3 dy x 3 dx x 4 K16 steps of a_hi*w_hi   (36 MMAs)
    corr : the same for a_lo*w_hi and a_hi*w_lo      (72 MMAs)

Schemes:
    one      all 108 MMAs into one accumulator (the first kernel: 3.4e-5 on B200)
    split2   main and corr in two accumulators, summed in fp32 by the epilogue
    dy3      main split into 3 accumulators by dy (+ corr), summed in the epilogue
    debias   split2 with the expected truncation loss of the main accumulator
             added back: 0.5 ulp(|partial sum|) per MMA, estimated from the
             final value

    python tools/emulate_split_accum.py [golden-case ...]
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

WS = 256.0  # weight scale of the split pack
DEBIAS = float(__import__("os").environ.get("DEBIAS", "0.72"))


def rz32(x):
    """Round float64 -> float32 toward zero."""
    r = x.astype(np.float32)
    over = np.abs(r.astype(np.float64)) > np.abs(x)
    r[over] = np.nextafter(r[over], np.float32(0))
    return r.astype(np.float64)


def split16(x):
    hi = x.astype(np.float16).astype(np.float64)
    lo = (x - hi).astype(np.float16).astype(np.float64)
    return hi, lo


def layer(a, w, scheme):
    """a: (H, W, 64) float32 activations (>= 0), w: (64co, 64ci, 3, 3) folded fp32
    weights -> pre-activation (H, W, 64) as the kernel would produce it."""
    H, W, C = a.shape
    ah, al = split16(a.astype(np.float64))
    wf = (w.astype(np.float32) * np.float32(WS)).astype(np.float64)
    wh, wl = split16(wf)
    pad = lambda t: np.pad(t, ((1, 1), (1, 1), (0, 0)))
    ahp, alp = pad(ah), pad(al)
    accs = {}

    def add(key, s):
        if scheme == "exact":  # fp64 accumulation, one fp32 rounding at the end: the floor
            accs[key] = s if key not in accs else accs[key] + s
            return
        accs[key] = rz32(s) if key not in accs else rz32(accs[key] + s)

    nmain = 0
    for dyi, dy in enumerate((-1, 0, 1)):        # input row order for an output row: q-1, q, q+1
        for p in range(3):
            for dx in (-1, 0, 1):
                for k in range(4):
                    cs = slice(16 * k, 16 * k + 16)
                    A = (ahp if p != 1 else alp)[1 + dy:1 + dy + H, 1 + dx:1 + dx + W, cs]
                    Wt = (wh if p != 2 else wl)[:, cs, dy + 1, dx + 1]  # (co, 16)
                    s = np.einsum("hwc,oc->hwo", A, Wt)
                    if scheme in ("one", "exact"):
                        add("m", s)
                    elif scheme in ("split2", "debias", "debias_lin"):
                        add("m" if p == 0 else "c", s)
                    elif scheme == "main2":  # main split by K half (channels 0-31 / 32-63) + corr
                        add(("m0" if k < 2 else "m1") if p == 0 else "c", s)
                    elif scheme == "main2dy":  # main split: dy=0 vs dy=+-1
                        add(("m0" if dy == 0 else "m1") if p == 0 else "c", s)
                    elif scheme == "dy3":
                        add(f"m{dyi}" if p == 0 else "c", s)
                    if p == 0:
                        nmain += 1
    if scheme in ("main2", "main2dy"):
        for key in ("m0", "m1"):
            accs[key] = (accs[key].astype(np.float32) *
                         np.float32(1.0 + 0.5 * 0.7213 * 2.0**-23 * (nmain / 4) * DEBIAS)).astype(np.float64)
    if scheme == "debias_lin":
        # expected loss for a linearly growing partial sum: 0.5 * sum_i ulp(|z| i / n)
        m = accs["m"]
        az = np.abs(m).astype(np.float64)
        loss = np.zeros_like(az)
        for i in range(1, nmain + 1):
            loss += np.spacing((az * i / nmain).astype(np.float32)).astype(np.float64)
        accs["m"] = (m + np.sign(m) * 0.5 * loss * DEBIAS).astype(np.float32).astype(np.float64)
    if scheme == "debias":
        m = accs["m"]
        # mean truncation loss per MMA ~ 0.5 ulp of the running sum; with the
        # partial sums growing ~linearly, sum_i ulp(acc_i) ~ n/2 ulp(final)
        # smooth form: E[ulp(x)/|x|] over a binade = 0.7213 * 2^-23
        accs["m"] = (m.astype(np.float32) * np.float32(1.0 + 0.5 * 0.7213 * 2.0**-23 * (nmain / 2) * DEBIAS)).astype(np.float64)
    tot = np.zeros_like(next(iter(accs.values())))
    for key in sorted(accs):
        tot = (tot.astype(np.float32) + accs[key].astype(np.float32)).astype(np.float64)
    return (tot / WS).astype(np.float32)


def forward(x, state, scheme):
    """x (H, W) float32 -> (K, H, W) bands with split layers emulated."""
    w0, b0 = state["body.0.weight"].numpy(), state["body.0.bias"].numpy()
    H, W = x.shape
    xp = np.pad(x.astype(np.float64), 1)
    a = np.zeros((H, W, w0.shape[0]))
    for ky in range(3):
        for kx in range(3):
            a += xp[ky:ky + H, kx:kx + W, None] * w0[:, 0, ky, kx][None, None, :].astype(np.float64)
    a = np.maximum(a + b0, 0).astype(np.float32)
    depth = 2 + sum(1 for k, v in state.items() if k.endswith(".weight") and v.ndim == 4) - 2
    for l in range(depth - 2):
        conv = state[f"body.{2 + 3 * l}.weight"].numpy()
        bn = f"body.{3 + 3 * l}"
        g, bta = state[f"{bn}.weight"].numpy(), state[f"{bn}.bias"].numpy()
        mu, var = state[f"{bn}.running_mean"].numpy(), state[f"{bn}.running_var"].numpy()
        s = (g / np.sqrt(var + 1e-5)).astype(np.float32)
        shift = (bta - mu * s).astype(np.float32)
        wf = conv * s[:, None, None, None]
        z = layer(a, wf, scheme)
        a = np.maximum(z + shift, 0).astype(np.float32)
    wh = state[f"body.{3 * depth - 4}.weight"].numpy().astype(np.float64)
    bh = state[f"body.{3 * depth - 4}.bias"].numpy().astype(np.float64)
    ap = np.pad(a.astype(np.float64), ((1, 1), (1, 1), (0, 0)))
    out = np.zeros((wh.shape[0], H, W))
    for ky in range(3):
        for kx in range(3):
            out += np.einsum("hwc,kc->khw", ap[ky:ky + H, kx:kx + W], wh[:, :, ky, kx])
    return (out + bh[:, None, None]).astype(np.float32)


def main():
    from oracle.tvspecnet_oracle import band_rel_l2, build_seeded_state

    g = dict(np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / "golden.npz"))
    state = build_seeded_state()
    cases = sys.argv[1:] or ["small"]
    if "crop" in cases:  # a 64x64 crop of config 1 (piecewise constant), reference = oracle fp32
        import torch

        from oracle.tvspecnet_oracle import oracle_from_state

        y0, x0, sz = (int(v) for v in __import__("os").environ.get("CROP", "96,96,64").split(","))
        xc = g["cfg1_x"][:, :, y0:y0 + sz, x0:x0 + sz].copy()
        m = oracle_from_state(state)
        with torch.no_grad():
            g["crop_x"], g["crop_y"] = xc, m(torch.from_numpy(xc)).numpy()
    for case in cases:
        x, ref = g[f"{case}_x"], g[f"{case}_y"]
        for scheme in __import__("os").environ.get("SCHEMES", "one,split2,dy3,debias").split(","):
            out = np.stack([forward(x[b, 0], state, scheme) for b in range(x.shape[0])])
            err = band_rel_l2(out, ref)
            print(f"{case:6s} {scheme:7s} worst band rel-L2 {err.max():.3e}  mean {err.mean():.3e}", flush=True)


if __name__ == "__main__":
    main()
