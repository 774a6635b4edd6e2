"""Emulate candidate fast-mode operand formats on CPU against the fp32 oracle.

Usage: python tools/emulate_precision.py [--images N]
Prints worst-band relative L2 (per image, per band) and closure error for
each scheme, on config-1/2/3 images (SURVEY.md §8(d) generator) with the
seeded seed-0 Kaiming model.  Used to pick the tcgen05 operand kind.
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np
import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import band_rel_l2, build_seeded_state, oracle_from_state  # noqa: E402
from paper_2006_10004_b200.workloads import CONFIGS, make_image  # noqa: E402


def fold(state, depth):
    """BN fold in fp64: returns list of (W, b) for the depth convs."""
    layers = []
    w0 = state["body.0.weight"].double(); b0 = state["body.0.bias"].double()
    layers.append((w0, b0))
    for j in range(depth - 2):
        ci = 2 + 3 * j
        w = state[f"body.{ci}.weight"].double()
        g = state[f"body.{ci+1}.weight"].double(); be = state[f"body.{ci+1}.bias"].double()
        mu = state[f"body.{ci+1}.running_mean"].double(); var = state[f"body.{ci+1}.running_var"].double()
        s = g / torch.sqrt(var + 1e-5)
        layers.append((w * s[:, None, None, None], be - mu * s))
    hi = 3 * depth - 4
    layers.append((state[f"body.{hi}.weight"].double(), state[f"body.{hi}.bias"].double()))
    return layers


def q(t, fmt):
    if fmt == "f32":
        return t.float().double()
    if fmt == "f16":
        return t.half().double()
    if fmt == "bf16":
        return t.bfloat16().double()
    raise ValueError(fmt)


def dc_round_fp16(w):
    """Rounding with per-(co,ci) tap-sum compensation: flip the rounding
    direction of the taps with the largest rounding residual until the sum of
    residuals over the 9 taps is as close to zero as possible."""
    w = w.double()
    lo = w.half().double()
    # the other candidate: next representable in the other direction
    up = torch.where(lo < w, torch.nextafter(lo.half().float(), torch.tensor(float("inf"))).double(), lo)
    dn = torch.where(lo > w, torch.nextafter(lo.half().float(), torch.tensor(float("-inf"))).double(), lo)
    # nextafter on float32 is not fp16-next; compute fp16 neighbours properly
    h = w.half()
    bits = h.view(torch.int16).to(torch.int32)
    def from_bits(b):
        return b.to(torch.int16).view(torch.float16).double()
    sign = torch.sign(h.double())
    nb_up = torch.where(h.double() >= 0, bits + 1, bits - 1)
    nb_dn = torch.where(h.double() > 0, bits - 1, bits + 1)
    cand_up = from_bits(nb_up)
    cand_dn = from_bits(nb_dn)
    rn = h.double()
    alt = torch.where(rn < w, cand_up, cand_dn)  # the other side of w
    alt = torch.where(rn == w, rn, alt)
    co, ci = w.shape[:2]
    res = (rn - w).reshape(co, ci, 9)
    alt_res = (alt - w).reshape(co, ci, 9)
    out = rn.reshape(co, ci, 9).clone()
    s = res.sum(-1)
    # greedy: for each (co,ci), flip taps in order of |cost| while it reduces |sum|
    delta = alt_res - res  # change of sum if flipped
    order = torch.argsort((alt_res.abs() - res.abs()), dim=-1)
    for t in range(9):
        idx = order[..., t]
        d = torch.gather(delta, -1, idx[..., None])[..., 0]
        better = (s + d).abs() < s.abs()
        s = torch.where(better, s + d, s)
        cur = torch.gather(out, -1, idx[..., None])[..., 0]
        newv = torch.gather(alt.reshape(co, ci, 9), -1, idx[..., None])[..., 0]
        out.scatter_(-1, idx[..., None], torch.where(better, newv, cur)[..., None])
    return out.reshape(w.shape)


def run(layers, x, wfmt, afmt, exact_ends=True, wq_fn=None, corr=None):
    a = torch.from_numpy(x).double()
    n = len(layers)
    for i, (w, b) in enumerate(layers):
        last = i == n - 1
        first = i == 0
        if exact_ends and (first or last):
            wq = w.float().double(); aq = q(a, afmt) if (last and afmt != "f32") else a.float().double()
        else:
            wq = wq_fn(w) if wq_fn else q(w, wfmt)
            aq = q(a, afmt)
        y = F.conv2d(aq.float(), wq.float(), None, padding=1).double()
        if corr is not None and not (exact_ends and (first or last)):
            y = y + corr(aq, w, wq)
        y = y + b[None, :, None, None]
        if not last:
            y = torch.relu(y)
            if afmt != "f32":
                y = q(y, afmt)
        a = y
    return a.numpy()


def e4m3_corr(aq, w, wq):
    lo = (w - wq) * 2.0**14
    lo8 = lo.float().to(torch.float8_e4m3fn).float()
    a8 = aq.float().to(torch.float8_e4m3fn).float()
    return F.conv2d(a8, lo8, None, padding=1).double() / 2.0**14


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=2)
    args = ap.parse_args()
    torch.set_num_threads(8)
    state = build_seeded_state()
    model = oracle_from_state(state)
    layers = fold(state, 17)
    cases = [("cfg1", CONFIGS[1], 0)] + [("cfg2", CONFIGS[2], i) for i in range(args.images)]
    cases += [("cfg3", CONFIGS[3], 0)]
    schemes = {
        "bf16": dict(wfmt="bf16", afmt="bf16"),
        "f16": dict(wfmt="f16", afmt="f16"),
        "f16 dc-round": dict(wfmt="f16", afmt="f16", wq_fn=dc_round_fp16),
        "f16 + e4m3 corr": dict(wfmt="f16", afmt="f16", corr=e4m3_corr),
        "f16 W, f32 act": dict(wfmt="f16", afmt="f32"),
    }
    for name, spec, idx in cases:
        img = make_image(spec, idx)[None, None]
        with torch.no_grad():
            ref = model(torch.from_numpy(img)).numpy()
        cref = img[:, 0] - ref.sum(1)
        line = [f"{name}[{idx}]"]
        for sname, kw in schemes.items():
            out = run(layers, img, **kw)
            e = band_rel_l2(out, ref).max()
            c = band_rel_l2((img[:, 0] - out.sum(1))[:, None], cref[:, None]).max()
            line.append(f"{sname}: {e:.3e}/{c:.2e}")
        print("  ".join(line), flush=True)


if __name__ == "__main__":
    main()
