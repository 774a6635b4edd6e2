"""Ground-truth producer throughput.

GPU: ModelDrivenDecomposer.analyze_batch_device over N seeded standardized
images (default config: dt 0.2, 100 steps, dyadic bands, accelerated PDHG,
gap_tol 1e-6), one launch, CUDA-event timed.  CPU: the reference algorithm
(oracle restatement, bit-identical to spectv) on one image of the same size,
single process.  Prints one JSON line.

    python tools/bench_producer.py --images 148 --size 64
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=148)
    ap.add_argument("--size", type=int, default=64)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--cpu-images", type=int, default=1)
    ap.add_argument("--repeats", type=int, default=1)
    args = ap.parse_args()
    from paper_2006_10004_b200.producer import DecompositionConfig, ModelDrivenDecomposer

    rng = np.random.default_rng(0)
    f = rng.standard_normal((args.images, args.size, args.size))
    sched = () if args.steps == 100 else (max(1, args.steps // 4), args.steps - 1)
    cfg = DecompositionConfig(n_steps=args.steps, schedule=sched)
    dec = ModelDrivenDecomposer(cfg)
    x = torch.from_numpy(f).cuda()
    dec.analyze_batch_device(x[:1])  # load + warm
    torch.cuda.synchronize()
    times = []
    for _ in range(args.repeats):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = dec.analyze_batch_device(x)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    t = min(times)
    iters = out.iterations.abs().cpu().numpy().astype(np.int64)
    iters = np.where(out.iterations.cpu().numpy() < 0, iters - 1, iters)
    px = args.size * args.size
    res = {"images": args.images, "size": args.size, "n_steps": args.steps, "gpu_s": t,
           "gpu_images_per_s": args.images / t, "gpu_ms_per_image": 1e3 * t / args.images,
           "mean_prox_iters": float(iters.mean()), "pd_iter_px_per_s": float(iters.sum()) * px / t}
    if args.cpu_images > 0:
        import oracle.tvflow_oracle as O

        t0 = time.perf_counter()
        for n in range(args.cpu_images):
            O.analyze(f[n], dt=cfg.dt, n_steps=args.steps, schedule=cfg.schedule)
        tc = (time.perf_counter() - t0) / args.cpu_images
        res.update({"cpu_s_per_image": tc, "cpu_kind": "port (bit-identical to spectv)", "cpu_cores": 1,
                    "speedup_per_image_throughput": tc / (t / args.images)})
    print(json.dumps(res))


if __name__ == "__main__":
    main()
