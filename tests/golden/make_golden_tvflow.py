"""Golden fixtures for the ground-truth producer, made by the REFERENCE.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_tvflow.py

Imports ``spectv`` from /root/reference/pkg/src and runs its own
ModelDrivenDecomposer.analyze (pipeline.py:105-145) on small seeded images;
the per-step prox iteration counts come from its rof_prox (solver.py:323-372)
called in analyze's order with its warm duals.  Writes golden_tvflow.npz.

Cases: name -> (image, dt, n_steps, schedule or None, solver kwargs), plus
gt_planes / gt_manifest: a dataset written by the reference's
generate_ground_truth (dataset.py:131-200) from gt_images.make_images.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

from spectv.pipeline import DecompositionConfig, ModelDrivenDecomposer  # noqa: E402  (reference)
from spectv.solver import SolverConfig, rof_prox  # noqa: E402  (reference)


def cases():
    rng = np.random.default_rng(21)
    yy, xx = np.mgrid[0:32, 0:32]
    disk = ((yy - 15.5) ** 2 + (xx - 12.0) ** 2 < 81).astype(np.float64) * 2.0 - 0.5
    disk += 0.05 * rng.standard_normal(disk.shape)
    ramp = np.add.outer(np.linspace(-1, 1, 12), np.linspace(0, 0.5, 12))
    return {
        "gauss": (rng.standard_normal((24, 20)), 0.2, 100, None, {}),
        "disk": (disk, 0.2, 100, None, {}),
        "const": (np.full((8, 8), 0.7), 0.2, 12, (2, 5, 11), {}),
        "row": (rng.standard_normal((1, 17)), 0.2, 12, (2, 5, 11), {}),
        "col": (rng.standard_normal((13, 1)), 0.2, 12, (2, 5, 11), {}),
        "cap": (rng.standard_normal((16, 16)), 0.2, 10, (3, 9), {"max_iters": 15}),
        "noaccel": (ramp + 0.3 * rng.standard_normal((12, 12)), 0.2, 8, (2, 4, 7), {"pd_accel": False,
                                                                                   "max_iters": 300}),
        "wide": (rng.standard_normal((9, 300)), 0.25, 6, (2, 5), {}),
        "tol": (rng.standard_normal((20, 28)), 0.1, 16, (3, 7, 15), {"gap_tol": 1e-9, "max_iters": 4000}),
    }


def main():
    out = {}
    for name, (f, dt, n, sched, solver) in cases().items():
        cfg = DecompositionConfig(dt=dt, n_steps=n, schedule=tuple(sched) if sched else (),
                                  solver=SolverConfig(**solver))
        r = ModelDrivenDecomposer(cfg).analyze(f)
        its, dual, u = [], None, f
        for _ in range(n):
            p = rof_prox(u, dt, cfg.solver, warm_dual=dual)
            its.append(p.iterations)
            dual, u = p.dual_field, p.v
        out[f"{name}_f"] = f
        out[f"{name}_meta"] = np.array([dt, n], dtype=np.float64)
        out[f"{name}_schedule"] = np.array(cfg.schedule, dtype=np.int64)
        out[f"{name}_solver"] = np.array([cfg.solver.max_iters, cfg.solver.gap_tol, float(cfg.solver.pd_accel)])
        out[f"{name}_bands"] = r.bands.bands
        out[f"{name}_spectrum"] = r.spectrum.values
        out[f"{name}_residual"] = r.residual
        out[f"{name}_warnings"] = np.array(r.warnings, dtype=np.int64)
        out[f"{name}_iterations"] = np.array(its, dtype=np.int64)
        print(name, f.shape, "warnings", r.warnings, "iters", its[:6], "...")
    # a ground-truth dataset made by the reference generator (dataset.py:131-200)
    import json
    import tempfile

    from gt_images import GT_CFG, GT_KW, make_images
    from spectv.dataset import generate_ground_truth
    from spectv.tensorfile import read_tensor

    with tempfile.TemporaryDirectory() as td:
        paths = make_images(Path(td) / "img")
        cfg = DecompositionConfig(**GT_CFG)
        man = generate_ground_truth(paths, Path(td) / "ds", config=cfg, **GT_KW)
        out["gt_planes"] = np.stack([read_tensor(Path(td) / "ds" / e["tensor_file"]) for e in man["entries"]])
        for e in man["entries"]:
            e["source"] = Path(e["source"]).name
        out["gt_manifest"] = np.array(json.dumps(man, sort_keys=True))
    np.savez_compressed(HERE / "golden_tvflow.npz", **out)
    print("wrote", HERE / "golden_tvflow.npz")


if __name__ == "__main__":
    main()
