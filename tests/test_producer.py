"""CPU tests for the ground-truth producer row: the oracle restatement is
pinned bit-for-bit to the reference's own outputs (golden_tvflow.npz, made by
make_golden_tvflow.py from spectv), the host-side config mirrors validate
like the reference, and the C-ABI rejects invalid arguments before any
device work."""

import ctypes
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).parent / "golden" / "golden_tvflow.npz"
FAST = ["const", "row", "col", "cap", "noaccel", "wide", "gauss"]


@pytest.fixture(scope="module")
def golden_tv():
    return np.load(GOLD)


@pytest.mark.parametrize("name", FAST)
def test_oracle_bitwise_vs_reference(golden_tv, name):
    import oracle.tvflow_oracle as O

    g = golden_tv
    dt, n = g[f"{name}_meta"]
    mi, tol, acc = g[f"{name}_solver"]
    r = O.analyze(g[f"{name}_f"], dt=float(dt), n_steps=int(n), schedule=tuple(g[f"{name}_schedule"]),
                  max_iters=int(mi), gap_tol=float(tol), accel=bool(acc))
    assert np.array_equal(r["bands"], g[f"{name}_bands"])
    assert np.array_equal(r["spectrum"], g[f"{name}_spectrum"])
    assert np.array_equal(r["residual"], g[f"{name}_residual"])
    assert np.array_equal(r["iterations"], g[f"{name}_iterations"])
    assert r["warnings"] == [int(w) for w in g[f"{name}_warnings"]]


def test_golden_properties(golden_tv):
    """Reference outputs telescope to the input (transform.py:1-14)."""
    for name in ("gauss", "disk", "wide"):
        f = golden_tv[f"{name}_f"]
        assert np.abs(golden_tv[f"{name}_bands"].sum(0) - f).max() < 1e-10


def test_config_mirror():
    from paper_2006_10004_b200.producer import DecompositionConfig, SolverConfig, dyadic_schedule

    assert DecompositionConfig().schedule == (2, 4, 8, 16, 32, 99)
    assert dyadic_schedule(0.1, 200) == (4, 8, 16, 32, 64, 199)
    for bad in (dict(max_iters=0), dict(gap_tol=0.0), dict(pd_step_tau=1.0), dict(method="x")):
        with pytest.raises(ValueError):
            SolverConfig(**bad)
    with pytest.raises(ValueError):
        DecompositionConfig(n_steps=1)
    with pytest.raises(ValueError):
        DecompositionConfig(n_steps=10, schedule=(3, 2, 9))
    with pytest.raises(ValueError):
        DecompositionConfig(n_steps=10, schedule=(3, 8))
    d = DecompositionConfig(dt=0.1, n_steps=50, schedule=(3, 49))
    assert DecompositionConfig.from_dict(d.to_dict()) == d


def test_chambolle_rejected():
    from paper_2006_10004_b200.producer import DecompositionConfig, ModelDrivenDecomposer, SolverConfig

    with pytest.raises(ValueError):
        ModelDrivenDecomposer(DecompositionConfig(solver=SolverConfig(method="chambolle-projection")))


def test_abi_validation():
    """Argument checks run on the host before any launch (no GPU needed)."""
    from paper_2006_10004_b200 import _native

    lib = _native.load()
    assert lib.tvs_tvflow_workspace_bytes(3, 4, 5) == 3 * 6 * 4 * 5 * 8
    fake = ctypes.c_void_p(0x1000)
    sched = (ctypes.c_int * 3)(2, 5, 9)
    s = ctypes.cast(sched, ctypes.c_void_p)
    args = dict(N=0, H=4, W=4, dt=0.2, n=10, nb=3, mi=100, tol=1e-6, tau=0.3, sig=0.3, acc=1)

    def call(**kw):
        a = {**args, **kw}
        return lib.tvs_tvflow_analyze(fake, a["N"], a["H"], a["W"], a["dt"], a["n"], s, a["nb"], a["mi"], a["tol"],
                                      a["tau"], a["sig"], a["acc"], fake, fake, fake, fake, fake, None)

    assert call() == 0  # N = 0: validated no-op
    for bad in (dict(n=9), dict(dt=0.0), dict(W=2049), dict(mi=0), dict(tol=0.0), dict(tau=1.0), dict(nb=17),
                dict(H=0), dict(n=1)):
        assert call(**bad) == _native.TVS_E_INVALID, bad


def test_dataset_crops_match_reference(golden_tv, tmp_path):
    """Host half of generate_ground_truth (dataset.py:113-170): seeded crops,
    2x box-mean augmentation, dataset-global standardisation -> plane 0 of
    every entry and the manifest bookkeeping, bitwise vs the reference."""
    import json
    import sys

    sys.path.insert(0, str(GOLD.parent))
    from gt_images import GT_KW, make_images

    from paper_2006_10004_b200 import groundtruth as gt

    ref = json.loads(str(golden_tv["gt_manifest"]))
    paths = make_images(tmp_path / "img")
    cache = {}
    specs = gt.plan_crops([str(p) for p in paths], GT_KW["count"], GT_KW["crop_size"], GT_KW["seed"],
                          GT_KW["augment_fraction"], cache)
    stacked = np.stack([gt._cut(cache[s.source], s.crop_size, s.row, s.col, s.factor) for s in specs])
    mean, std = float(stacked.mean()), float(stacked.std())
    assert mean == ref["preprocessing"]["mean"] and std == ref["preprocessing"]["std"]
    grids = ((stacked - mean) / std).astype("<f4")
    assert np.array_equal(grids, golden_tv["gt_planes"][:, 0])
    for s, e in zip(specs, ref["entries"]):
        m = s.manifest_entry(e["solver_warnings"])
        assert m["crop_offset"] == e["crop_offset"] and m["downsample_factor"] == e["downsample_factor"]
        assert m["crop_size"] == e["crop_size"] and m["seed_spawn"] == e["seed_spawn"]
    # preprocess() reproduces an entry's input plane (dataset.py:96-110)
    e0 = ref["entries"][1]
    one = gt.preprocess(paths[1], GT_KW["crop_size"], GT_KW["seed"], mean, std, index=1,
                        augment=e0["downsample_factor"] == 2)
    assert np.array_equal(one.astype("<f4"), golden_tv["gt_planes"][1, 0])
