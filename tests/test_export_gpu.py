"""Export path on the GPU vs the reference flow (oracle forward + complete_planes),
inference.py:45-77 and the reference tests test_inference.py:41-84."""
import json

import numpy as np
import pytest
import torch

from oracle.tvspecnet_oracle import band_rel_l2, build_seeded_state, complete_planes, oracle_from_state
from paper_2006_10004_b200 import TVSpecNet
from paper_2006_10004_b200.cli import main as cli_main
from paper_2006_10004_b200.export import export_for_eval, export_for_probes, read_tensor, write_tensor

pytestmark = pytest.mark.gpu
TOL = {"fast": 1e-2, "fp32": 1e-5}


def _model(prec):
    m = TVSpecNet(precision=prec).eval()
    m.load_state_dict(build_seeded_state())
    return m


@pytest.mark.parametrize("prec", ["fast", "fp32"])
@pytest.mark.parametrize("closure", ["fused", "host"])
def test_export_for_eval_matches_reference_flow(dataset_dir, tmp_path, prec, closure):
    oracle = oracle_from_state(build_seeded_state())
    out = tmp_path / "pred"
    n = export_for_eval(_model(prec), dataset_dir, out, batch_images=3, closure=closure)
    assert n == 8
    for i in range(8):
        name = f"entry_{i:05d}.btf"
        planes = read_tensor(out / name)
        gt = read_tensor(dataset_dir / name)
        assert planes.shape == (7, 16, 16)
        np.testing.assert_array_equal(planes[0], gt[0])  # input passed through bitwise
        img = gt[0].astype(np.float64)
        with torch.no_grad():
            ref_bands = oracle(torch.from_numpy(img.astype(np.float32))[None, None])[0].numpy()
        ref = complete_planes(img, ref_bands)
        assert band_rel_l2(planes[1:6], ref[1:6]).max() <= TOL[prec]
        np.testing.assert_allclose(planes[1:].sum(axis=0), planes[0], atol=1e-5)
        if closure == "host":  # reference closure semantics, exactly
            exp = (img[None] - planes[1:6].sum(axis=0, keepdims=True)).astype("<f4")
            np.testing.assert_array_equal(planes[6:7], exp)


def test_export_for_probes(tmp_path):
    probes = tmp_path / "probes"
    probes.mkdir()
    grid = np.random.default_rng(2).standard_normal((16, 24)).astype("<f4")
    variants = {"": grid, "__x2": 2.0 * grid, "__shift8_0": np.roll(grid, 8, axis=0), "__rot90": np.rot90(grid).copy()}
    for sfx, plane in variants.items():
        write_tensor(probes / f"probe_0000{sfx}.btf", plane[None])
    (probes / "probes.json").write_text(json.dumps({"ids": ["probe_0000"], "variants": ["x2", "shift8_0", "rot90"],
                                                    "shift": [8, 0], "rotation_deg": 90}))
    out = tmp_path / "pred"
    assert export_for_probes(_model("fast"), probes, out) == 4
    assert (out / "probes.json").exists()
    assert read_tensor(out / "probe_0000__rot90.btf").shape == (7, 24, 16)  # mixed shapes batch separately
    assert read_tensor(out / "probe_0000.btf").shape == (7, 16, 24)


def test_cli_predict_with_reference_checkpoint(dataset_dir, tmp_path):
    """A checkpoint in the reference schema (training.py:127-135) drives `predict`."""
    ck = tmp_path / "checkpoint.pt"
    torch.save({"arch": {"depth": 17, "channels": 64, "kernel": 3, "out_bands": 5, "batch_norm": True,
                         "receptive_field": 35},
                "state_dict": build_seeded_state(), "config": {}, "dataset_hash": "", "plane_layout": None,
                "torch_version": torch.__version__}, ck)
    out = tmp_path / "pred"
    assert cli_main(["predict", str(ck), str(dataset_dir), "--out", str(out)]) == 0
    assert len(list(out.glob("*.btf"))) == 8
