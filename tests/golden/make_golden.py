"""Generate the golden parity fixtures by executing the REFERENCE module.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``tvsurrogate`` from /root/reference/pkg/trainer/src (the
reference's own TVSpecNet, model.py:29-56, and complete_planes,
inference.py:34-42), builds the seeded weights with the recipe of
``oracle.build_seeded_state`` applied to the REFERENCE class, and stores
inputs, outputs and hashes in ``golden.npz``.  The GPU box has no
/root/reference: tests read only the committed .npz.

Fixtures (all float32):
  * state_sha256_<arch>      sha256 of the seeded state_dict bytes (key order)
  * small_x / small_y        seed-0 default model, (2,1,16,20) N(0,1) input
  * nonsq_x / nonsq_y        (1,1,32,40) N(0,1)       (test_model.py:8-13 shape)
  * tiny_x / tiny_y          (3,1,1,1), (1,1,2,3) edge sizes
  * cfg1_x / cfg1_y          config 1 input (256^2, generator seed 1) -> bands
  * cfg1_planes              complete_planes(cfg1 image, bands) (7,256,256)
  * wide_x / wide_y          (26, 128, 5) model, seed 0, (1,1,24,24)
  * d3_x / d3_y              depth-3 model, seed 0, (1,1,9,11)
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np
import torch
from torch import nn

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, "/root/reference/pkg/trainer/src")

from tvsurrogate.inference import complete_planes  # noqa: E402  (reference)
from tvsurrogate.model import TVSpecNet  # noqa: E402  (reference)

from paper_2006_10004_b200.workloads import CONFIGS, make_image  # noqa: E402


def seeded_reference(depth=17, channels=64, out_bands=5, seed=0):
    torch.manual_seed(seed)
    m = TVSpecNet(depth, channels, out_bands)
    for mod in m.modules():
        if isinstance(mod, nn.Conv2d):
            nn.init.kaiming_normal_(mod.weight, mode="fan_in", nonlinearity="relu")
    return m.eval()


def state_sha(m) -> str:
    h = hashlib.sha256()
    for k, v in m.state_dict().items():
        h.update(k.encode())
        h.update(v.detach().cpu().contiguous().numpy().tobytes())
    return h.hexdigest()


@torch.no_grad()
def main():
    torch.set_num_threads(8)
    out = {}
    m = seeded_reference()
    out["state_sha256_default"] = np.array(state_sha(m))
    rng = np.random.default_rng(0)
    cases = {
        "small": rng.standard_normal((2, 1, 16, 20)).astype(np.float32),
        "nonsq": rng.standard_normal((1, 1, 32, 40)).astype(np.float32),
        "tiny": rng.standard_normal((3, 1, 1, 1)).astype(np.float32),
        "tiny2": rng.standard_normal((1, 1, 2, 3)).astype(np.float32),
        "cfg1": make_image(CONFIGS[1], 0)[None, None],
    }
    for name, x in cases.items():
        out[f"{name}_x"] = x
        out[f"{name}_y"] = m(torch.from_numpy(x)).numpy()
    img = cases["cfg1"][0, 0].astype(np.float64)
    out["cfg1_planes"] = complete_planes(img, out["cfg1_y"][0])

    wide = seeded_reference(26, 128, 5)
    out["state_sha256_wide"] = np.array(state_sha(wide))
    x = rng.standard_normal((1, 1, 24, 24)).astype(np.float32)
    out["wide_x"], out["wide_y"] = x, wide(torch.from_numpy(x)).numpy()

    d3 = seeded_reference(3, 64, 5)
    out["state_sha256_d3"] = np.array(state_sha(d3))
    x = rng.standard_normal((1, 1, 9, 11)).astype(np.float32)
    out["d3_x"], out["d3_y"] = x, d3(torch.from_numpy(x)).numpy()

    # a BTF file written by the reference writer (tensorfile.py:51-59), byte for byte
    import tempfile

    from tvsurrogate.tensorfile import write_tensor as ref_write

    with tempfile.TemporaryDirectory() as td:
        arr = np.random.default_rng(11).standard_normal((3, 5, 7))
        ref_write(Path(td) / "t.btf", arr)
        out["btf_array"] = arr
        out["btf_bytes"] = np.frombuffer((Path(td) / "t.btf").read_bytes(), dtype=np.uint8)

    # band scoring cases from the REFERENCE producer metrics (spectv/metrics.py:211-237)
    sys.path.insert(0, "/root/reference/pkg/src")
    from spectv.metrics import band_metrics as ref_band_metrics

    mrng = np.random.default_rng(5)
    gt = mrng.standard_normal((5, 40, 57)).astype(np.float32)
    cases = {
        "noisy": (gt, (gt + 0.1 * mrng.standard_normal(gt.shape)).astype(np.float32)),
        "exact": (gt, gt.copy()),
        "zero_pred": (gt, np.zeros_like(gt)),
        "const_gt": (np.full((2, 24, 24), 0.5, np.float32), mrng.random((2, 24, 24)).astype(np.float32)),
        "square_aligned": (mrng.random((3, 64, 64)).astype(np.float32), mrng.random((3, 64, 64)).astype(np.float32)),
    }
    for name, (g, p) in cases.items():
        rep = ref_band_metrics(g, p)
        out[f"metrics_{name}_gt"], out[f"metrics_{name}_pred"] = g, p
        out[f"metrics_{name}_per_band"] = np.array(rep.per_band, dtype=np.float64)
        out[f"metrics_{name}_max_i"] = np.array(rep.max_i, dtype=np.float64)

    out["torch_version"] = np.array(torch.__version__)
    np.savez_compressed(HERE / "golden.npz", **out)
    print("wrote", HERE / "golden.npz", sorted(out))


if __name__ == "__main__":
    main()
