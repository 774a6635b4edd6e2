"""Pin the CPU oracle (test infrastructure) against fixtures produced by the
REFERENCE module (tests/golden/make_golden.py) — SURVEY.md §8(c)."""
import hashlib

import numpy as np
import pytest
import torch

from oracle.tvspecnet_oracle import (
    ARCH_SPEC,
    TVSpecNetOracle,
    band_rel_l2,
    build_seeded_state,
    complete_planes,
    oracle_from_state,
    receptive_field,
)


def _sha(state):
    h = hashlib.sha256()
    for k, v in state.items():
        h.update(k.encode())
        h.update(v.detach().cpu().contiguous().numpy().tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("arch,key", [((17, 64, 5), "default"), ((26, 128, 5), "wide"), ((3, 64, 5), "d3")])
def test_seeded_state_matches_reference(golden, arch, key):
    assert _sha(build_seeded_state(*arch)) == str(golden[f"state_sha256_{key}"])


@pytest.mark.parametrize("case", ["small", "nonsq", "tiny", "tiny2", "cfg1"])
def test_oracle_matches_reference_outputs(golden, seeded_state, case):
    m = oracle_from_state(seeded_state)
    with torch.no_grad():
        y = m(torch.from_numpy(golden[f"{case}_x"])).numpy()
    ref = golden[f"{case}_y"]
    assert y.shape == ref.shape
    # same torch CPU ops: bitwise here; other CPUs may pick other oneDNN kernels
    np.testing.assert_allclose(y, ref, rtol=1e-5, atol=1e-6)
    assert band_rel_l2(y, ref).max() < 1e-6


def test_oracle_wide_and_shallow(golden):
    for arch, key in (((26, 128, 5), "wide"), ((3, 64, 5), "d3")):
        m = oracle_from_state(build_seeded_state(*arch), *arch)
        with torch.no_grad():
            y = m(torch.from_numpy(golden[f"{key}_x"])).numpy()
        assert band_rel_l2(y, golden[f"{key}_y"]).max() < 1e-6


def test_complete_planes_matches_reference(golden):
    img = golden["cfg1_x"][0, 0].astype(np.float64)
    planes = complete_planes(img, golden["cfg1_y"][0])
    np.testing.assert_array_equal(planes, golden["cfg1_planes"])
    np.testing.assert_allclose(planes[1:].sum(0), planes[0], atol=1e-5)


def test_oracle_contracts():
    assert receptive_field(17, 3) == 35 == ARCH_SPEC["receptive_field"]
    with pytest.raises(ValueError):
        TVSpecNetOracle(depth=2)
    with pytest.raises(ValueError):
        TVSpecNetOracle()(torch.zeros(2, 3, 16, 16))
    assert len(TVSpecNetOracle().state_dict()) == 94
