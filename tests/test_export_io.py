"""Exchange formats of the export path, no GPU needed:
BTF container and manifest contracts of the reference trainer
(pkg/trainer/tests/test_tensorfile.py, test_manifest.py), plus byte-identity
with a file written by the reference writer (tests/golden)."""
import json

import numpy as np
import pytest

from paper_2006_10004_b200.export import load_dataset, read_tensor, write_tensor


def test_round_trip(tmp_path):
    arr = np.random.default_rng(0).standard_normal((4, 9, 13)).astype("<f4")
    write_tensor(tmp_path / "t.btf", arr)
    back = read_tensor(tmp_path / "t.btf")
    assert back.shape == (4, 9, 13) and back.dtype == np.dtype("<f4")
    np.testing.assert_array_equal(back, arr)


def test_bytes_identical_to_reference_writer(golden, tmp_path):
    write_tensor(tmp_path / "t.btf", golden["btf_array"])
    assert (tmp_path / "t.btf").read_bytes() == golden["btf_bytes"].tobytes()
    raw = golden["btf_bytes"].tobytes()
    assert raw[:8] == b"BANDTNSR" and raw[8:28] == np.array([1, 1, 3, 5, 7], "<u4").tobytes()


def test_write_casts_float64(tmp_path):
    arr = np.linspace(0, 1, 30).reshape(2, 3, 5)
    write_tensor(tmp_path / "t.btf", arr)
    np.testing.assert_allclose(read_tensor(tmp_path / "t.btf"), arr, atol=1e-7)


def test_rejects(tmp_path):
    with pytest.raises(ValueError):
        write_tensor(tmp_path / "t.btf", np.zeros((4, 4)))
    p = tmp_path / "t.btf"
    write_tensor(p, np.zeros((1, 2, 2), dtype="<f4"))
    raw = bytearray(p.read_bytes())
    raw[:4] = b"XXXX"
    p.write_bytes(bytes(raw))
    with pytest.raises(ValueError, match="magic"):
        read_tensor(p)
    write_tensor(p, np.zeros((2, 4, 4), dtype="<f4"))
    p.write_bytes(p.read_bytes()[:-8])
    with pytest.raises(ValueError):
        read_tensor(p)
    p.write_bytes(b"BANDTNSR")
    with pytest.raises(ValueError):
        read_tensor(p)


def test_load_dataset(dataset_dir):
    index = load_dataset(dataset_dir)
    assert len(index) == 8 and index.n_bands == 6 and index.crop_size == 16
    img, bands = index.load_entry(0)
    assert img.shape == (16, 16) and bands.shape == (6, 16, 16)
    np.testing.assert_allclose(bands.sum(axis=0), img, atol=1e-5)
    assert len(index.content_hash()) == 64


def test_manifest_errors(dataset_dir):
    m = json.loads((dataset_dir / "manifest.json").read_text())
    bad = dict(m, plane_layout=["band1", "input"])
    (dataset_dir / "manifest.json").write_text(json.dumps(bad))
    with pytest.raises(ValueError):
        load_dataset(dataset_dir)
    (dataset_dir / "manifest.json").write_text(json.dumps(dict(m, entries=[])))
    with pytest.raises(ValueError):
        load_dataset(dataset_dir)
    (dataset_dir / "manifest.json").write_text(json.dumps(m))
    (dataset_dir / "entry_00003.btf").unlink()
    with pytest.raises(FileNotFoundError):
        load_dataset(dataset_dir)
