"""Export path on B200: dataset / probe prediction in
the producer's exchange formats, batched through the drop-in TVSpecNet.

Mirrors /root/reference/pkg/trainer/src/tvsurrogate:

* ``read_tensor`` / ``write_tensor``  — tensorfile.py:33-59: the BTF container
  (8-byte magic "BANDTNSR", u32 version=1, u32 dtype=1 (f32), u32 n, h, w,
  then a little-endian float32 C-order payload), same validation errors.
* ``load_dataset`` / ``DatasetIndex`` — manifest.py:27-83.
* ``export_for_eval``   — inference.py:45-56: every dataset entry ->
  ``[input, bands..., closure]`` under the same file name.
* ``export_for_probes`` — inference.py:59-77: every probe variant, plus
  probes.json copied next to the predictions.
* ``load_checkpoint``   — training.py:163-172 (builds the drop-in instead).

What changes is the execution: the reference runs one entry at a time on the
CPU (``predict_bands`` with batch 1).  Here entries of equal shape are stacked
into batches, the forward runs on the GPU with the closure plane computed in
the head kernel's epilogue (``forward_planes(closure=True)``), and file reads
/ writes overlap the GPU work on a small thread pool.  The input plane is
written back bit-for-bit; bands and closure are float32 as in
``complete_planes`` (the reference forms the closure in float64 and rounds
once, the fused epilogue in float32: the two differ by at most a few ulp).
Pass ``closure="host"`` to build the closure exactly like the reference.
"""

from __future__ import annotations

import hashlib
import json
import shutil
import struct
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

__all__ = [
    "MAGIC",
    "read_tensor",
    "write_tensor",
    "DatasetIndex",
    "load_dataset",
    "export_for_eval",
    "export_for_probes",
    "load_checkpoint",
]

MAGIC = b"BANDTNSR"
_VERSION = 1
_DTYPE_F32 = 1
_HEADER = struct.Struct("<8sIIIII")
MANIFEST_NAME = "manifest.json"


# ------------------------------------------------------------------ BTF ----
def read_tensor(path) -> np.ndarray:
    """Read a 3-D float32 BTF tensor, validating the header (tensorfile.py:33-48)."""
    raw = Path(path).read_bytes()
    if len(raw) < _HEADER.size:
        raise ValueError(f"{path}: truncated header ({len(raw)} bytes)")
    magic, version, dtype, n, h, w = _HEADER.unpack_from(raw)
    if magic != MAGIC:
        raise ValueError(f"{path}: bad magic {magic!r}")
    if version != _VERSION:
        raise ValueError(f"{path}: unsupported version {version}")
    if dtype != _DTYPE_F32:
        raise ValueError(f"{path}: unsupported dtype code {dtype}")
    expected = _HEADER.size + 4 * n * h * w
    if len(raw) != expected:
        raise ValueError(f"{path}: payload size {len(raw)} != expected {expected}")
    return np.frombuffer(raw, dtype="<f4", offset=_HEADER.size).reshape(n, h, w)


def write_tensor(path, planes: np.ndarray) -> None:
    """Write a 3-D array as a float32 BTF tensor (tensorfile.py:51-59)."""
    planes = np.ascontiguousarray(planes, dtype="<f4")
    if planes.ndim != 3:
        raise ValueError(f"tensor must be 3-D, got shape {planes.shape}")
    n, h, w = planes.shape
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(MAGIC, _VERSION, _DTYPE_F32, n, h, w))
        fh.write(planes.tobytes())


# ------------------------------------------------------------- manifest ----
@dataclass(frozen=True)
class DatasetIndex:
    """Resolved view of a dataset directory (manifest.py:27-50)."""

    root: Path
    manifest: dict
    tensor_files: tuple[str, ...]
    n_bands: int
    crop_size: int

    def load_entry(self, i: int) -> tuple[np.ndarray, np.ndarray]:
        planes = read_tensor(self.root / self.tensor_files[i])
        return planes[0], planes[1:]

    def __len__(self) -> int:
        return len(self.tensor_files)

    def content_hash(self) -> str:
        digest = hashlib.sha256()
        digest.update(json.dumps(self.manifest, sort_keys=True).encode())
        for name in self.tensor_files:
            digest.update((self.root / name).read_bytes())
        return digest.hexdigest()


def load_dataset(dataset_dir) -> DatasetIndex:
    """manifest.py:53-83: validate manifest.json and resolve the entries."""
    root = Path(dataset_dir)
    path = root / MANIFEST_NAME
    if not path.exists():
        raise FileNotFoundError(f"no {MANIFEST_NAME} in {root}")
    manifest = json.loads(path.read_text())
    layout = manifest.get("plane_layout")
    if not layout or layout[0] != "input":
        raise ValueError(f"unsupported plane layout: {layout}")
    n_bands = len(layout) - 1
    if n_bands < 1:
        raise ValueError("manifest declares no band planes")
    entries = manifest.get("entries", [])
    if not entries:
        raise ValueError("manifest has no entries")
    files = tuple(e["tensor_file"] for e in entries)
    for name in files:
        if not (root / name).exists():
            raise FileNotFoundError(f"missing tensor file {name}")
    crop = int(manifest.get("preprocessing", {}).get("crop_size", 0))
    if crop <= 0:
        crop = read_tensor(root / files[0]).shape[-1]
    return DatasetIndex(root=root, manifest=manifest, tensor_files=files, n_bands=n_bands, crop_size=crop)


# --------------------------------------------------------------- export ----
def _predict_planes_batch(model, images: list[np.ndarray], closure: str) -> np.ndarray:
    """(n, h, w) input planes -> (n, 2+K, h, w) float32 [input, bands, closure]."""
    x = torch.from_numpy(np.stack([np.asarray(im, dtype=np.float32) for im in images])[:, None])
    if closure == "fused":
        # the head epilogue writes the closure plane and checks the band-sum
        # identity of every entry (tvs_forward_checked); 1e-5 is the tolerance
        # of the reference's closure test (test_inference.py:31-38)
        bands, clos, rel = model.forward_planes(x.pin_memory().cuda(non_blocking=True), check_reconstruction=True)
        worst = float(rel.max())
        if not worst <= 1e-5:
            raise ArithmeticError(f"band-sum reconstruction check failed: relative residual {worst:.3e}")
        bands, clos = bands.cpu().numpy(), clos.cpu().numpy()
    else:  # reference semantics: closure in float64 from the float64 image (inference.py:41)
        bands = model.forward_planes(x)[0].numpy()
        img64 = np.stack([np.asarray(im, dtype=np.float64) for im in images])[:, None]
        clos = (img64 - bands.sum(axis=1, keepdims=True)).astype(np.float32)
    return np.concatenate([x.numpy(), bands, clos], axis=1).astype("<f4", copy=False)


def _batched_export(model, jobs, batch_images: int, closure: str, io_threads: int) -> int:
    """jobs: list of (src_path, dst_path, plane_index).  Works through the jobs
    in bounded windows (a few batches of files at a time, so host memory does
    not grow with the dataset), groups equal shapes inside a window, and
    overlaps the next window's reads and this window's writes with the GPU
    forward."""
    if closure not in ("fused", "host"):
        raise ValueError("closure must be 'fused' or 'host'")
    window = max(1, batch_images) * 4

    def read_plane(job):  # copy the plane out so the rest of the file buffer is freed
        return np.array(read_tensor(job[0])[job[2]], copy=True)

    with ThreadPoolExecutor(max(1, io_threads)) as pool:
        writes = []
        nxt = [pool.submit(read_plane, j) for j in jobs[0:window]]
        for w0 in range(0, len(jobs), window):
            planes = [f.result() for f in nxt]
            nxt = [pool.submit(read_plane, j) for j in jobs[w0 + window:w0 + 2 * window]]
            by_shape: dict[tuple, list[int]] = {}
            for i, p in enumerate(planes):
                by_shape.setdefault(p.shape, []).append(i)
            for idx in by_shape.values():
                for s in range(0, len(idx), batch_images):
                    chunk = idx[s : s + batch_images]
                    out = _predict_planes_batch(model, [planes[i] for i in chunk], closure)
                    for k, i in enumerate(chunk):
                        writes.append(pool.submit(write_tensor, jobs[w0 + i][1], out[k]))
            del planes
            pending = []
            for w in writes:  # surface finished writes' errors, keep the rest
                if w.done():
                    w.result()
                else:
                    pending.append(w)
            writes = pending
        for w in writes:
            w.result()
    return len(jobs)


def export_for_eval(model, gt_dir, out_dir, batch_images: int = 64, closure: str = "fused",
                    io_threads: int = 8) -> int:
    """inference.py:45-56: predict every dataset entry, same-named tensors in out_dir."""
    gt_dir, out_dir = Path(gt_dir), Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    index = load_dataset(gt_dir)
    jobs = [(gt_dir / name, out_dir / name, 0) for name in index.tensor_files]
    return _batched_export(model, jobs, batch_images, closure, io_threads)


def export_for_probes(model, probes_dir, out_dir, batch_images: int = 64, closure: str = "fused",
                      io_threads: int = 8) -> int:
    """inference.py:59-77: predict every probe variant; copy probes.json."""
    probes_dir, out_dir = Path(probes_dir), Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    probes = json.loads((probes_dir / "probes.json").read_text())
    suffixes = ("",) + tuple("__" + v for v in probes["variants"])
    jobs = [(probes_dir / f"{stem}{sfx}.btf", out_dir / f"{stem}{sfx}.btf", 0)
            for stem in probes["ids"] for sfx in suffixes]
    n = _batched_export(model, jobs, batch_images, closure, io_threads)
    shutil.copy(probes_dir / "probes.json", out_dir / "probes.json")
    return n


def load_checkpoint(path, precision: str = "fast"):
    """training.py:163-172 with the B200 drop-in: torch.load -> TVSpecNet(**arch)
    -> strict load_state_dict -> eval()."""
    from .model import TVSpecNet

    payload = torch.load(path, map_location="cpu", weights_only=False)
    arch = payload["arch"]
    model = TVSpecNet(depth=arch["depth"], channels=arch["channels"], out_bands=arch["out_bands"],
                      precision=precision)
    model.load_state_dict(payload["state_dict"])
    model.eval()
    return model, payload
