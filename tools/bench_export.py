"""Export-path throughput: `export_for_eval` on a
synthetic dataset directory (N entries of size^2, 7 planes each, as the
producer writes them) through the B200 drop-in, vs the reference flow
(per-entry CPU forward + complete_planes + write, inference.py:45-56) timed on
a bounded subset.  Prints one JSON line.

    python tools/bench_export.py [--entries 256] [--size 256]
"""
import argparse, json, os, shutil, sys, tempfile, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tvspecnet_oracle import build_seeded_state, complete_planes, oracle_from_state  # noqa
from paper_2006_10004_b200 import TVSpecNet  # noqa
from paper_2006_10004_b200.export import export_for_eval, write_tensor, read_tensor  # noqa
from paper_2006_10004_b200.workloads import CONFIGS, make_image  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--entries", type=int, default=256)
ap.add_argument("--size", type=int, default=256)
ap.add_argument("--ref-seconds", type=float, default=10.0)
a = ap.parse_args()
root = Path(tempfile.mkdtemp(prefix="tvs_export_"))
ds, out = root / "ds", root / "pred"
ds.mkdir()
spec = CONFIGS[2]
entries = []
for i in range(a.entries):
    img = make_image(spec, i % spec.batch, a.size, a.size)
    planes = np.concatenate([img[None], np.repeat(img[None] / 6, 6, axis=0)])
    name = f"entry_{i:05d}.btf"
    write_tensor(ds / name, planes)
    entries.append({"tensor_file": name})
(ds / "manifest.json").write_text(json.dumps({"plane_layout": ["input"] + [f"band{k}" for k in range(1, 7)],
                                              "preprocessing": {"crop_size": a.size}, "entries": entries}))
state = build_seeded_state()
m = TVSpecNet().eval(); m.load_state_dict(state)
export_for_eval(m, ds, out)  # warm-up (plans, pinned buffers, page cache)
torch.cuda.synchronize()
t0 = time.perf_counter()
n = export_for_eval(m, ds, out)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
mp = n * a.size * a.size / 1e6
# reference flow on a bounded subset, all host threads
torch.set_num_threads(os.cpu_count() or 1)
oracle = oracle_from_state(state)
t1 = time.perf_counter(); k = 0
with torch.no_grad():
    while k < n and time.perf_counter() - t1 < a.ref_seconds:
        name = entries[k]["tensor_file"]
        image = read_tensor(ds / name)[0].astype(np.float64)
        bands = oracle(torch.from_numpy(image.astype(np.float32))[None, None])[0].numpy()
        write_tensor(root / "ref.btf", complete_planes(image, bands))
        k += 1
rdt = time.perf_counter() - t1
print(json.dumps({"metric": "export_for_eval megapixels/sec (read BTF -> forward -> write BTF)",
                  "value": round(mp / dt, 2), "unit": "MP/s", "entries": n, "size": a.size,
                  "seconds": round(dt, 3), "reference_flow": {"value": round(k * a.size * a.size / 1e6 / rdt, 4),
                  "unit": "MP/s", "entries_timed": k, "cores": os.cpu_count()}}))
shutil.rmtree(root)
