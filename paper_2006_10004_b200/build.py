"""Build libtvsb200.so (the C-ABI + sm_100a kernels) in-tree with nvcc.

    python -m paper_2006_10004_b200.build        # or __graft_entry__.build()

The .so lands next to this file so it travels with the repo snapshot to the
GPU box (it is git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libtvsb200.so"
# diagnostics build (--trace): the layer-stack row timeline compiled in
# (conv_tc.cu TVS_STACK_TRACE); tools/stack_trace.py loads it via TVS_LIB
TRACE_LIB = PKG / "libtvsb200_trace.so"
SOURCES = ["tvs_api.cu", "conv_tc.cu", "conv0_tc.cu", "conv_edge.cu", "metrics.cu", "tvflow.cu", "train.cu", "wgrad_tc.cu", "loss.cu"]
HEADERS = ["common.cuh", "sm100.cuh", "host_util.h"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xptxas", "-v", "--expt-relaxed-constexpr",
         "-Xcompiler", "-fPIC,-O2", "-shared"]
# cuBLAS: the training step's wgrad GEMMs (train.cu); rpath so the .so finds it outside torch too
LIBS = ["-lcublas", "-Xlinker", "-rpath,/usr/local/cuda/lib64"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [PKG.parent / "include" / "tvs_b200.h", Path(__file__)]
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> Path:
    lib = TRACE_LIB if trace else LIB
    if not force and not _stale(lib):
        return lib
    tmp = lib.with_suffix(".so.tmp")
    extra = ["-DTVS_STACK_TRACE"] if trace else []
    cmd = [nvcc(), *ARCH, *FLAGS, *extra, "-o", str(tmp), *[str(CSRC / s) for s in SOURCES], *LIBS]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = PKG / "build.log"
    log.write_text(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-6000:])
        raise RuntimeError(f"nvcc failed ({res.returncode}); see {log}")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, trace="--trace" in sys.argv))
