"""GPU ground-truth producer: model-driven spectral TV decomposition
(SURVEY.md §8(f) row 3).

Mirrors /root/reference/pkg/src/spectv:
  * ``SolverConfig``          solver.py:54-90   (primal-dual method only)
  * ``DecompositionConfig``   pipeline.py:22-82 (dt, n_steps, schedule, solver)
  * ``dyadic_schedule``       transform.py:186-207
  * ``ModelDrivenDecomposer`` pipeline.py:92-145: ``analyze`` -> bands +
    spectrum + residual + warnings, ``decompose`` -> bands, plus
    ``analyze_batch`` that decomposes a whole (N, H, W) stack in ONE kernel
    launch (one persistent CTA per image, csrc/tvflow.cu).

The flow runs on the GPU in fp64 with the reference's operation order
(libtvsb200 ``tvs_tvflow_analyze``); there is no host fallback.  Results
agree with the reference up to the reordering of reductions (sums inside
the gap certificate), see tests/test_producer_gpu.py for the tolerances.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native

__all__ = ["SolverConfig", "DecompositionConfig", "DecompositionResult", "BandSet", "SpectrumCurve",
           "ModelDrivenDecomposer", "dyadic_schedule"]

_GRAD_NORM_SQ = 8.0


@dataclass(frozen=True)
class SolverConfig:
    """solver.py:54-90 (validation identical; ``chambolle-projection`` is not
    provided on the GPU and is rejected by the decomposer)."""

    method: str = "primal-dual"
    max_iters: int = 2000
    gap_tol: float = 1e-6
    pd_step_tau: float = 1.0 / math.sqrt(_GRAD_NORM_SQ)
    pd_step_sigma: float = 1.0 / math.sqrt(_GRAD_NORM_SQ)
    projection_step: float = 0.125
    pd_accel: bool = True

    def __post_init__(self):
        if self.method not in ("chambolle-projection", "primal-dual"):
            raise ValueError(f"unknown solver method: {self.method!r}")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.gap_tol <= 0:
            raise ValueError("gap_tol must be positive")
        if self.pd_step_tau <= 0 or self.pd_step_sigma <= 0:
            raise ValueError("primal-dual steps must be positive")
        if self.pd_step_tau * self.pd_step_sigma * _GRAD_NORM_SQ > 1.0 + 1e-12:
            raise ValueError("pd_step_tau * pd_step_sigma * 8 must be <= 1")
        if not 0 < self.projection_step <= 0.125:
            raise ValueError("projection_step must lie in (0, 1/8]")


def dyadic_schedule(dt: float, n_steps: int, first_edge_time: float = 0.4, n_bands: int = 6):
    """transform.py:186-207: band end indices at first_edge_time * 2^k, last = n_steps-1."""
    if n_bands < 2:
        raise ValueError("need at least 2 bands")
    edges, t = [], first_edge_time
    for _ in range(n_bands - 1):
        edges.append(int(round(t / dt)))
        t *= 2.0
    edges.append(n_steps - 1)
    if edges[0] < 2:
        raise ValueError("first band edge falls below 2 fine steps; decrease dt")
    if edges[-2] >= n_steps - 1:
        raise ValueError("band edges exceed the time grid; increase n_steps or decrease edges")
    return tuple(edges)


def _check_schedule(schedule, n_responses: int):
    """transform.py:131-144."""
    schedule = tuple(int(e) for e in schedule)
    if len(schedule) < 1:
        raise ValueError("schedule must contain at least one band")
    prev = 0
    for e in schedule:
        if e <= prev:
            raise ValueError(f"schedule indices must be strictly increasing, got {schedule}")
        prev = e
    if schedule[-1] != n_responses:
        raise ValueError(f"schedule must cover fine indices 1..{n_responses}, last entry is {schedule[-1]}")
    return schedule


@dataclass(frozen=True)
class DecompositionConfig:
    """pipeline.py:22-82."""

    dt: float = 0.2
    n_steps: int = 100
    schedule: tuple = ()
    solver: SolverConfig = field(default_factory=SolverConfig)

    def __post_init__(self):
        if self.dt <= 0:
            raise ValueError("dt must be positive")
        if self.n_steps < 2:
            raise ValueError("n_steps must be >= 2")
        if not self.schedule:
            object.__setattr__(self, "schedule", dyadic_schedule(self.dt, self.n_steps))
        else:
            object.__setattr__(self, "schedule", _check_schedule(self.schedule, self.n_steps - 1))

    @property
    def edge_times(self):
        return tuple(e * self.dt for e in self.schedule)

    def to_dict(self) -> dict:
        s = self.solver
        return {"dt": self.dt, "n_steps": self.n_steps, "schedule": list(self.schedule),
                "solver": {"method": s.method, "max_iters": s.max_iters, "gap_tol": s.gap_tol,
                           "pd_step_tau": s.pd_step_tau, "pd_step_sigma": s.pd_step_sigma,
                           "projection_step": s.projection_step, "pd_accel": s.pd_accel}}

    @classmethod
    def from_dict(cls, d: dict) -> "DecompositionConfig":
        return cls(dt=d.get("dt", 0.2), n_steps=d.get("n_steps", 100), schedule=tuple(d.get("schedule", ())),
                   solver=SolverConfig(**d.get("solver", {})))


@dataclass(frozen=True)
class BandSet:
    """transform.py:71-90."""

    bands: np.ndarray
    schedule: tuple
    includes_residual: bool

    @property
    def n_bands(self) -> int:
        return self.bands.shape[0]

    def reconstruction(self) -> np.ndarray:
        return self.bands.sum(axis=0)


@dataclass(frozen=True)
class SpectrumCurve:
    """transform.py:56-68 (CSV writer with the reference's format)."""

    scales: np.ndarray
    values: np.ndarray

    def write_csv(self, path) -> None:
        import csv

        with open(path, "w", newline="") as fh:
            writer = csv.writer(fh)
            writer.writerow(["t", "S"])
            for t, s in zip(self.scales, self.values):
                writer.writerow([f"{t:.10g}", f"{s:.10g}"])


@dataclass
class DecompositionResult:
    """pipeline.py:85-89 plus the per-step prox iteration counts."""

    bands: BandSet
    spectrum: SpectrumCurve
    residual: np.ndarray
    warnings: list
    iterations: np.ndarray | None = None


@dataclass
class BatchResult:
    """Device-resident output of :meth:`ModelDrivenDecomposer.analyze_batch_device`."""

    bands: torch.Tensor       # (N, n_bands, H, W) fp64
    spectrum: torch.Tensor    # (N, n_steps-1) fp64
    residual: torch.Tensor    # (N, H, W) fp64
    iterations: torch.Tensor  # (N, n_steps) int32, -(k+1) = not certified after k iterations


class ModelDrivenDecomposer:
    """pipeline.py:92-145 on the GPU."""

    def __init__(self, config: DecompositionConfig | None = None, device=None):
        self.config = config or DecompositionConfig()
        if self.config.solver.method != "primal-dual":
            raise ValueError("the GPU decomposer implements the primal-dual solver only")
        self.device = torch.device(device) if device is not None else None

    @property
    def n_bands(self) -> int:
        return len(self.config.schedule)

    def schedule_times(self):
        return self.config.edge_times

    def _dev(self):
        if self.device is not None:
            return self.device
        if not torch.cuda.is_available():
            raise RuntimeError("ModelDrivenDecomposer needs a CUDA device (libtvsb200 tvs_tvflow_analyze)")
        return torch.device("cuda", torch.cuda.current_device())

    def analyze_batch_device(self, f: torch.Tensor) -> BatchResult:
        """(N, H, W) images (any float dtype, any device) -> device-resident results."""
        cfg, s = self.config, self.config.solver
        dev = self._dev()
        x = torch.as_tensor(f).to(dev, torch.float64).contiguous()
        if x.ndim != 3:
            raise ValueError(f"expected (N, H, W) images, got shape {tuple(x.shape)}")
        if not bool(torch.isfinite(x).all()):
            raise ValueError("image grid contains NaN or Inf samples")
        N, H, W = x.shape
        nb = len(cfg.schedule)
        lib = _native.load()
        ws = torch.empty(max(1, lib.tvs_tvflow_workspace_bytes(N, H, W)), dtype=torch.uint8, device=dev)
        bands = torch.empty((N, nb, H, W), dtype=torch.float64, device=dev)
        spec = torch.empty((N, cfg.n_steps - 1), dtype=torch.float64, device=dev)
        resid = torch.empty((N, H, W), dtype=torch.float64, device=dev)
        iters = torch.empty((N, cfg.n_steps), dtype=torch.int32, device=dev)
        sched = (ctypes.c_int * nb)(*cfg.schedule)
        with torch.cuda.device(dev):
            _native.check(lib.tvs_tvflow_analyze(
                x.data_ptr(), N, H, W, float(cfg.dt), int(cfg.n_steps), ctypes.cast(sched, ctypes.c_void_p), nb,
                int(s.max_iters), float(s.gap_tol), float(s.pd_step_tau), float(s.pd_step_sigma),
                1 if s.pd_accel else 0, ws.data_ptr(), bands.data_ptr(), spec.data_ptr(), resid.data_ptr(),
                iters.data_ptr(), torch.cuda.current_stream(dev).cuda_stream))
        return BatchResult(bands=bands, spectrum=spec, residual=resid, iterations=iters)

    def analyze_batch(self, f) -> list[DecompositionResult]:
        """(N, H, W) stack -> N DecompositionResults, one launch for the whole stack."""
        cfg = self.config
        r = self.analyze_batch_device(torch.as_tensor(np.asarray(f) if not torch.is_tensor(f) else f))
        bands, spec = r.bands.cpu().numpy(), r.spectrum.cpu().numpy()
        resid, iters = r.residual.cpu().numpy(), r.iterations.cpu().numpy()
        scales = cfg.dt * np.arange(1, cfg.n_steps)
        out = []
        for n in range(bands.shape[0]):
            warnings = [int(i) + 1 for i in np.nonzero(iters[n] < 0)[0]]
            its = np.where(iters[n] < 0, -iters[n] - 1, iters[n])
            out.append(DecompositionResult(
                bands=BandSet(bands=bands[n], schedule=cfg.schedule, includes_residual=True),
                spectrum=SpectrumCurve(scales=scales, values=spec[n]), residual=resid[n], warnings=warnings,
                iterations=its))
        return out

    def analyze(self, f) -> DecompositionResult:
        """pipeline.py:105-145 for one 2-D image."""
        a = np.asarray(f, dtype=np.float64)
        if a.ndim != 2:
            raise ValueError(f"image grid must be 2-D, got shape {a.shape}")
        return self.analyze_batch(a[None])[0]

    def decompose(self, f) -> BandSet:
        return self.analyze(f).bands
