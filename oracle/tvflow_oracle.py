"""CPU oracle for the GPU ground-truth producer.

TEST INFRASTRUCTURE ONLY: imported by tests/ and bench tooling as the
checker; the product path (paper_2006_10004_b200.producer ->
libtvsb200 tvs_tvflow_analyze) never calls it.

A numpy restatement of the reference's model-driven decomposition:
  * ``rof_prox_pd``  /root/reference/pkg/src/spectv/solver.py:242-320 (accelerated
    primal-dual with certified relative gap every 10 iterations, adaptive
    restart at factor 0.98) wrapped as rof_prox :323-372 (flat-input
    shortcut, warm dual stored on the unit ball and rescaled by dt)
  * ``certified_pair`` solver.py:134-150, ``scale_floor`` :173-174
  * ``analyze``      pipeline.py:105-145 (phi_i = i*(u_{i+1}-2u_i+u_{i-1})/dt into
    dyadic bands, spectrum sum|phi_i|, residual u_N - N(u_N - u_{N-1}))
It additionally returns the iteration count of every prox (the reference's
analyze only exposes the non-converged step list).

Pinned against outputs of the reference itself: tests/golden/golden_tvflow.npz
(made by tests/golden/make_golden_tvflow.py importing spectv), checked in
tests/test_producer.py.
"""

from __future__ import annotations

import numpy as np

GAP_CHECK_EVERY = 10
RESTART_FACTOR = 0.98


def _div(px, py):
    """grid.py:64-91 (negative adjoint of the forward-difference gradient)."""
    h, w = px.shape
    d = np.zeros_like(px)
    if w > 1:
        d[:, 0] = px[:, 0]
        d[:, 1:-1] = px[:, 1:-1] - px[:, :-2]
        d[:, -1] = -px[:, -2]
    if h > 1:
        d[0, :] += py[0, :]
        d[1:-1, :] += py[1:-1, :]
        d[1:-1, :] -= py[:-2, :]
        d[-1, :] -= py[-2, :]
    return d


def _tv(v):
    """grid.py:94-101."""
    gx = np.zeros_like(v)
    gy = np.zeros_like(v)
    gx[:, :-1] = v[:, 1:] - v[:, :-1]
    gy[:-1, :] = v[1:, :] - v[:-1, :]
    return float(np.sqrt(gx * gx + gy * gy).sum())


def scale_floor(u):
    return 1e-12 * (1.0 + float(np.sum(u * u)))


def certified_pair(u, v, w, dt):
    primal = 0.5 * float(np.sum((u - v) ** 2)) + dt * _tv(v)
    uw = float(np.sum(u * w))
    ww = float(np.sum(w * w))
    c = 1.0 if ww == 0.0 else min(max(-uw / ww, 0.0), 1.0)
    return primal, -c * uw - 0.5 * c * c * ww, c


def rel_gap(primal, dual, floor):
    return (primal - dual) / max(abs(primal), abs(dual), floor)


def rof_prox_pd(u, dt, max_iters=2000, gap_tol=1e-6, tau0=1 / np.sqrt(8.0), sigma0=1 / np.sqrt(8.0), accel=True,
                warm=None):
    """-> (v, iterations, converged, unit-ball dual (qx, qy))."""
    mean = float(u.mean())
    flat_gap = 0.5 * float(np.sum((u - mean) ** 2))
    floor = scale_floor(u)
    if flat_gap <= gap_tol * floor:
        z = np.zeros_like(u)
        return np.full_like(u, mean), 0, True, (z, z.copy())
    h, w = u.shape
    qx = np.zeros_like(u) if warm is None else warm[0] * dt
    qy = np.zeros_like(u) if warm is None else warm[1] * dt
    v = u.copy()
    vbar = v.copy()
    tau, sigma, theta = tau0, sigma0, 1.0
    iters, prev = 0, np.inf
    while True:
        for _ in range(min(GAP_CHECK_EVERY, max_iters - iters)):
            gx = np.zeros_like(u)
            gy = np.zeros_like(u)
            gx[:, :-1] = (vbar[:, 1:] - vbar[:, :-1]) * sigma
            gy[:-1, :] = (vbar[1:, :] - vbar[:-1, :]) * sigma
            qx = qx + gx
            qy = qy + gy
            scale = np.maximum(np.hypot(qx, qy) / dt, 1.0)
            qx = qx / scale
            qy = qy / scale
            dq = np.empty_like(u)  # div(q) + u, boundary folding of solver.py:284-295
            if w > 1:
                dq[:, 0] = qx[:, 0] + u[:, 0]
                dq[:, 1:-1] = (qx[:, 1:-1] - qx[:, :-2]) + u[:, 1:-1]
                dq[:, -1] = u[:, -1] - qx[:, -2]
            else:
                dq[:, 0] = u[:, 0]
            if h > 1:
                dq[0, :] += qy[0, :]
                dq[1:-1, :] += qy[1:-1, :]
                dq[1:-1, :] -= qy[:-2, :]
                dq[-1, :] -= qy[-2, :]
            v_new = (dq * tau + v) / (1.0 + tau)
            if accel:
                theta = 1.0 / np.sqrt(1.0 + 2.0 * tau)
                tau *= theta
                sigma /= theta
            vbar = (v_new - v) * theta + v_new
            v = v_new
            iters += 1
        primal, dual, c = certified_pair(u, v, _div(qx, qy), dt)
        rel = rel_gap(primal, dual, floor)
        if rel <= gap_tol or iters >= max_iters:
            break
        if accel and rel > RESTART_FACTOR * prev:
            tau, sigma, theta = tau0, sigma0, 1.0
            vbar = v.copy()
        prev = rel
    return v.copy(), iters, rel <= gap_tol, (c * qx / dt, c * qy / dt)


def dyadic_schedule(dt, n_steps, first_edge_time=0.4, n_bands=6):
    """transform.py:186-207."""
    edges, t = [], first_edge_time
    for _ in range(n_bands - 1):
        edges.append(int(round(t / dt)))
        t *= 2.0
    edges.append(n_steps - 1)
    return tuple(edges)


def analyze(f, dt=0.2, n_steps=100, schedule=None, **solver):
    """pipeline.py:105-145 -> dict(bands, spectrum, residual, warnings, iterations)."""
    f = np.asarray(f, dtype=np.float64)
    schedule = tuple(schedule) if schedule else dyadic_schedule(dt, n_steps)
    bands = np.zeros((len(schedule),) + f.shape)
    spec = np.empty(n_steps - 1)
    iters = np.zeros(n_steps, dtype=np.int64)
    warnings = []
    u_prev = f
    u_curr, iters[0], ok, dual = rof_prox_pd(u_prev, dt, warm=None, **solver)
    if not ok:
        warnings.append(1)
    b = 0
    for i in range(1, n_steps):
        u_next, iters[i], ok, dual = rof_prox_pd(u_curr, dt, warm=dual, **solver)
        if not ok:
            warnings.append(i + 1)
        phi = float(i) * (u_next - 2.0 * u_curr + u_prev) / dt
        while i > schedule[b]:
            b += 1
        bands[b] += phi
        spec[i - 1] = np.abs(phi).sum()
        u_prev, u_curr = u_curr, u_next
    bands *= dt
    fr = u_curr - n_steps * (u_curr - u_prev)
    bands[-1] += fr
    return {"bands": bands, "spectrum": spec, "residual": fr, "warnings": warnings, "iterations": iters,
            "schedule": schedule}
