"""Batched Dormand-Prince field-line tracer (reference trace_fieldline,
src/postprocess.py:244-357).

Every line is a small state machine (a generator) that yields the points
where it needs E; the driver gathers the requests of all live lines into
ONE batched device evaluation per round (lockstep over lines), so the
device sees (#live lines)-point N-body launches instead of one launch per
stage per line.  The control logic -- stage points, error norm, accept /
reject, step control, surface-hit arming and snapping, termination order --
is the reference's, evaluated in the same floating-point order.
"""

from __future__ import annotations

import numpy as np

from . import _fp
from .postprocess import (
    LEFT_DOMAIN,
    MAX_LENGTH,
    SURFACE_HIT,
    WEAK_FIELD,
    FieldLine,
    TraceError,
    _DP_A,
    _DP_B4,
    _DP_B5,
    _surface_distance,
)


class _Coincident:
    """Marker result for an E request at a mesh vertex (ValueError)."""


def _line(x0, sign, p, geo, mesh):
    """Generator: yields a point, receives E (3,) or _Coincident."""
    center, half, diag, h_min, h_max, l_max = geo

    def tangent(e):
        mag = float(_fp.norm3_fused(e))
        if mag <= p.e_floor or mag == 0.0:
            return None, mag
        return sign * e / mag, mag

    x = np.asarray(x0, dtype=float)
    e = yield x
    if isinstance(e, _Coincident):
        raise ValueError("evaluation point coincides with a mesh vertex")
    t0, mag0 = tangent(e)
    if t0 is None:
        raise TraceError(
            f"|E| = {mag0:.3e} V/m at the start point is not above the weak-field floor {p.e_floor:.3e}"
        )
    points = [x.copy()]
    mags = [mag0]
    arcs = [0.0]
    term = MAX_LENGTH
    h = h_max
    s = 0.0
    k1 = t0
    armed = False
    while True:
        d_surf, local_r = _surface_distance(mesh, x)
        hit_tol = p.surface_tol_frac * local_r
        if d_surf > 2.0 * hit_tol:
            armed = True
        if armed and d_surf < hit_tol:
            term = SURFACE_HIT
            x_end = x + k1 * d_surf
            points[-1] = x_end
            arcs[-1] += d_surf
            e = yield x_end
            if not isinstance(e, _Coincident):
                mags[-1] = float(_fp.norm3_fused(e))
            break
        if s >= l_max:
            term = MAX_LENGTH
            break
        if np.any(np.abs(x - center) > half):
            term = LEFT_DOMAIN
            break
        h_cap = h_max if d_surf > 4.0 * h_max else max(h_min, 0.45 * d_surf)
        h = min(h, h_cap, l_max - s + h_min)
        ks = [k1]
        failed = False
        for stage in range(1, 7):
            acc = 0
            for a, k in zip(_DP_A[stage], ks):
                acc = acc + a * k
            xi = x + h * acc
            e = yield xi
            if isinstance(e, _Coincident):
                raise ValueError("evaluation point coincides with a mesh vertex")
            ti, _ = tangent(e)
            if ti is None:
                term = WEAK_FIELD
                failed = True
                break
            ks.append(ti)
        if failed:
            break
        K = np.array(ks)
        x5 = x + h * (_DP_B5 @ K)
        x4 = x + h * (_DP_B4 @ K)
        err = float(_fp.norm3_fused(x5 - x4))
        tol = p.rel_tol * max(1.0, float(_fp.norm3_fused(x5)) / diag) * diag
        if err <= tol or h <= h_min * 1.0000001:
            x = x5
            s += h
            e = yield x
            if isinstance(e, _Coincident):
                raise ValueError("evaluation point coincides with a mesh vertex")
            t_new, mag_new = tangent(e)
            if t_new is None:
                points.append(x.copy())
                mags.append(mag_new)
                arcs.append(s)
                term = WEAK_FIELD
                break
            k1 = t_new
            points.append(x.copy())
            mags.append(mag_new)
            arcs.append(s)
        factor = 0.9 * (tol / err) ** 0.2 if err > 0.0 else 2.0
        h = float(np.clip(h * np.clip(factor, 0.2, 2.0), h_min, h_max))
    return FieldLine(points=np.array(points), e_magnitudes=np.array(mags), arc_lengths=np.array(arcs),
                     termination=term)


def trace_batch(solution, mesh, starts, orientations, params, cfg, raise_weak=False):
    import torch

    from .device import device_mesh
    from .postprocess import _check_points, _sources, _u_device, field_points_device

    lo, hi = mesh.bounding_box()
    center = 0.5 * (lo + hi)
    half = 0.5 * (hi - lo) * params.bbox_factor
    diag = float(_fp.norm3_fused(hi - lo))
    geo = (center, half, diag, params.h_min_frac * diag, params.h_max_frac * diag, params.max_length_frac * diag)
    dm = device_mesh(mesh, cfg)
    u_dev, key = _u_device(solution, dm)
    src = _sources(dm, u_dev, key)

    starts = np.asarray(starts, dtype=float).reshape(-1, 3)
    gens = []
    pending = {}
    results = [None] * len(starts)
    for i, (x0, o) in enumerate(zip(starts, orientations)):
        g = _line(x0, 1.0 if o >= 0 else -1.0, params, geo, mesh)
        gens.append(g)
        pending[i] = next(g)
    while pending:
        idx = list(pending)
        X = np.array([pending[i] for i in idx])
        # coincidence check per request (reference raises inside eval_efield)
        bad = set()
        for j, i in enumerate(idx):
            try:
                _check_points(mesh, X[j:j + 1])
            except ValueError:
                bad.add(j)
        ok = [j for j in range(len(idx)) if j not in bad]
        E = np.zeros((len(idx), 3))
        if ok:
            Xd = torch.as_tensor(np.ascontiguousarray(X[ok]), device=dm.device)
            E[ok] = field_points_device(dm, u_dev, src, Xd, False).cpu().numpy()
        nxt = {}
        for j, i in enumerate(idx):
            val = _Coincident() if j in bad else E[j]
            try:
                nxt[i] = gens[i].send(val)
            except StopIteration as stop:
                results[i] = stop.value
            except TraceError:
                if raise_weak:
                    raise
                results[i] = None
        pending = nxt
    return results
