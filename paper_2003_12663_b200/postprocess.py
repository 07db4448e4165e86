"""Field evaluation, surface field, seeds, field-line tracing, streamer check.

Public API of reference ``src/postprocess.py``.  Potentials and fields run
as device N-body sums over density-contracted panel sources (csrc/field.cu)
with the reference's pair classification; near-singular panels go through
the same deferred composite-rule kernel as the assembly (csrc/near.cu).
Batched entry points (``eval_efield_batch``, ``eval_potential_batch``,
``trace_fieldlines``) are the throughput API; the single-point functions
are thin wrappers with identical results.
"""

from __future__ import annotations

import os
import csv
from dataclasses import dataclass

import numpy as np

from . import _fp, _lib
from .mesh import SurfaceMesh
from .quadrature import QuadConfig

__all__ = [
    "IonizationModel",
    "FieldLine",
    "TraceParams",
    "TraceError",
    "eval_potential",
    "eval_efield",
    "eval_potential_batch",
    "eval_efield_batch",
    "trace_fieldline",
    "trace_fieldlines",
    "streamer_integral",
    "surface_field_magnitudes",
    "pick_start_points",
    "load_ionization_model",
    "write_fieldline_csv",
]

VERTEX_PROXIMITY = 1e-12
SURFACE_HIT = "SurfaceHit"
WEAK_FIELD = "WeakField"
MAX_LENGTH = "MaxLength"
LEFT_DOMAIN = "LeftDomain"
MAX_STEPS = "MaxSteps"


class TraceError(ValueError):
    """Field-line tracing could not start (weak field at the start point)."""


@dataclass(frozen=True)
class IonizationModel:
    """alpha_eff(|E|) table + streamer constant (src/postprocess.py:47-67)."""

    e_values: np.ndarray
    alpha_values: np.ndarray
    k_str: float

    def __post_init__(self):
        e = np.asarray(self.e_values, dtype=float)
        a = np.asarray(self.alpha_values, dtype=float)
        if e.ndim != 1 or e.shape != a.shape or len(e) == 0:
            raise ValueError("ionization table must be two equal 1-d columns")
        if np.any(np.diff(e) <= 0.0):
            raise ValueError("ionization table must be strictly increasing in |E|")
        object.__setattr__(self, "e_values", e)
        object.__setattr__(self, "alpha_values", a)

    def alpha(self, e_mag):
        return np.interp(e_mag, self.e_values, self.alpha_values)


@dataclass
class FieldLine:
    points: np.ndarray
    e_magnitudes: np.ndarray
    arc_lengths: np.ndarray
    termination: str

    def __post_init__(self):
        if not (len(self.points) == len(self.e_magnitudes) == len(self.arc_lengths)):
            raise ValueError("points, |E| samples and arc lengths must align")
        if np.any(np.diff(self.arc_lengths) <= 0.0):
            raise ValueError("arc lengths must increase strictly")

    @property
    def length(self) -> float:
        return float(self.arc_lengths[-1])


@dataclass(frozen=True)
class TraceParams:
    rel_tol: float = 1e-6
    h_min_frac: float = 1e-6
    h_max_frac: float = 0.05
    surface_tol_frac: float = 0.1
    e_floor: float = 0.0
    max_length_frac: float = 4.0
    bbox_factor: float = 1.5
    # extension (not in the reference): end a line after this many Runge-Kutta
    # steps (accepted + rejected) with termination "MaxSteps"; None = the
    # reference's unbounded loop (a line hugging a surface it never armed
    # against can crawl at h_min for millions of steps)
    max_steps: int | None = None


# ---------------------------------------------------------------------------
# device field evaluation
# ---------------------------------------------------------------------------


def _check_points(mesh: SurfaceMesh, X: np.ndarray):
    """Reference _check_point (src/postprocess.py:104-109) for a batch."""
    if len(X) <= 8:
        for x in X:
            d = _fp.norm3_axis(mesh.vertices - x[None, :])
            if d.min() < VERTEX_PROXIMITY:
                raise ValueError(f"evaluation point coincides with mesh vertex {int(d.argmin())}")
        return
    from scipy.spatial import cKDTree

    tree = mesh._device_cache.get("kdtree")
    if tree is None:
        tree = cKDTree(mesh.vertices)
        mesh._device_cache["kdtree"] = tree
    # bounded search: only candidates within 1e-9 matter (far queries are free)
    dist, idx = tree.query(X, k=1, distance_upper_bound=1e-9, workers=-1)
    bad = np.nonzero(np.isfinite(dist))[0]
    for i in bad:
        d = _fp.norm3_axis(mesh.vertices - X[i][None, :])
        if d.min() < VERTEX_PROXIMITY:
            raise ValueError(f"evaluation point coincides with mesh vertex {int(d.argmin())}")


def _sources(dm, u_dev, key):
    """Density-contracted panel sources, cached per (solution, device)."""
    import torch

    cache = dm.__dict__.setdefault("_src_cache", {})
    src = cache.get(key)
    if src is None:
        src = torch.empty((dm.nt, dm.nq, 4), dtype=torch.float64, device=dm.device)
        _lib.call("hvb_contract", _lib.ptr(dm.table), dm.nt, dm.nq, _lib.ptr(dm.tri_cols), _lib.ptr(u_dev),
                  _lib.ptr(src), _lib.stream_ptr(dm.device))
        cache.clear()
        cache[key] = src
    return src


def _u_device(solution, dm):
    """Device copy of solution.u plus a key that changes on EVERY upload (the
    contracted-source cache of ``_sources`` is keyed on it): the host array
    is compared by content, so an in-place edit of u re-uploads it and
    invalidates the sources."""
    import torch

    cache = dm.__dict__.setdefault("_u_cache", {})
    hit = cache.get("u")
    if hit is None or hit[2].shape != solution.u.shape or not np.array_equal(hit[2], solution.u):
        u = torch.as_tensor(np.ascontiguousarray(solution.u, dtype=np.float64), device=dm.device)
        serial = cache.get("serial", 0) + 1
        cache["serial"] = serial
        hit = (("u", serial), u, np.array(solution.u, copy=True))
        cache["u"] = hit
    return hit[1], hit[0]


PANELS_PER_SPLIT = int(os.environ.get("HVB_PANELS_PER_SPLIT", "256"))


def panel_split(nt: int) -> int:
    """Panel-range split of the N-body launch (grid.y): chunks of ~256
    panels.  A function of the mesh only, so every target's sum has the
    same order whatever the batch (results independent of batch size and
    GPU count), and small batches (the tracer's tail rounds) still spread
    over hundreds of CTAs."""
    return int(max(1, min(4096, -(-nt // PANELS_PER_SPLIT))))


TARGET_BATCH = 1 << 17  # targets per launch (bounds the split x m partial buffer)


def field_points_device(dm, u_dev, src, X_dev, potential: bool, own_col=None, coincide_flag=None):
    """(m, 3) field (or potential in column 0) at device points X_dev (m,3).
    ``coincide_flag`` (m,) int32: set to 1 for targets within
    VERTEX_PROXIMITY of a node of one of their near panels.  Targets are
    processed in launches of TARGET_BATCH (per-target results do not depend
    on the batching)."""
    import torch

    m = int(X_dev.shape[0])
    if m <= TARGET_BATCH:
        return _field_points(dm, u_dev, src, X_dev, potential, own_col, coincide_flag)
    out = torch.empty((m, 3), dtype=torch.float64, device=dm.device)
    near = 0
    for a in range(0, m, TARGET_BATCH):
        b = min(m, a + TARGET_BATCH)
        part = _field_points(dm, u_dev, src, X_dev[a:b], potential, None if own_col is None else own_col[a:b],
                             None if coincide_flag is None else coincide_flag[a:b])
        out[a:b] = part
        near += part.near_pairs
    out.near_pairs = near  # type: ignore[attr-defined]
    return out


def _field_points(dm, u_dev, src, X_dev, potential: bool, own_col=None, coincide_flag=None):
    import torch

    dev = dm.device
    s = _lib.stream_ptr(dev)
    m = int(X_dev.shape[0])
    out = torch.zeros((m, 3), dtype=torch.float64, device=dev)
    if m == 0:
        return out
    split = panel_split(dm.nt)
    part = torch.empty((split, m, 4), dtype=torch.float64, device=dev)
    cap = max(4096, 8 * m)
    while True:
        near = torch.empty((cap, 2), dtype=torch.int32, device=dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        _lib.call("hvb_field", _lib.ptr(src), _lib.ptr(dm.cls), _lib.ptr(dm.groups), _lib.ptr(dm.tri_cols), dm.nt,
                  dm.nq,
                  _lib.ptr(X_dev), _lib.ptr(own_col), m, split, int(potential), _lib.ptr(part), _lib.ptr(near),
                  _lib.ptr(cnt), cap, s)
        n_near = int(cnt.item())
        if n_near <= cap:
            break
        cap = n_near + 1024
    _lib.call("hvb_field_reduce", _lib.ptr(part), split, m, _lib.ptr(out), s)
    if n_near:
        from .assembly import _segments, _sort_pairs

        pairs = _sort_pairs(near[:n_near], dm.nt)
        pts = torch.zeros((m, 6), dtype=torch.float64, device=dev)
        pts[:, :3] = X_dev
        kind = torch.full((m,), 3 if potential else 2, dtype=torch.int32, device=dev)
        contrib = torch.empty((n_near, 9), dtype=torch.float64, device=dev)
        _lib.call("hvb_near_pairs", _lib.ptr(pairs), n_near, _lib.ptr(pts), _lib.ptr(kind), _lib.ptr(dm.nodes6),
                  _lib.ptr(dm.radii), _lib.ptr(dm.rule_near), len(dm.rule_near), _lib.ptr(dm.rule_graded),
                  len(dm.rule_graded), int(dm.cfg.bisect_depth), float(dm.cfg.bisect_trigger),
                  _lib.ptr(contrib), s)
        if coincide_flag is not None:
            _lib.call("hvb_near_coincide", _lib.ptr(pairs), n_near, _lib.ptr(X_dev), _lib.ptr(dm.nodes6),
                      VERTEX_PROXIMITY, _lib.ptr(coincide_flag), s)
        seg = _segments(pairs[:, 0])
        _lib.call("hvb_near_apply_points", _lib.ptr(seg), len(seg) - 1, _lib.ptr(pairs), _lib.ptr(contrib),
                  _lib.ptr(dm.tri_cols), _lib.ptr(u_dev), int(potential), _lib.ptr(out), s)
    out_n = n_near
    out.near_pairs = out_n  # type: ignore[attr-defined]
    return out


def _eval_batch(solution, mesh, X, cfg, potential):
    import torch

    from .device import device_mesh

    cfg = cfg or QuadConfig()
    X = np.ascontiguousarray(np.asarray(X, dtype=np.float64).reshape(-1, 3))
    if len(X) <= 1024:
        _check_points(mesh, X)
        checker = None
    else:
        # the coincidence check (host kd-tree, GIL released) runs beside the
        # device evaluation; a coincident point still raises, nothing is returned
        checker = _CheckThread(mesh, X)
    try:
        dm = device_mesh(mesh, cfg)
        u_dev, key = _u_device(solution, dm)
        src = _sources(dm, u_dev, key)
        X_dev = torch.as_tensor(X, device=dm.device)
        out = field_points_device(dm, u_dev, src, X_dev, potential)
        res = out.cpu().numpy()
    finally:
        if checker is not None:
            checker.result()  # a coincident point raises first
    return res


class _CheckThread:
    """_check_points on a worker thread; result() re-raises its error."""

    def __init__(self, mesh, X):
        import threading

        self._err = None
        self._t = threading.Thread(target=self._run, args=(mesh, X), daemon=True)
        self._t.start()

    def _run(self, mesh, X):
        try:
            _check_points(mesh, X)
        except BaseException as e:  # noqa: BLE001 - re-raised in result()
            self._err = e

    def result(self):
        self._t.join()
        if self._err is not None:
            raise self._err


def eval_potential_batch(solution, mesh: SurfaceMesh, X, cfg: QuadConfig | None = None) -> np.ndarray:
    """Single-layer potential at many points, (m,)."""
    return _eval_batch(solution, mesh, X, cfg, True)[:, 0].copy()


def eval_efield_batch(solution, mesh: SurfaceMesh, X, cfg: QuadConfig | None = None) -> np.ndarray:
    """Electric field at many points, (m, 3)."""
    return _eval_batch(solution, mesh, X, cfg, False)


def eval_potential(solution, mesh: SurfaceMesh, x, cfg: QuadConfig | None = None) -> float:
    """Reference src/postprocess.py:112-121."""
    return float(eval_potential_batch(solution, mesh, np.asarray(x, dtype=float)[None], cfg)[0])


def eval_efield(solution, mesh: SurfaceMesh, x, cfg: QuadConfig | None = None) -> np.ndarray:
    """Reference src/postprocess.py:124-133."""
    return eval_efield_batch(solution, mesh, np.asarray(x, dtype=float)[None], cfg)[0]


def surface_field_magnitudes(mesh: SurfaceMesh, solution, cfg: QuadConfig | None = None, side: float = +1.0,
                             workers: int = 1, *, indices=None) -> np.ndarray:
    """|E| at every collocation point on the side the normal points into
    (reference src/postprocess.py:141-170).  ``indices`` (extension):
    only these collocation points, in that order (a rank's share)."""
    import torch

    from .device import device_mesh

    cfg = cfg or QuadConfig()
    dm = device_mesh(mesh, cfg)
    u_dev, key = _u_device(solution, dm)
    src = _sources(dm, u_dev, key)
    if indices is None:
        own = torch.arange(mesh.n_collocation, dtype=torch.int32, device=dm.device)
        pts = dm.points
    else:
        own = torch.as_tensor(np.asarray(indices, dtype=np.int32), device=dm.device)
        pts = dm.points[own.long()].contiguous()
    m = int(own.shape[0])
    if m == 0:
        return np.zeros(0)
    E = field_points_device(dm, u_dev, src, pts, False, own_col=own)
    emag = torch.empty(m, dtype=torch.float64, device=dm.device)
    _lib.call("hvb_field_singular", _lib.ptr(dm.nodes6), _lib.ptr(dm.tri_cols), _lib.ptr(dm.vc_ptr),
              _lib.ptr(dm.vc_tri), _lib.ptr(dm.vc_corner), _lib.ptr(dm.rule_duffy), dm.n_duffy,
              _lib.ptr(pts), _lib.ptr(dm.normals), _lib.ptr(own), m, _lib.ptr(u_dev),
              float(side), _lib.ptr(E), _lib.ptr(emag), _lib.stream_ptr(dm.device))
    return emag.cpu().numpy()


# ---------------------------------------------------------------------------
# seeds and surface distance (host; reference src/postprocess.py:173-222)
# ---------------------------------------------------------------------------


def surface_distance_batch(mesh: SurfaceMesh, X, cfg: QuadConfig | None = None):
    """(d_surf (m,), local circumradius (m,)) at many points on the device
    (reference _surface_distance, src/postprocess.py:198-218, per point)."""
    import torch

    from .device import device_mesh
    from .tracer import surface_distance_device

    dm = device_mesh(mesh, cfg or QuadConfig())
    X = np.ascontiguousarray(np.asarray(X, dtype=np.float64).reshape(-1, 3))
    out = surface_distance_device(dm, torch.as_tensor(X, device=dm.device)).cpu().numpy()
    return out[:, 0].copy(), out[:, 1].copy()


def _surface_distance(mesh: SurfaceMesh, x: np.ndarray, candidates: int = 12):
    """Reference src/postprocess.py:198-218 for one point (device kernel)."""
    if candidates != 12:
        raise ValueError("the device surface distance ranks 12 candidates (reference default)")
    d, r = surface_distance_batch(mesh, np.asarray(x, dtype=float)[None])
    return float(d[0]), float(r[0])


def _local_circumradius(mesh: SurfaceMesh, x: np.ndarray) -> float:
    return _surface_distance(mesh, x)[1]


def pick_start_points(mesh: SurfaceMesh, solution, k: int, offset_frac: float = 0.25,
                      cfg: QuadConfig | None = None, surface_e: np.ndarray | None = None):
    """Seeds at the k strongest surface-field vertices (src/postprocess.py:173-190)."""
    if surface_e is None:
        surface_e = surface_field_magnitudes(mesh, solution, cfg=cfg)
    order = np.argsort(surface_e)[::-1][:k]
    if len(order) == 0:
        return np.zeros((0, 3)), order, surface_e
    _, local = surface_distance_batch(mesh, mesh.colloc_points[order], cfg)
    starts = mesh.colloc_points[order] + (offset_frac * local)[:, None] * mesh.colloc_normals[order]
    return starts, order, surface_e


# ---------------------------------------------------------------------------
# tracing (Dormand-Prince 5(4) on the unit tangent; src/postprocess.py:229-357)
# ---------------------------------------------------------------------------

_DP_A = (
    (),
    (1 / 5,),
    (3 / 40, 9 / 40),
    (44 / 45, -56 / 15, 32 / 9),
    (19372 / 6561, -25360 / 2187, 64448 / 6561, -212 / 729),
    (9017 / 3168, -355 / 33, 46732 / 5247, 49 / 176, -5103 / 18656),
    (35 / 384, 0.0, 500 / 1113, 125 / 192, -2187 / 6784, 11 / 84),
)
_DP_B5 = np.array([35 / 384, 0.0, 500 / 1113, 125 / 192, -2187 / 6784, 11 / 84, 0.0])
_DP_B4 = np.array([5179 / 57600, 0.0, 7571 / 16695, 393 / 640, -92097 / 339200, 187 / 2100, 1 / 40])


def trace_fieldline(solution, mesh: SurfaceMesh, start, orientation: int = +1, params: TraceParams | None = None,
                    cfg: QuadConfig | None = None) -> FieldLine:
    """Integrate dx/ds = orientation * E/|E| from `start` (one line)."""
    return trace_fieldlines(solution, mesh, np.asarray(start, dtype=float)[None], [orientation],
                            params=params, cfg=cfg, _raise_weak=True)[0]


def trace_fieldlines(solution, mesh: SurfaceMesh, starts, orientations, params: TraceParams | None = None,
                     cfg: QuadConfig | None = None, _raise_weak: bool = False) -> list:
    """Trace many lines; every Runge-Kutta stage of all live lines is one
    batched device field evaluation (lines advance in lockstep)."""
    from .tracer import trace_batch

    return trace_batch(solution, mesh, starts, orientations, params or TraceParams(), cfg or QuadConfig(),
                       raise_weak=_raise_weak)


# ---------------------------------------------------------------------------
# streamer criterion and files
# ---------------------------------------------------------------------------


def streamer_integral(line: FieldLine, model: IonizationModel):
    """Trapezoid integral of alpha(|E|) ds and value > K_str (src/postprocess.py:365-374)."""
    if len(line.points) < 2:
        raise ValueError("field line needs at least two points")
    a = model.alpha(line.e_magnitudes)
    value = float(np.sum(0.5 * (a[1:] + a[:-1]) * np.diff(line.arc_lengths)))
    return value, value > model.k_str


def load_ionization_model(path) -> IonizationModel:
    e_vals, a_vals = [], []
    k_str = None
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            body = raw.split("#", 1)[0].strip()
            if not body:
                continue
            parts = body.split()
            if parts[0] == "kstr":
                k_str = float(parts[1])
                continue
            if len(parts) != 2:
                raise ValueError(f"{path}:{lineno}: expected '<E> <alpha>'")
            e_vals.append(float(parts[0]))
            a_vals.append(float(parts[1]))
    if k_str is None:
        raise ValueError(f"{path}: missing 'kstr <value>' line")
    return IonizationModel(np.array(e_vals), np.array(a_vals), k_str)


def write_fieldline_csv(line: FieldLine, model: IonizationModel | None, path):
    alpha = model.alpha(line.e_magnitudes) if model is not None else np.zeros_like(line.e_magnitudes)
    cum = np.concatenate([[0.0], np.cumsum(0.5 * (alpha[1:] + alpha[:-1]) * np.diff(line.arc_lengths))])
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(["x", "y", "z", "s", "E", "alpha", "cumulative_integral"])
        for i in range(len(line.points)):
            p = line.points[i]
            w.writerow([repr(float(p[0])), repr(float(p[1])), repr(float(p[2])), repr(float(line.arc_lengths[i])),
                        repr(float(line.e_magnitudes[i])), repr(float(alpha[i])), repr(float(cum[i]))])
