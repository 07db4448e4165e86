"""Device-resident Dormand-Prince field-line tracer (reference
trace_fieldline, src/postprocess.py:244-357; surface distance 198-218;
streamer integral 365-374).

Every line is a state machine in HBM (csrc/trace.cu, ``LineState``).  The
host drives *rounds*; per round it launches

    k_field_dyn + reduce      ONE batched N-body over all requests
    k_trace_near              per flagged target: near panels in index order
                              (+ vertex-coincidence flags)
    k_trace_ctrl(mode=1)      consume E at each live line's last request
    k_surface_distance        lines that need d_surf(x) (once per step)
    k_trace_ctrl(mode=2)      consume d_surf, issue the next E request

as ONE C-ABI call (hvb_trace_round) with every count kept on the device:
rounds are enqueued back to back and the host reads the counters (pending
requests, longest polyline) only every ROUNDS_PER_SYNC rounds.  Lines
advance in lockstep, one field evaluation per round, and
the control arithmetic -- stage points, error norm, accept / reject, step
control, surface-hit arming and snapping, termination order -- is the
reference's, statement by statement, on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import ctypes
import os

import numpy as np

from . import _fp, _lib

TERMINATIONS = ("SurfaceHit", "WeakField", "MaxLength", "LeftDomain", "MaxSteps")
STATUS_RUNNING, STATUS_DONE, STATUS_WEAK_START, STATUS_COINCIDENT = 0, 1, 2, 3
VERTEX_PROXIMITY = 1e-12
_LOG = int(os.environ.get("HVB_TRACE_LOG", "0"))  # print progress every N rounds


@dataclass
class TraceResult:
    """Device polylines of a traced batch (torch tensors on the device)."""

    polylines: object   # (L, cap, 5): x, y, z, |E|, s
    info: np.ndarray    # (L, 4): npts, termination code, status, phase
    start_mag: np.ndarray
    state: object
    cap: int
    rounds: int
    field_points: int   # total E evaluations

    @property
    def n_lines(self) -> int:
        return len(self.info)


def _geometry(mesh, params):
    lo, hi = mesh.bounding_box()
    center = 0.5 * (lo + hi)
    half = 0.5 * (hi - lo) * params.bbox_factor
    diag = float(_fp.norm3_fused(hi - lo))
    max_steps = getattr(params, "max_steps", None)
    geo = np.concatenate([center, half, [diag, params.h_min_frac * diag, params.h_max_frac * diag,
                                         params.max_length_frac * diag, params.rel_tol, params.surface_tol_frac,
                                         params.e_floor, float(max_steps) if max_steps else 0.0]])
    return geo.astype(np.float64)


def surface_distance_device(dm, X_dev):
    """(m, 2) = (d_surf, local circumradius) at device points (K12)."""
    import torch

    m = int(X_dev.shape[0])
    out = torch.empty((m, 2), dtype=torch.float64, device=dm.device)
    if m:
        _lib.call("hvb_surface_distance", _lib.ptr(X_dev), m, _lib.ptr(dm.ccr), _lib.ptr(dm.groups), dm.nt,
                  _lib.ptr(dm.nodes6),
                  _lib.ptr(out), _lib.stream_ptr(dm.device))
    return out


ROUNDS_PER_SYNC = 16  # rounds enqueued between host reads of the counters


def _morton_order(X: np.ndarray) -> np.ndarray:
    """Permutation sorting points along a 3-d Morton (Z-order) curve."""
    if len(X) < 2:
        return np.arange(len(X))
    lo, hi = X.min(axis=0), X.max(axis=0)
    q = ((X - lo) / np.maximum(hi - lo, 1e-300) * 1023.0).astype(np.uint64)  # 10 bits per axis
    code = np.zeros(len(X), dtype=np.uint64)
    for b in range(10):
        for d in range(3):
            code |= ((q[:, d] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + d)
    return np.argsort(code, kind="stable")


ROUND_PROBE = None  # dev: list receiving (pending, start event, end event) per round


def trace_device(solution, mesh, starts, orientations, params, cfg, initial_cap: int = 64,
                 max_rounds: int | None = None) -> TraceResult:
    import torch

    from .device import device_mesh
    from .postprocess import _sources, _u_device, panel_split

    dm = device_mesh(mesh, cfg)
    dev = dm.device
    st = _lib.stream_ptr(dev)
    u_dev, key = _u_device(solution, dm)
    src = _sources(dm, u_dev, key)
    starts = np.ascontiguousarray(np.asarray(starts, dtype=np.float64).reshape(-1, 3))
    L = len(starts)
    orient = np.asarray(orientations, dtype=np.float64).reshape(-1)
    if orient.shape != (L,):
        raise ValueError(f"{L} start points but {orient.size} orientations")
    # trace in Morton order of the seeds: the request lists are compacted in
    # roughly line order, so neighbouring lines share warps of the N-body and
    # the far-group classification skip stays coherent.  Per-target results
    # do not depend on the slot, so this changes no result; outputs are put
    # back in the caller's order below.
    order = _morton_order(starts)
    starts = np.ascontiguousarray(starts[order])
    orient = orient[order]
    f64 = dict(dtype=torch.float64, device=dev)
    i32 = dict(dtype=torch.int32, device=dev)
    n = max(1, L)
    sbytes = _lib.lib().hvb_line_state_bytes()
    state = torch.zeros(n * sbytes, dtype=torch.uint8, device=dev)
    geo = np.ascontiguousarray(_geometry(mesh, params))  # host parameters (14 doubles)
    geo_p = geo.ctypes.data_as(ctypes.c_void_p)
    starts_d = torch.as_tensor(starts, **f64)
    orient_d = torch.as_tensor(np.where(orient >= 0, 1, -1).astype(np.int32), **i32)
    K = ROUNDS_PER_SYNC
    cap = max(2 * K + 2, int(initial_cap))
    poly = torch.empty((n, cap, 5), **f64)
    e_pts = [torch.empty((n, 3), **f64), torch.empty((n, 3), **f64)]
    e_line = [torch.empty(n, **i32), torch.empty(n, **i32)]
    sd_pts = torch.empty((n, 3), **f64)
    sd_line = torch.empty(n, **i32)
    sd_out = torch.empty((n, 2), **f64)
    e_out = torch.empty((n, 3), **f64)
    e_flag = torch.zeros(n, **i32)
    split = panel_split(dm.nt)
    has_near = torch.zeros((split, n), **i32)  # chunk flags; the near pass clears what it reads
    part = torch.empty((split, n, 4), **f64)
    counters = torch.zeros(6, dtype=torch.int64, device=dev)  # csrc/launch.cuh TraceArgs.counters
    cfgq = dm.cfg
    rounds = 0
    if L:
        _lib.call("hvb_trace_ctrl", _lib.ptr(state), L, _lib.ptr(starts_d), _lib.ptr(orient_d), geo_p, 0,
                  _lib.ptr(e_pts[0]), _lib.ptr(e_line[0]), _lib.ptr(sd_pts), _lib.ptr(sd_line),
                  _lib.ptr(counters), _lib.ptr(e_out), _lib.ptr(e_flag), _lib.ptr(sd_out), _lib.ptr(poly), cap, st)
    cur = 0
    pending = L
    while pending > 0 and (max_rounds is None or rounds < max_rounds):
        for _ in range(K):
            if ROUND_PROBE is not None:  # dev probe (tools/trace_rounds.py): one round per sync
                ev = [torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)]
                ROUND_PROBE.append([int(counters[0].item()), *ev])
                ev[0].record()
            nxt = 1 - cur
            _lib.call("hvb_trace_round", _lib.ptr(state), L, geo_p, _lib.ptr(e_pts[cur]), _lib.ptr(e_pts[nxt]),
                      _lib.ptr(e_line[nxt]), _lib.ptr(sd_pts), _lib.ptr(sd_line), _lib.ptr(sd_out),
                      _lib.ptr(counters), _lib.ptr(e_out), _lib.ptr(e_flag), _lib.ptr(has_near), _lib.ptr(part),
                      _lib.ptr(src), _lib.ptr(dm.cls), _lib.ptr(dm.groups), _lib.ptr(dm.tri_cols), dm.nt, dm.nq,
                      split,
                      _lib.ptr(dm.nodes6), _lib.ptr(dm.radii), _lib.ptr(dm.ccr), _lib.ptr(u_dev),
                      _lib.ptr(dm.rule_near), len(dm.rule_near), _lib.ptr(dm.rule_graded), len(dm.rule_graded),
                      int(cfgq.bisect_depth), float(cfgq.bisect_trigger), VERTEX_PROXIMITY, _lib.ptr(poly), cap, st)
            cur = nxt
            rounds += 1
            if ROUND_PROBE is not None:
                ROUND_PROBE[-1][2].record()
        c = counters.cpu().numpy()
        pending, max_pts = int(c[0]), int(c[2])
        if _LOG:
            print(f"[trace] round {rounds}: {pending} requests, longest {max_pts} points", flush=True)
        if pending and max_pts + K + 1 >= cap:  # at most one point per line per round
            new_cap = cap
            while max_pts + K + 1 >= new_cap:
                new_cap *= 2
            new = torch.empty((n, new_cap, 5), **f64)
            new[:, :cap] = poly
            poly, cap = new, new_cap

    info = torch.empty((n, 4), **i32)
    dinfo = torch.empty(n, **f64)
    _lib.call("hvb_trace_summary", _lib.ptr(state), L, _lib.ptr(info), _lib.ptr(dinfo), st)
    evals = int(counters[3].item())
    if L > 1:  # back to the caller's line order
        inv = torch.as_tensor(np.argsort(order), device=dev)
        poly = poly[inv]
        state = state.view(n, sbytes)[inv].reshape(-1)
        info = info[inv]
        dinfo = dinfo[inv]
    return TraceResult(polylines=poly, info=info[:L].cpu().numpy(), start_mag=dinfo[:L].cpu().numpy(), state=state,
                       cap=cap, rounds=rounds, field_points=evals)


# host view of csrc/launch.cuh LineState (diagnostics only)
LINE_STATE_DTYPE = np.dtype([("x", "<f8", 3), ("k", "<f8", (7, 3)), ("req", "<f8", 3), ("h", "<f8"), ("s", "<f8"),
                             ("err", "<f8"), ("tol", "<f8"), ("d_surf", "<f8"), ("local_r", "<f8"), ("sign", "<f8"),
                             ("phase", "<i4"), ("stage", "<i4"), ("npts", "<i4"), ("armed", "<i4"), ("term", "<i4"),
                             ("status", "<i4"), ("slot", "<i4"), ("steps", "<i4")])


def line_states(res: TraceResult) -> np.ndarray:
    """Structured host copy of every line's state machine."""
    raw = res.state.cpu().numpy()
    return raw.view(LINE_STATE_DTYPE)[: res.n_lines]


def streamer_device(res: TraceResult, model):
    """(values, verdicts) of every traced line on the device (K14)."""
    import torch

    dev = res.polylines.device
    L = res.n_lines
    e_tab = torch.as_tensor(np.asarray(model.e_values, dtype=np.float64), device=dev)
    a_tab = torch.as_tensor(np.asarray(model.alpha_values, dtype=np.float64), device=dev)
    val = torch.empty(max(1, L), dtype=torch.float64, device=dev)
    ver = torch.empty(max(1, L), dtype=torch.int32, device=dev)
    _lib.call("hvb_streamer", _lib.ptr(res.polylines), _lib.ptr(res.state), L, res.cap, _lib.ptr(e_tab),
              _lib.ptr(a_tab), len(e_tab), float(model.k_str), _lib.ptr(val), _lib.ptr(ver), _lib.stream_ptr(dev))
    return val[:L], ver[:L]


def raise_for_status(res: TraceResult, params, raise_weak: bool):
    from .postprocess import TraceError

    st = res.info[:, 2]
    bad = np.nonzero(st == STATUS_COINCIDENT)[0]
    if len(bad):
        raise ValueError(f"evaluation point coincides with a mesh vertex (line {int(bad[0])})")
    weak = np.nonzero(st == STATUS_WEAK_START)[0]
    if len(weak) and raise_weak:
        mag = float(res.start_mag[weak[0]])
        raise TraceError(
            f"|E| = {mag:.3e} V/m at the start point is not above the weak-field floor {params.e_floor:.3e}")


def field_lines(res: TraceResult) -> list:
    """FieldLine objects (host copies) for every line; None for lines that
    could not start (weak field)."""
    from .postprocess import FieldLine

    L = res.n_lines
    if L == 0:
        return []
    npts = res.info[:, 0]
    m = int(npts.max()) if L else 0
    host = res.polylines[:, :max(1, m)].cpu().numpy()
    out = []
    for i in range(L):
        if res.info[i, 2] != STATUS_DONE:
            out.append(None)
            continue
        k = int(npts[i])
        P = host[i, :k]
        out.append(FieldLine(points=P[:, :3].copy(), e_magnitudes=P[:, 3].copy(), arc_lengths=P[:, 4].copy(),
                             termination=TERMINATIONS[int(res.info[i, 1])]))
    return out


def trace_batch(solution, mesh, starts, orientations, params, cfg, raise_weak=False):
    res = trace_device(solution, mesh, starts, orientations, params, cfg)
    raise_for_status(res, params, raise_weak)
    return field_lines(res)
