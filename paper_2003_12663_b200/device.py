"""Device-resident mesh data and the column-tile schedule of the regular sweep.

Host side (NumPy, once per mesh):

* ``column_tiling`` -- the matrix is stored in a *device column order*:
  recursive coordinate bisection of the collocation points into compact
  column tiles, each swept along its longest axis.  A panel that touches a
  tile contributes to its *owned* corners only; within a tile the owned
  corners of every aligned group of GROUP consecutive records lie within
  ``band`` columns of the group's first owned column, which is what lets
  the assembly warp keep a WINDOW-column sliding window of running sums
  (csrc/assemble.cu: WINDOW 48, flushes of 16 columns, band 32).
  Panels with corners in several tiles are evaluated once per tile
  (``redundancy``, 1.14 at config 4).
* entries (tile, panel) sorted by (tile, first owned column).
* ``panel_groups`` -- bounds of aligned 32-panel groups for the N-body and
  surface-distance kernels.

Device side (``DeviceMesh``, cached per device/config): panel nodes,
circumcircles, sample tables (K1), the packed panel streams, rule tables
(regular, corner Duffy, near Duffy, graded composite), CSR stars.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .quadrature import QuadConfig, duffy_rule, graded_rule, regular_rule

__all__ = ["ColumnTiling", "column_tiling", "DeviceMesh", "device_mesh", "WINDOW"]

# regular-sweep geometry (csrc/assemble.cu): a 48-column window per warp,
# flushed 16 columns at a time, so the panel band over every aligned group of
# GROUP = 4 records (one bulk-copy stage) must stay within WINDOW - FLUSH = 32
# columns.  Measured on cfg4 in round 1: 48 columns beat 40/44/56/64.
WINDOW = 48
FLUSH = 16
GROUP = 4
MAX_TILE = 32767


@dataclass
class ColumnTiling:
    perm: np.ndarray        # device col -> original col (n,)
    inv: np.ndarray         # original col -> device col (n,)
    tile_col0: np.ndarray   # (n_tiles,)
    tile_width: np.ndarray  # (n_tiles,)
    tile_ptr: np.ndarray    # (n_tiles+1,) entry offsets
    ent_tri: np.ndarray     # (ne,) panel of each entry
    ent_meta: np.ndarray    # (ne, 5): mfirst, l0, l1, l2, flags
    band: int
    redundancy: float


def _rcb(points: np.ndarray, idx: np.ndarray, max_tile: int, out: list):
    """Recursive coordinate bisection (median split on the longest axis)."""
    stack = [idx]
    while stack:
        cur = stack.pop()
        if len(cur) <= max_tile:
            out.append(cur)
            continue
        p = points[cur]
        ax = int(np.argmax(p.max(axis=0) - p.min(axis=0)))
        order = np.argsort(p[:, ax], kind="stable")
        h = len(cur) // 2
        # push the second half first so tiles come out in sweep order
        stack.append(cur[order[h:]])
        stack.append(cur[order[:h]])


def _sweep(points: np.ndarray, tile: np.ndarray) -> np.ndarray:
    p = points[tile]
    ax = int(np.argmax(p.max(axis=0) - p.min(axis=0)))
    return tile[np.argsort(p[:, ax], kind="stable")]


def _entries(tri_cols: np.ndarray, tile_of: np.ndarray, local: np.ndarray):
    nt = len(tri_cols)
    ct = tile_of[tri_cols]  # (nt, 3) tile of each corner
    cl = local[tri_cols]
    tri = np.repeat(np.arange(nt), 3)
    tl = ct.ravel()
    # unique (panel, tile) pairs
    key = tri.astype(np.int64) * (int(tile_of.max()) + 1) + tl
    key = np.unique(key)
    e_tri = key // (int(tile_of.max()) + 1)
    e_tile = key % (int(tile_of.max()) + 1)
    owned = ct[e_tri] == e_tile[:, None]  # (ne, 3)
    loc = np.where(owned, cl[e_tri], -1)
    big = np.iinfo(np.int64).max
    mfirst = np.where(owned, loc, big).min(axis=1)
    mlast = np.where(owned, loc, -1).max(axis=1)
    primary = (ct[e_tri, 0] == e_tile).astype(np.int64)
    return e_tri, e_tile, loc, mfirst, mlast, primary


def _split_across(points: np.ndarray, tile: np.ndarray):
    """Halve a tile across its sweep direction (median split on the
    second-longest axis): the sweep front halves, the tile stays a strip."""
    p = points[tile]
    ext = p.max(axis=0) - p.min(axis=0)
    ax = int(np.argsort(ext)[-2])
    order = np.argsort(p[:, ax], kind="stable")
    h = len(tile) // 2
    return [tile[order[:h]], tile[order[h:]]]


def column_tiling(points: np.ndarray, tri_cols: np.ndarray, max_tile: int = 2048,
                  band_max: int = WINDOW - FLUSH, group: int = GROUP, strips: bool = False) -> ColumnTiling:
    """Column tiles + sorted (tile, panel) entries.  The band is measured
    over groups of ``group`` consecutive records of each tile (starting at
    the tile's first record), as the grouped assembly kernel keeps a whole
    group in its window at once.  ``strips``: tiles of up to ``max_tile``
    columns that violate the band are split ACROSS their sweep axis (long
    strips, fewer boundary panels) instead of recursively bisected."""
    n = len(points)
    tri_cols = np.asarray(tri_cols, dtype=np.int64)
    tiles: list = []
    _rcb(points, np.arange(n), max_tile, tiles)
    for _ in range(40):
        tiles = [_sweep(points, t) for t in tiles]
        tile_of = np.empty(n, dtype=np.int64)
        local = np.empty(n, dtype=np.int64)
        for k, t in enumerate(tiles):
            tile_of[t] = k
            local[t] = np.arange(len(t))
        e_tri, e_tile, loc, mfirst, mlast, primary = _entries(tri_cols, tile_of, local)
        order = np.lexsort((e_tri, mfirst, e_tile))
        e_tri, e_tile, loc, mfirst, mlast, primary = (x[order] for x in (e_tri, e_tile, loc, mfirst, mlast,
                                                                          primary))
        counts = np.bincount(e_tile, minlength=len(tiles))
        tile_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        band_e = mlast - mfirst
        if group > 1 and len(e_tri):
            pos = np.arange(len(e_tri)) - tile_ptr[e_tile]
            gid = e_tile * (int(counts.max()) + group) + pos // group  # group key
            first = np.nonzero(pos % group == 0)[0]
            gmax = np.full(len(e_tri), -1, dtype=np.int64)
            np.maximum.at(gmax, np.searchsorted(gid[first], gid), mlast)
            band_e = np.zeros_like(band_e)
            band_e[first] = gmax[: len(first)] - mfirst[first]
        per_tile = np.zeros(len(tiles), dtype=np.int64)
        np.maximum.at(per_tile, e_tile, band_e)
        bad = np.nonzero(per_tile > band_max)[0]
        if len(bad) == 0:
            break
        bad_set = set(bad.tolist())
        nxt: list = []
        for k, t in enumerate(tiles):
            if k in bad_set and len(t) > 1:
                if strips:
                    nxt.extend(_split_across(points, t))
                else:
                    _rcb(points, t, max(1, len(t) // 2), nxt)
            else:
                nxt.append(t)
        tiles = nxt
    else:  # pragma: no cover - pathological mesh
        raise RuntimeError("column tiling: could not bound the panel band")
    perm = np.concatenate(tiles).astype(np.int64)
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n)
    widths = np.array([len(t) for t in tiles], dtype=np.int64)
    col0 = np.concatenate([[0], np.cumsum(widths)[:-1]])
    meta = np.column_stack([mfirst, loc, primary]).astype(np.int32)
    return ColumnTiling(
        perm=perm, inv=inv, tile_col0=col0.astype(np.int32), tile_width=widths.astype(np.int32),
        tile_ptr=tile_ptr, ent_tri=e_tri.astype(np.int32), ent_meta=meta,
        band=int(per_tile.max()) if len(per_tile) else 0,
        redundancy=float(len(e_tri)) / max(1, len(tri_cols)),
    )


def _rule4(rule) -> np.ndarray:
    out = np.zeros((len(rule), 4))
    out[:, :2] = rule.nodes
    out[:, 2] = rule.weights
    return out


class DeviceMesh:
    """All per-mesh device buffers for one (device, quadrature config)."""

    def __init__(self, mesh, cfg: QuadConfig, device, max_tile: int = MAX_TILE):
        import torch

        self.device = device
        self.cfg = cfg
        f64 = dict(dtype=torch.float64, device=device)
        i32 = dict(dtype=torch.int32, device=device)
        self.n = mesh.n_collocation
        self.nt = mesh.n_triangles
        h2d = []  # host arrays copied to the device (bench.py e2e byte count)

        def up(x, **kw):
            t = torch.as_tensor(x, **kw).contiguous()
            h2d.append(t.numel() * t.element_size())
            return t

        self.nodes6 = up(mesh.tri_nodes.reshape(self.nt, 18), **f64)
        self.tri_cols = up(mesh.tri_corner_cols, **i32)
        self.radii = up(mesh.circumradii, **f64)
        self.points = up(mesh.colloc_points, **f64)
        self.normals = up(mesh.colloc_normals, **f64)
        self.vc_ptr = up(mesh.vc_ptr, **i32)
        self.vc_tri = up(mesh.vc_tri, **i32)
        self.vc_corner = up(mesh.vc_corner, **i32)
        st = _lib.stream_ptr(device)
        # per-panel classification arrays and the 32-panel group bounds, built
        # on the device from the circumcircles (csrc/tables.cu k_panel_data;
        # equal to the host statement panel_groups below)
        cc = up(mesh.circumcenters, **f64)
        self.ccr = torch.empty((self.nt, 4), **f64)     # cc, R
        self.cls = torch.empty((self.nt, 6), **f64)     # cc, thr, lo, hi
        self.groups = torch.empty((-(-self.nt // PANEL_GROUP), 8), **f64)
        _lib.call("hvb_panel_data", _lib.ptr(cc), _lib.ptr(self.radii), self.nt, float(cfg.eta), _lib.ptr(self.ccr),
                  _lib.ptr(self.cls), _lib.ptr(self.groups), st)

        # rule tables
        reg = regular_rule(cfg.regular_order)
        self.nq = len(reg)
        self.rule_regular = torch.as_tensor(_rule4(reg), **f64)
        self.rule_duffy = torch.as_tensor(
            np.concatenate([_rule4(duffy_rule(c, cfg.duffy_points)) for c in range(3)]), **f64)
        self.n_duffy = len(duffy_rule(0, cfg.duffy_points))
        self.rule_near = torch.as_tensor(_rule4(duffy_rule(0, cfg.near_duffy_points)), **f64)
        self.rule_graded = torch.as_tensor(
            _rule4(graded_rule(cfg.bisect_depth, cfg.near_duffy_points, cfg.near_outer_order)), **f64)

        # K1 sample table
        self.table = torch.empty((self.nt, self.nq, 6), **f64)
        _lib.call("hvb_build_table", _lib.ptr(self.nodes6), self.nt, self.nq, _lib.ptr(self.rule_regular),
                  _lib.ptr(self.table), st)

        # column tiling + panel streams
        self.window = WINDOW
        tiling = mesh_tiling(mesh, max_tile, WINDOW, True, GROUP, FLUSH)
        self.tiling = tiling
        self.perm = up(tiling.perm, **i32)
        self.col_dev = up(tiling.inv, **i32)
        self.tile_ptr = up(tiling.tile_ptr, dtype=torch.int64, device=device)
        self.tile_col0 = up(tiling.tile_col0, **i32)
        self.tile_width = up(tiling.tile_width, **i32)
        self._ent_tri = up(tiling.ent_tri, **i32)
        self._ent_meta = up(tiling.ent_meta, **i32)  # (mfirst, l0, l1, l2, flags); slots = l % WINDOW on the device
        self.n_entries = len(tiling.ent_tri)
        self.hats = np.ascontiguousarray(
            np.column_stack([1.0 - reg.nodes[:, 0] - reg.nodes[:, 1], reg.nodes[:, 0], reg.nodes[:, 1]]))
        self._streams = {}
        self.stream_for(0)  # SL rows; the ADL stream is built on first use
        self.n_tiles = len(tiling.tile_width)
        self.h2d_bytes = int(sum(h2d))

    def stream_for(self, mode: int):
        """Packed panel stream of the regular sweep: mode 0 (SL rows) or 1
        (ADL rows) record format (csrc/assemble.cu)."""
        import torch

        st = self._streams.get(mode)
        if st is None:
            rec = _lib.lib().hvb_stream_record_doubles(self.nq, mode)
            if rec <= 0:
                raise ValueError(f"no sweep record format for nq={self.nq}")
            st = torch.empty((self.n_entries, rec), dtype=torch.float64, device=self.device)
            with torch.cuda.device(self.device):
                _lib.call("hvb_build_stream", _lib.ptr(self.table), self.nq, _lib.ptr(self.ccr), float(self.cfg.eta),
                          _lib.ptr(self._ent_tri), _lib.ptr(self._ent_meta), self.n_entries, mode, WINDOW,
                          _lib.ptr(st), _lib.stream_ptr(self.device))
            self._streams[mode] = st
        return st


PANEL_GROUP = 32  # csrc/field.cu FCH: panels per shared-memory batch / bound group


def panel_groups(cc: np.ndarray, radii: np.ndarray, thr: np.ndarray) -> np.ndarray:
    """Bounding data of aligned groups of PANEL_GROUP consecutive panels,
    (n_groups, 8) = centre (3), rho_cls, rho_sd, pad: every panel t of the
    group satisfies ||cc_t - C|| + fl(eta R_t) <= rho_cls and ||cc_t - C|| +
    R_t <= rho_sd (inflated by 1e-12 relative).  A target with ||x - C|| >
    rho_cls (1 + 1e-12) classifies every panel of the group regular, and
    ||x - C|| - rho_sd bounds the group's surface-distance keys from below
    -- both exactly, far beyond FP64 rounding (csrc/field.cu, trace.cu)."""
    nt = len(cc)
    ng = -(-nt // PANEL_GROUP)
    pad = ng * PANEL_GROUP - nt
    idx = np.concatenate([np.arange(nt), np.full(pad, nt - 1)]).reshape(ng, PANEL_GROUP)
    c = cc[idx]                              # (ng, G, 3)
    lo, hi = c.min(axis=1), c.max(axis=1)
    C = 0.5 * (lo + hi)
    d = np.sqrt(((c - C[:, None, :]) ** 2).sum(axis=2))
    out = np.zeros((ng, 8))
    out[:, :3] = C
    out[:, 3] = (d + thr[idx]).max(axis=1) * (1.0 + 1e-12)
    out[:, 4] = (d + radii[idx]).max(axis=1) * (1.0 + 1e-12)
    return out


def mesh_tiling(mesh, max_tile: int = 2048, window: int = 96, strips: bool = False, group: int = 2,
                flush: int = 32) -> ColumnTiling:
    """Host column tiling of a mesh (a mesh-derived array, cached on it)."""
    key = ("tiling", max_tile, window, strips, group, flush)
    cache = mesh._device_cache
    t = cache.get(key)
    if t is None:
        t = column_tiling(mesh.colloc_points, mesh.tri_corner_cols, max_tile=max_tile, band_max=window - flush,
                          group=group, strips=strips)
        cache[key] = t
    return t


def device_mesh(mesh, cfg: QuadConfig | None = None, device=None) -> DeviceMesh:
    cfg = cfg or QuadConfig()
    dev = _lib.require_device(device)
    key = ("dm", str(dev), cfg)
    dm = mesh._device_cache.get(key)
    if dm is None:
        import torch

        with torch.cuda.device(dev):
            dm = DeviceMesh(mesh, cfg, dev)
        mesh._device_cache[key] = dm
    return dm
