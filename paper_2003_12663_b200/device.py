"""Device-resident mesh data and the column-tile schedule of the regular sweep.

Host side (NumPy, once per mesh):

* ``column_tiling`` -- the matrix is stored in a *device column order*:
  recursive coordinate bisection of the collocation points into compact
  column tiles, each swept along its longest axis (csrc/tiling.cpp).  Every
  panel is evaluated once, in the lowest-numbered tile owning one of its
  corners; its corners owned by later tiles are that tile's *halo* columns,
  whose partial sums the owning tile imports (fixed order) before writing
  them.  Within a tile the corners of every stage of GROUP consecutive
  records lie within ``band`` columns of the stage's first column, which is
  what lets the assembly warp keep a WINDOW-column sliding window of running
  sums (csrc/assemble.cu, sweep_geometry(): WINDOW 64, flushes of 16
  columns, band 48).  ``redundancy`` = local columns per device column
  (1.15 at config 4: the halo).
* records (tile, panel) sorted by (tile, first local column).
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

__all__ = ["ColumnTiling", "column_tiling", "DeviceMesh", "device_mesh", "sweep_geometry"]

MAX_TILE = 32767


def sweep_geometry():
    """(window, flush, group, stride) of the built regular sweep
    (csrc/assemble.cu, hvb_sweep_geometry): a WINDOW-column window per warp
    flushed FLUSH columns at a time, so the owned corners of every stage of
    GROUP records must lie within band = WINDOW - FLUSH columns."""
    global _GEOM
    if _GEOM is None:
        import ctypes

        out = (ctypes.c_int * 4)()
        _lib.call("hvb_sweep_geometry", out)
        _GEOM = tuple(int(v) for v in out)
    return _GEOM


_GEOM = None


@dataclass
class ColumnTiling:
    perm: np.ndarray        # device col -> original col (n,)
    inv: np.ndarray         # original col -> device col (n,)
    tile_col0: np.ndarray   # (n_tiles,)
    tile_width: np.ndarray  # (n_tiles,)
    tile_ptr: np.ndarray    # (n_tiles+1,) entry offsets
    tile_lptr: np.ndarray   # (n_tiles+1,) local column offsets
    lcol: np.ndarray        # (n_local,): device column, or ~slot (halo copy / partial)
    tile_xptr: np.ndarray   # (n_tiles+1,) exchange entry offsets
    xent: np.ndarray        # (n_xent, 4): slot, device column, first, last
    tile_pptr: np.ndarray   # (n_tiles+1,) producer offsets
    prods: np.ndarray       # distinct producer tiles per tile
    tile_cptr: np.ndarray   # (n_tiles+1,) consumer offsets
    cons: np.ndarray        # distinct consumer tiles per tile
    n_slots: int            # halo copies + partials
    n_halo: int
    ent_tri: np.ndarray     # (ne,) panel of each entry
    ent_meta: np.ndarray    # (ne, 5): mfirst, l0, l1, l2, flags
    band: int
    redundancy: float


def column_tiling(points: np.ndarray, tri_cols: np.ndarray, max_tile: int = MAX_TILE, band_max: int | None = None,
                  group: int | None = None) -> ColumnTiling:
    """Column tiles + grouped (tile, panel) records, built natively
    (csrc/tiling.cpp, host C++): recursive coordinate bisection into tiles
    of <= max_tile owned columns swept along their longest axis; one record
    per panel, in the lowest-numbered tile owning one of its corners; a
    tile's local columns (owned + halo: its panels' corners owned by later
    tiles) numbered along the sweep axis; records sorted by first local
    column and grouped in stages of ``group`` whose corners are disjoint and
    lie within ``band_max`` columns of the stage's first record (short
    stages padded with dummy records, panel -1); tiles whose records span
    more than ``band_max`` columns are halved across their sweep direction.
    Halo partial sums travel through slots to the owning tile, which sums
    its own partial and the copies in producer order (``xent``).
    ``redundancy`` = local columns per device column."""
    import ctypes

    win, flush, grp, _ = sweep_geometry()
    band_max = win - flush if band_max is None else band_max
    group = grp if group is None else group
    pts = np.ascontiguousarray(points, dtype=np.float64)
    tc = np.ascontiguousarray(tri_cols, dtype=np.int32)
    n, nt = len(pts), len(tc)
    h = _lib.lib()
    sizes = np.zeros(9, dtype=np.int64)
    handle = ctypes.c_void_p()
    rc = h.hvb_tiling_build(pts.ctypes.data_as(ctypes.c_void_p), n, tc.ctypes.data_as(ctypes.c_void_p), nt,
                            int(max_tile), int(band_max), int(group), sizes.ctypes.data_as(ctypes.c_void_p),
                            ctypes.byref(handle))
    if rc != 0:
        raise RuntimeError("column tiling failed" + (": could not bound the panel band" if rc == 2 else ""))
    n_tiles, ne, band, real, n_local, n_x, n_slots, n_halo, n_prod = (int(x) for x in sizes)
    perm = np.empty(n, dtype=np.int32)
    col0 = np.empty(n_tiles, dtype=np.int32)
    width = np.empty(n_tiles, dtype=np.int32)
    ptr = np.empty(n_tiles + 1, dtype=np.int64)
    ent_tri = np.empty(ne, dtype=np.int32)
    ent_meta = np.empty((ne, 5), dtype=np.int32)
    lptr = np.empty(n_tiles + 1, dtype=np.int32)
    lcol = np.empty(n_local, dtype=np.int32)
    xptr = np.empty(n_tiles + 1, dtype=np.int32)
    xent = np.empty((n_x, 4), dtype=np.int32)
    pptr = np.empty(n_tiles + 1, dtype=np.int32)
    prods = np.empty(n_prod, dtype=np.int32)
    cptr = np.empty(n_tiles + 1, dtype=np.int32)
    cons = np.empty(n_prod, dtype=np.int32)
    try:
        h.hvb_tiling_fetch(handle, *(a.ctypes.data_as(ctypes.c_void_p) for a in (perm, col0, width, ptr, ent_tri,
                                                                                 ent_meta, lptr, lcol, xptr, xent,
                                                                                 pptr, prods, cptr, cons)))
    finally:
        h.hvb_tiling_free(handle)
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n)
    return ColumnTiling(perm=perm.astype(np.int64), inv=inv, tile_col0=col0, tile_width=width, tile_ptr=ptr,
                        tile_lptr=lptr, lcol=lcol, tile_xptr=xptr, xent=xent, tile_pptr=pptr, prods=prods,
                        tile_cptr=cptr, cons=cons,
                        n_slots=n_slots, n_halo=n_halo,
                        ent_tri=ent_tri, ent_meta=ent_meta, band=band, redundancy=n_local / max(1, n))


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
        self.window, _, _, self.window_stride = sweep_geometry()
        tiling = mesh_tiling(mesh, max_tile)
        self.tiling = tiling
        self.perm = up(tiling.perm, **i32)
        self.col_dev = up(tiling.inv, **i32)
        self.tile_ptr = up(tiling.tile_ptr, dtype=torch.int64, device=device)
        # launch order of the tiles: most records first (a shorter last wave)
        self.tile_order = up(np.argsort(-np.diff(tiling.tile_ptr), kind="stable").astype(np.int32), **i32)
        self.tile_lptr = up(tiling.tile_lptr, **i32)
        self.lcol = up(tiling.lcol, **i32)
        self.tile_xptr = up(tiling.tile_xptr, **i32)
        self.xent = up(tiling.xent, **i32)
        self.tile_pptr = up(tiling.tile_pptr, **i32)
        self.prods = up(tiling.prods, **i32)
        self.tile_cptr = up(tiling.tile_cptr, **i32)
        self.cons = up(tiling.cons, **i32)
        self.n_slots = tiling.n_slots
        self._ent_tri = up(tiling.ent_tri, **i32)
        self._ent_meta = up(tiling.ent_meta, **i32)  # (mfirst, l0, l1, l2, flags); slots = l % WINDOW on the device
        self.n_entries = len(tiling.ent_tri)
        self.hats = np.ascontiguousarray(
            np.column_stack([1.0 - reg.nodes[:, 0] - reg.nodes[:, 1], reg.nodes[:, 0], reg.nodes[:, 1]]))
        self._streams = {}
        self.stream_for(0)  # SL rows; the ADL stream is built on first use
        self.n_tiles = len(tiling.tile_width)
        self.h2d_bytes = int(sum(h2d))

    def sweep_slots(self, n_doubles: int):
        """Exchange-slot scratch of the regular sweep (csrc/tiling.cpp 5),
        kept across assemblies (grown on demand): the allocation is tens of
        GB at config 4 and must not be re-made per call."""
        import torch

        buf = getattr(self, "_slots", None)
        if buf is None or buf.numel() < n_doubles:
            self._slots = None
            buf = self._slots = torch.empty(max(1, n_doubles), dtype=torch.float64, device=self.device)
        return buf

    def release_scratch(self) -> None:
        """Drop the kept exchange-slot scratch (it is re-made on the next
        assembly); the memory returns to torch's caching allocator."""
        self._slots = None

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
                          _lib.ptr(self._ent_tri), _lib.ptr(self._ent_meta), self.n_entries, mode, self.window,
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


def mesh_tiling(mesh, max_tile: int = MAX_TILE) -> ColumnTiling:
    """Column tiling of a mesh (a mesh-derived array, cached on it)."""
    key = ("tiling", max_tile) + sweep_geometry()
    cache = mesh._device_cache
    t = cache.get(key)
    if t is None:
        t = column_tiling(mesh.colloc_points, mesh.tri_corner_cols, max_tile=max_tile)
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
