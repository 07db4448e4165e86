"""Dense collocation-system assembly on the device.

Public API of reference ``src/assembly.py`` (assemble, SystemMatrix,
RowBlock, matvec, partition_rows, charge_row, assemble_kernel_row,
save_matrix, load_matrix, TriangleTables, KERNEL_*).  All arithmetic runs in
libhvb.so; this module plans the launches and owns the device buffers.

Row equations (reference ``_row_equation`` src/assembly.py:408-468):

* Dirichlet / floating rows: SL row (+ -1 in the floating column), rhs v0 / 0;
* dielectric rows: (eps+ - eps-) ADL row + (eps+ + eps-)/2 on the diagonal;
* neutrality row n+k: sum over the surface's rows of w_i*adl*ADL_i plus
  w_i*id on column i, with (adl, id) = (eps+-eps-, (eps++eps-)/2) for sheets,
  else (EPS0, EPS0/2).

Pass structure per row block (one CUDA stream, no host sync until the
near-pair count is read): regular sweep (writes every collocation entry
once, emits near pairs) -> near pairs sorted by (row, panel) -> near kernel
-> ordered apply -> singular Duffy pass (+ dielectric diagonal) ->
floating columns.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .mesh import EPS0, KIND_DIELECTRIC, KIND_FLOATING, SurfaceMesh, shape_functions, shape_gradients
from .quadrature import QuadConfig, regular_rule
from . import _fp

__all__ = [
    "AssemblyError",
    "Neutrality",
    "RowBlock",
    "SystemMatrix",
    "TriangleTables",
    "assemble",
    "partition_rows",
    "matvec",
    "charge_row",
    "assemble_kernel_row",
    "adl_chunk_sum",
    "save_matrix",
    "load_matrix",
    "KERNEL_SL",
    "KERNEL_ADL",
    "KERNEL_E",
]

FOUR_PI = 4.0 * np.pi
KERNEL_SL = "sl"
KERNEL_ADL = "adl"
KERNEL_E = "efield"
LDA_ALIGN = 32  # row pitch in elements (256-byte aligned rows for the GEMV)
HALO_BYTES = 40 << 30  # scratch cap of one regular-sweep launch (exchange slots; also <= 1/3 of free memory)
# precision="single" matrices: False (default) reduces every row in float32
# as the reference's float32 dot does; True keeps float32 products but sums
# in double (more accurate, not the reference's arithmetic)
SINGLE_SUMS_F64 = False


class AssemblyError(RuntimeError):
    """Mesh admits no consistent system (reference src/assembly.py:53)."""


@dataclass(frozen=True)
class Neutrality:
    index: int
    sheet: bool
    eps_plus: float
    eps_minus: float


class TriangleTables:
    """Host regular-rule sample tables (reference src/assembly.py:73-103);
    kept for API parity -- the device uses hvb_build_table."""

    def __init__(self, mesh: SurfaceMesh, order: int):
        rule = regular_rule(order)
        self.mesh = mesh
        self.order = order
        self.rule = rule
        self.nq = len(rule)
        sh = shape_functions(rule.nodes)
        gu, gv = shape_gradients(rule.nodes)
        nodes = mesh.tri_nodes
        pts = np.einsum("qk,tkd->tqd", sh, nodes)
        cr = _fp.cross3(np.einsum("qk,tkd->tqd", gu, nodes), np.einsum("qk,tkd->tqd", gv, nodes))
        jac = _fp.norm3_axis(cr)
        self.points_flat = pts.reshape(-1, 3)
        self.jw = rule.weights[None, :] * jac
        self.normals = cr / jac[..., None]
        self.hats = np.column_stack([1.0 - rule.nodes[:, 0] - rule.nodes[:, 1], rule.nodes[:, 0], rule.nodes[:, 1]])


def partition_rows(total: int, n_blocks: int) -> list:
    """Contiguous ranges, sizes differing by at most one (src/assembly.py:362-373)."""
    if n_blocks < 1 or n_blocks > total:
        raise ValueError(f"need 1 <= n_blocks <= {total}, got {n_blocks}")
    q, r = divmod(total, n_blocks)
    bounds = np.cumsum([0] + [q + (1 if b < r else 0) for b in range(n_blocks)])
    return [(int(bounds[b]), int(bounds[b + 1])) for b in range(n_blocks)]


# ---------------------------------------------------------------------------
# matrix container
# ---------------------------------------------------------------------------


class DeviceStore:
    """Row-major (rows, lda) device matrix in device column order."""

    def __init__(self, tensor, n: int, size: int, perm_t, perm_np, row0: int = 0):
        self.A = tensor          # torch (rows, lda)
        self.n = n
        self.size = size
        self.perm_t = perm_t     # torch int32 (n,) device col -> original col, or None
        self.perm = perm_np      # numpy (n,) or None (identity)
        self.row0 = row0         # global index of the first stored row

    @property
    def lda(self) -> int:
        return int(self.A.shape[1])

    @property
    def is_f32(self) -> bool:
        import torch

        return self.A.dtype == torch.float32

    @property
    def prec(self) -> int:
        """hvb_gemv storage/summation code: 0 double; 1 float32 storage with
        the reference's float32 row sums (src/assembly.py:386-392); 2 float32
        storage with double sums (opt-in, SINGLE_SUMS_F64)."""
        if not self.is_f32:
            return 0
        return 2 if SINGLE_SUMS_F64 else 1

    def host_rows(self, start: int, stop: int) -> np.ndarray:
        dev = self.A[start:stop, : self.size].cpu().numpy()
        if self.perm is None:
            return np.ascontiguousarray(dev)
        out = np.empty_like(dev)
        out[:, self.perm] = dev[:, : self.n]
        out[:, self.n:] = dev[:, self.n:]
        return out


class RowBlock:
    """Contiguous row range of a SystemMatrix.  ``data`` is a host view in
    the original column order (a copy for device-resident matrices)."""

    def __init__(self, start: int, stop: int, data=None, *, store: DeviceStore | None = None):
        self.start = int(start)
        self.stop = int(stop)
        self._data = None if data is None else np.asarray(data)
        self._store = store
        self.version = 0  # bumped when ``data`` is replaced (SystemMatrix re-uploads)

    def __len__(self):
        return self.stop - self.start

    @property
    def data(self) -> np.ndarray:
        if self._data is None:
            return self._store.host_rows(self.start, self.stop)
        return self._data

    @data.setter
    def data(self, value):
        self._data = np.asarray(value)
        self._store = None
        self.version += 1

    @property
    def device_resident(self) -> bool:
        return self._data is None


@dataclass
class SystemMatrix:
    """Row-partitioned dense system (reference src/assembly.py:319-359).

    Device-assembled matrices keep their blocks in HBM (``store``); host
    arrays passed by callers are uploaded on first use."""

    n: int
    n_floating: int
    blocks: list
    diagnostics: dict = field(default_factory=dict)
    store: DeviceStore | None = None

    @property
    def shape(self):
        s = self.n + self.n_floating
        return (s, s)

    @property
    def size(self) -> int:
        return self.n + self.n_floating

    def row(self, i: int) -> np.ndarray:
        for b in self.blocks:
            if b.start <= i < b.stop:
                if b.device_resident:
                    return self.store.host_rows(i, i + 1)[0]
                return b.data[i - b.start]
        raise IndexError(i)

    def diagonal(self) -> np.ndarray:
        st = self.device_store()
        rowmax, diag = _rowmax_diag(st)
        return diag.cpu().numpy()

    def toarray(self) -> np.ndarray:
        return np.vstack([b.data for b in self.blocks])

    def matvec(self, v, workers: int = 1) -> np.ndarray:
        return matvec(self, v, workers=workers)

    def device_store(self) -> DeviceStore:
        """The device copy.  Host-backed blocks are uploaded on first use and
        again whenever a block's ``data`` was replaced since (the reference
        reads the blocks on every call; an in-place edit of a block's array
        needs ``invalidate()``)."""
        stamp = tuple((id(b), b.version, id(b._data)) for b in self.blocks if not b.device_resident)
        if self.store is not None and stamp and stamp != getattr(self, "_host_stamp", None):
            self.store = None
        if self.store is None:
            import torch

            dev = _lib.require_device()
            data = np.vstack([np.asarray(b.data) for b in self.blocks])
            dt = torch.float32 if data.dtype == np.float32 else torch.float64
            lda = -(-self.size // LDA_ALIGN) * LDA_ALIGN
            A = torch.zeros((self.size, lda), dtype=dt, device=dev)
            A[:, : self.size] = torch.as_tensor(data, dtype=dt, device=dev)
            self.store = DeviceStore(A, self.n, self.size, None, None)
            self._host_stamp = stamp
        return self.store

    def invalidate(self):
        """Drop the device copy of host-backed blocks (re-uploaded on use)."""
        if any(not b.device_resident for b in self.blocks):
            self.store = None


def _rowmax_diag(st: DeviceStore):
    import torch

    dev = st.A.device
    rows = st.A.shape[0]
    g = np.arange(st.row0, st.row0 + rows)  # global row -> its diagonal column
    if st.perm is not None:
        inv = np.empty(st.n, dtype=np.int64)
        inv[st.perm] = np.arange(st.n)
        g = np.where(g < st.n, inv[np.minimum(g, st.n - 1)], g)
    diag_col = torch.as_tensor(g, dtype=torch.int32, device=dev)
    rowmax = torch.empty(rows, dtype=torch.float64, device=dev)
    diag = torch.empty(rows, dtype=torch.float64, device=dev)
    _lib.call("hvb_rowmax_diag", _lib.ptr(st.A), int(st.is_f32), st.lda, rows, st.size,
              _lib.ptr(diag_col), _lib.ptr(rowmax), _lib.ptr(diag), _lib.stream_ptr(dev))
    return rowmax, diag


def gather_operand(st: DeviceStore, z, right=None):
    """xp = (z ./ right) in the store's device column order."""
    import torch

    dev = st.A.device
    xp = torch.empty(st.size, dtype=torch.float64, device=dev)
    s = _lib.stream_ptr(dev)
    if st.perm_t is None:
        _lib.call("hvb_gather_scale", _lib.ptr(z), _lib.ptr(right), None, st.size, _lib.ptr(xp), s)
    else:
        _lib.call("hvb_gather_scale", _lib.ptr(z), _lib.ptr(right), _lib.ptr(st.perm_t), st.n, _lib.ptr(xp), s)
        if st.size > st.n:
            zt = z[st.n:]
            xp[st.n:] = zt / right[st.n:] if right is not None else zt
    return xp


def device_matvec(st: DeviceStore, z, right=None, left=None, out=None):
    """y = left .* (A (z ./ right)) on the device; z/right/left in original
    order (torch float64 tensors)."""
    import torch

    dev = st.A.device
    xp = gather_operand(st, z, right)
    s = _lib.stream_ptr(dev)
    rows = st.A.shape[0]
    y = out if out is not None else torch.empty(rows, dtype=torch.float64, device=dev)
    _lib.call("hvb_gemv", _lib.ptr(st.A), st.prec, st.lda, rows, st.size, _lib.ptr(xp),
              _lib.ptr(left), _lib.ptr(y), s)
    return y


def matvec(matrix: SystemMatrix, v, workers: int = 1) -> np.ndarray:
    """Dense product (reference src/assembly.py:376-400), on the device.
    Per-row reduction order depends only on the column count, so results
    are bitwise identical for any block partition."""
    import torch

    v = np.asarray(v)
    if v.shape != (matrix.size,):
        raise ValueError(f"vector of length {len(v)} against size {matrix.size}")
    st = matrix.device_store()
    z = torch.as_tensor(np.asarray(v, dtype=np.float64), device=st.A.device)
    return device_matvec(st, z).cpu().numpy()


# ---------------------------------------------------------------------------
# row planning
# ---------------------------------------------------------------------------


@dataclass
class RowPlan:
    """Row list of one kernel launch set (device tensors)."""

    rowdata: object    # (m, 6) x, n
    kind: object       # (m,) 0 SL, 1 ADL
    col: object        # (m,) own collocation col (original) or -1
    scale: object      # (m,)
    diag: object       # (m,)
    out: object        # (m,) int64 element offset of the row in A
    m: int
    n_sl: int          # rows [0, n_sl) are SL, the rest ADL


def _plan(dev, x, nrm, kind, col, scale, diag, out_off) -> RowPlan:
    import torch

    order = np.argsort(kind, kind="stable")  # SL rows first
    f64 = dict(dtype=torch.float64, device=dev)
    rd = np.column_stack([x, nrm])[order]
    return RowPlan(
        rowdata=torch.as_tensor(np.ascontiguousarray(rd), **f64),
        kind=torch.as_tensor(kind[order].astype(np.int32), device=dev),
        col=torch.as_tensor(col[order].astype(np.int32), device=dev),
        scale=torch.as_tensor(scale[order], **f64),
        diag=torch.as_tensor(diag[order], **f64),
        out=torch.as_tensor(out_off[order].astype(np.int64), device=dev),
        m=len(order),
        n_sl=int(np.count_nonzero(kind == 0)),
    )


LAST_NEAR_ROWS = None  # near pairs per collocation row of the last assembly (bench roofline)

# Optional phase profiler (bench.py): a list that receives
# (label, start_event, end_event) triples recorded on the launching stream.
PROFILE = None


def _mark():
    if PROFILE is None:
        return None
    import torch

    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def _span(label, e0):
    if PROFILE is not None and e0 is not None:
        PROFILE.append((label, e0, _mark()))


def _run_rows(dm, plan: RowPlan, A, counts: dict, part_ld: int = 0):
    """Regular + near + singular passes for one row plan writing into A.
    part_ld > 0 (charge-reduce mode, ADL rows only): A holds one partial row
    per 32-row tile and plan.out[r] must be (r // 32) * part_ld."""
    import torch

    dev = dm.device
    if plan.m == 0:
        return
    with torch.cuda.device(dev):
        _run_rows_on(dm, plan, A, counts, part_ld)


def _run_rows_on(dm, plan: RowPlan, A, counts: dict, part_ld: int = 0):
    import torch

    dev = dm.device
    s = _lib.stream_ptr(dev)
    hats = dm.hats.ctypes.data_as(ctypes.c_void_p)
    cap = max(4096, 16 * plan.m)
    e_reg = _mark()
    while True:
        near = torch.empty((cap, 2), dtype=torch.int32, device=dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        for lo, hi, mode in ((0, plan.n_sl, 0), (plan.n_sl, plan.m, 1)):
            # launches of <= HALO_BYTES of exchange slots (csrc/tiling.cpp 5):
            # one launch per row kind when memory allows (each launch has a tail)
            have = getattr(dm, "_slots", None)
            cap = max(0 if have is None else have.numel() * 8,
                      min(HALO_BYTES, torch.cuda.mem_get_info(dev)[0] // 3))
            step = max(128, cap // (8 * max(1, dm.n_slots)) // 128 * 128)
            for a in range(lo, hi, step):
                b = min(hi, a + step)
                halo = dm.sweep_slots(dm.n_slots * (b - a))
                sched = torch.empty(int(_lib.lib().hvb_sweep_sched_ints(b - a, dm.n_tiles)), dtype=torch.int32,
                                    device=dev)
                _lib.call(
                    "hvb_assemble_regular", _lib.ptr(dm.stream_for(mode)), _lib.ptr(dm.tile_ptr),
                    _lib.ptr(dm.tile_order), _lib.ptr(dm.tile_lptr), _lib.ptr(dm.lcol), _lib.ptr(dm.tile_xptr), _lib.ptr(dm.xent),
                    _lib.ptr(dm.tile_pptr), _lib.ptr(dm.prods), _lib.ptr(dm.tile_cptr), _lib.ptr(dm.cons),
                    dm.n_tiles, dm.nq, hats, a, b - a, _lib.ptr(plan.rowdata), _lib.ptr(plan.col),
                    _lib.ptr(plan.scale), _lib.ptr(plan.out), _lib.ptr(A), part_ld, _lib.ptr(dm.tri_cols), mode,
                    _lib.ptr(halo), _lib.ptr(sched), _lib.ptr(near), _lib.ptr(cnt), cap, s)
        n_near = int(cnt.item())
        if n_near <= cap:
            break
        cap = n_near + 1024  # overflow: rerun with room (regular entries are simply rewritten)
    _span("regular", e_reg)
    counts["near"] += n_near
    if n_near:
        per = torch.bincount(near[:n_near, 0].long(), minlength=plan.m).cpu().numpy()
        counts.setdefault("near_rows", []).append((plan.col.cpu().numpy(), per))
    e_near = _mark()
    if n_near:
        pairs = _sort_pairs(near[:n_near], dm.nt)
        contrib = torch.empty((n_near, 9), dtype=torch.float64, device=dev)
        _lib.call("hvb_near_pairs", _lib.ptr(pairs), n_near, _lib.ptr(plan.rowdata), _lib.ptr(plan.kind),
                  _lib.ptr(dm.nodes6), _lib.ptr(dm.radii), _lib.ptr(dm.rule_near), len(dm.rule_near),
                  _lib.ptr(dm.rule_graded), len(dm.rule_graded), int(dm.cfg.bisect_depth),
                  float(dm.cfg.bisect_trigger), _lib.ptr(contrib), s)
        # one sequential segment per row (per 32-row tile in charge-reduce mode)
        seg = _segments(pairs[:, 0] // 32 if part_ld else pairs[:, 0])
        _lib.call("hvb_near_apply_rows", _lib.ptr(seg), len(seg) - 1, _lib.ptr(pairs), _lib.ptr(contrib),
                  _lib.ptr(dm.tri_cols), _lib.ptr(dm.col_dev), _lib.ptr(plan.scale), _lib.ptr(plan.out),
                  _lib.ptr(A), s)
    _span("near", e_near)
    e_sing = _mark()
    _lib.call("hvb_assemble_singular", _lib.ptr(dm.nodes6), _lib.ptr(dm.tri_cols), _lib.ptr(dm.col_dev),
              _lib.ptr(dm.vc_ptr), _lib.ptr(dm.vc_tri), _lib.ptr(dm.vc_corner), _lib.ptr(dm.rule_duffy),
              dm.n_duffy, plan.m, _lib.ptr(plan.rowdata), _lib.ptr(plan.kind), _lib.ptr(plan.col),
              _lib.ptr(plan.scale), _lib.ptr(plan.diag), _lib.ptr(plan.out), _lib.ptr(A), 32 if part_ld else 1, s)
    _span("singular", e_sing)


def _sort_pairs(pairs, nt: int):
    import torch

    key = pairs[:, 0].to(torch.int64) * (nt + 1) + pairs[:, 1].to(torch.int64)
    order = torch.sort(key, stable=True).indices
    return pairs[order].contiguous()


def _segments(first_col):
    """CSR pointer over runs of equal (sorted) keys."""
    import torch

    keys = first_col.to(torch.int64)
    change = torch.ones_like(keys, dtype=torch.bool)
    change[1:] = keys[1:] != keys[:-1]
    starts = torch.nonzero(change).flatten()
    ptr = torch.cat([starts, torch.tensor([keys.shape[0]], device=keys.device)])
    return ptr.to(torch.int32).contiguous()


def _row_coeffs(mesh, rows):
    """(kind 0/1, scale, diag) of collocation rows (reference _row_equation)."""
    code = mesh.row_kind_code[rows]
    diel = code == KIND_DIELECTRIC
    ep = mesh.row_eps_plus[rows]
    em = mesh.row_eps_minus[rows]
    kind = diel.astype(np.int64)
    scale = np.where(diel, ep - em, 1.0)
    diag = np.where(diel, 0.5 * (ep + em), 0.0)
    return kind, scale, diag


def _neutrality_scales(mesh, k: int):
    """(adl_scale, id_scale) of floating surface k (src/assembly.py:441-457)."""
    sheet = False
    ep = em = EPS0
    for p in mesh.patches.values():
        if p.is_floating and p.index == k and p.kind == "sheet":
            sheet = True
            ep, em = p.eps_plus, p.eps_minus
    if sheet:
        return ep - em, 0.5 * (ep + em)
    return ep, 0.5 * ep


NEUTRALITY_CHUNK = 4096  # members per partial sum of a neutrality / charge row


def _charge_chunk(mesh, dm, mem, adl_scale, id_scale, out, accumulate: bool):
    """out (+)= sum_i w_i adl ADL_i + w_i id e_i over one chunk of members, in
    DEVICE column order, fused (csrc/assemble.cu charge-reduce mode): the
    sweep writes one partial row per 32 members, the near / singular /
    diagonal terms are added into the same partial rows in a fixed order and
    hvb_charge_reduce sums the partial rows in order -- no (members, N)
    scratch."""
    import torch

    n = mesh.n_collocation
    lda = -(-n // LDA_ALIGN) * LDA_ALIGN
    mem = np.asarray(mem, dtype=np.int64)
    m = len(mem)
    tiles = -(-m // 32)
    w = mesh.lumped_weights[mem]
    part = torch.empty((tiles, lda), dtype=torch.float64, device=dm.device)
    plan = _plan(dm.device, mesh.colloc_points[mem], mesh.colloc_normals[mem], np.ones(m, np.int64), mem,
                 w * adl_scale, w * id_scale, (np.arange(m) // 32) * lda)
    _run_rows(dm, plan, part, {"near": 0}, part_ld=lda)
    with torch.cuda.device(dm.device):
        _lib.call("hvb_charge_reduce", _lib.ptr(part), tiles, lda, n, _lib.ptr(out), int(accumulate),
                  _lib.stream_ptr(dm.device))
    return out


def adl_chunk_sum(mesh, dm, mem, adl_scale, id_scale):
    """Partial sum_i w_i adl ADL_i + w_i id e_i over one chunk of members, in
    DEVICE column order (the unit the neutrality rows are split into)."""
    import torch

    out = torch.empty(mesh.n_collocation, dtype=torch.float64, device=dm.device)
    return _charge_chunk(mesh, dm, mem, adl_scale, id_scale, out, accumulate=False)


def _weighted_adl_sum(mesh, dm, members, adl_scale, id_scale, chunk: int | None = None):
    """sum_i w_i adl ADL_i + w_i id e_i over `members`, in DEVICE column
    order: chunk partials added in chunk order -- the same order
    parallel.assemble_distributed uses when the chunks are spread over
    ranks, so the row is bitwise independent of the GPU count."""
    import torch

    chunk = chunk or NEUTRALITY_CHUNK
    acc = torch.zeros(mesh.n_collocation, dtype=torch.float64, device=dm.device)
    for c0 in range(0, len(members), chunk):
        _charge_chunk(mesh, dm, members[c0:c0 + chunk], adl_scale, id_scale, acc, accumulate=True)
    return acc


def assemble(mesh: SurfaceMesh, cfg: QuadConfig | None = None, n_blocks: int = 1, workers: int = 1,
             precision: str = "double", device=None):
    """Build the dense (n + N_fl) system and rhs (reference src/assembly.py:471-532).

    The matrix stays in HBM (row-major, device column order, 256-byte row
    pitch); ``n_blocks`` gives the reference's contiguous row blocks as
    views.  ``workers`` is accepted for signature compatibility."""
    import torch

    cfg = cfg or QuadConfig()
    n = mesh.n_collocation
    size = n + mesh.n_floating
    if precision not in ("double", "single"):
        raise AssemblyError(f"unknown precision {precision!r}")
    for k in range(mesh.n_floating):
        mem = mesh.floating_collocation(k)
        if len(mem) == 0:
            raise AssemblyError(
                f"floating surface {k} has no collocation points; cannot write its neutrality row"
            )
        if mesh.lumped_weights[mem].sum() <= 0.0:
            raise AssemblyError(f"floating surface {k} has zero area")
    ranges = partition_rows(size, n_blocks)
    dm = _device_mesh(mesh, cfg, device)
    A, counts = assemble_rows(mesh, dm, 0, size, precision)
    store = DeviceStore(A, n, size, dm.perm, dm.tiling.perm)
    blocks = [RowBlock(a, b, store=store) for a, b in ranges]
    rhs = np.where(mesh.row_kind_code == 0, mesh.row_v0, 0.0)
    rhs = np.concatenate([rhs, np.zeros(mesh.n_floating)])
    nt = mesh.n_triangles
    singular = int(mesh.vc_ptr[-1])
    matrix = SystemMatrix(n=n, n_floating=mesh.n_floating, blocks=blocks, store=store)
    matrix.diagnostics = {
        "pairs_regular": n * nt - singular - counts["near"],
        "pairs_singular": singular,
        "pairs_near_singular": counts["near"],
        "rows_with_integrals": n,
        "n_triangles": nt,
        "precision": precision,
        "quad": cfg,
        "column_tiles": dm.n_tiles,
        "tile_redundancy": dm.tiling.redundancy,
    }
    return matrix, rhs


def assemble_rows(mesh: SurfaceMesh, dm, start: int, stop: int, precision: str = "double", neutrality=None):
    """Device rows [start, stop) of the system (a row block of
    ``partition_rows``) as a (stop-start, lda) tensor in device column
    order, plus pair counts over its collocation rows.  Every row is computed
    independently of the block boundaries, so any partition gives bitwise
    identical rows (reference invariance, tests/test_assembly.py:146-158)."""
    import torch

    n = mesh.n_collocation
    size = n + mesh.n_floating
    dev = dm.device
    lda = -(-size // LDA_ALIGN) * LDA_ALIGN
    counts = {"near": 0}
    with torch.cuda.device(dev):
        e0 = _mark()
        A = torch.empty((stop - start, lda), dtype=torch.float64, device=dev)
        _span("alloc", e0)
        rows = np.arange(start, min(stop, n))
        if len(rows):
            e0 = _mark()
            # the row plan is mesh-derived (rows, kinds, scales, output
            # offsets): built and uploaded once per device mesh and row range
            # (re-checked against the mesh's current row coefficients: a
            # changed permittivity or potential rebuilds it)
            plans = dm.__dict__.setdefault("_plan_cache", {})
            kind, scale, diag = _row_coeffs(mesh, rows)
            hit = plans.get((start, stop, lda))
            off = (rows - start) * lda
            if hit is not None and all(np.array_equal(x, y) for x, y in zip(hit[1], (kind, scale, diag))):
                plan = hit[0]
            else:
                plan = _plan(dev, mesh.colloc_points[rows], mesh.colloc_normals[rows], kind, rows, scale, diag, off)
                plans[(start, stop, lda)] = (plan, (kind, scale, diag))
            _span("plan", e0)
            _run_rows(dm, plan, A, counts)
            global LAST_NEAR_ROWS
            LAST_NEAR_ROWS = np.zeros(n, dtype=np.int64)
            for cols, per in counts.get("near_rows", []):
                LAST_NEAR_ROWS[cols] += per
            if mesh.n_floating:
                rf = torch.as_tensor(mesh.row_float[rows].astype(np.int32), device=dev)
                ro = torch.as_tensor(off.astype(np.int64), device=dev)
                _lib.call("hvb_fill_float_cols", _lib.ptr(A), _lib.ptr(ro), _lib.ptr(rf), len(rows), n,
                          mesh.n_floating, _lib.stream_ptr(dev))
        for k in range(max(start, n), stop):
            adl, ids = _neutrality_scales(mesh, k - n)
            row = A[k - start]
            row[n:size] = 0.0
            if neutrality is not None:  # computed across ranks (parallel.assemble_distributed)
                row[:n] = neutrality[k - n]
            else:
                row[:n] = _weighted_adl_sum(mesh, dm, mesh.floating_collocation(k - n), adl, ids)
        if precision == "single":
            A = A.to(torch.float32)
    return A, counts


def _device_mesh(mesh, cfg, device):
    from .device import device_mesh

    return device_mesh(mesh, cfg, device)


def charge_row(mesh: SurfaceMesh, colloc_indices, eps_plus: float = EPS0, eps_minus: float | None = None,
               cfg: QuadConfig | None = None) -> np.ndarray:
    """q with q . u = charge through the given collocation set (reference
    src/assembly.py:540-569): weighted sum of ADL rows on the device."""
    import torch

    cfg = cfg or QuadConfig()
    if eps_minus is None:
        adl, ids = eps_plus, 0.5 * eps_plus
    else:
        adl, ids = eps_plus - eps_minus, 0.5 * (eps_plus + eps_minus)
    dm = _device_mesh(mesh, cfg, None)
    members = np.asarray(list(colloc_indices), dtype=np.int64)
    if len(members) == 0:
        return np.zeros(mesh.n_collocation)
    acc = _weighted_adl_sum(mesh, dm, members, adl, ids)
    return acc[dm.col_dev.long()].cpu().numpy()


def assemble_kernel_row(mesh, tables, x, vertex_id, kernel, n_x=None, cfg=None):
    """One full kernel row (reference src/assembly.py:295-301) on the device.
    KERNEL_E rows are three ADL rows with unit-vector normals."""
    import torch

    cfg = cfg or QuadConfig()
    if tables is not None and getattr(tables, "order", cfg.regular_order) != cfg.regular_order:
        cfg = QuadConfig(**{**cfg.__dict__, "regular_order": tables.order})
    dm = _device_mesh(mesh, cfg, None)
    dev = dm.device
    n = mesh.n_collocation
    x = np.asarray(x, dtype=np.float64)
    own = -1 if vertex_id is None else int(mesh.colloc_index[int(vertex_id)])
    if kernel == KERNEL_E:
        nrm = np.eye(3)
        kinds = np.ones(3, np.int64)
    elif kernel == KERNEL_ADL:
        nrm = np.asarray(n_x, dtype=np.float64)[None]
        kinds = np.ones(1, np.int64)
    else:
        nrm = np.zeros((1, 3))
        kinds = np.zeros(1, np.int64)
    m = len(kinds)
    lda = -(-n // LDA_ALIGN) * LDA_ALIGN
    A = torch.empty((m, lda), dtype=torch.float64, device=dev)
    plan = _plan(dev, np.repeat(x[None], m, 0), nrm, kinds, np.full(m, own), np.ones(m), np.zeros(m),
                 np.arange(m) * lda)
    counts = {"near": 0}
    _run_rows(dm, plan, A, counts)
    host = A[:, :n].cpu().numpy()
    rows = np.empty_like(host)
    rows[:, dm.tiling.perm] = host
    singular = 0 if own < 0 else int(mesh.vc_ptr[own + 1] - mesh.vc_ptr[own])
    near = counts["near"] // m
    c = {"regular": mesh.n_triangles - singular - near, "singular": singular, "near": near}
    if kernel == KERNEL_E:
        return rows.T.copy(), c
    return rows[0], c


# ---------------------------------------------------------------------------
# binary dump (reference src/assembly.py:576-609)
# ---------------------------------------------------------------------------

_MAGIC = b"HVBM\x01"


def save_matrix(matrix: SystemMatrix, path) -> None:
    first = matrix.blocks[0].data
    prec = 8 if first.dtype == np.float64 else 4
    with open(path, "wb") as fh:
        fh.write(_MAGIC)
        fh.write(struct.pack("<qqqq", matrix.size, matrix.n, matrix.n_floating, prec))
        fh.write(struct.pack("<q", len(matrix.blocks)))
        for b in matrix.blocks:
            fh.write(struct.pack("<qq", b.start, b.stop))
        for b in matrix.blocks:
            fh.write(np.ascontiguousarray(b.data).tobytes())


def load_matrix(path) -> SystemMatrix:
    with open(path, "rb") as fh:
        if fh.read(len(_MAGIC)) != _MAGIC:
            raise ValueError(f"{path}: not a matrix dump")
        size, n, n_fl, prec = struct.unpack("<qqqq", fh.read(32))
        dt = np.float64 if prec == 8 else np.float32
        (nb,) = struct.unpack("<q", fh.read(8))
        ranges = [struct.unpack("<qq", fh.read(16)) for _ in range(nb)]
        blocks = []
        for a, b in ranges:
            cnt = (b - a) * size
            data = np.frombuffer(fh.read(cnt * prec), dtype=dt).reshape(b - a, size).copy()
            blocks.append(RowBlock(a, b, data))
    return SystemMatrix(n=n, n_floating=n_fl, blocks=blocks)
