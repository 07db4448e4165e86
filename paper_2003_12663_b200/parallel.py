"""Row-block sharding over GPUs (one process per GPU, torch.distributed).

Reference: the only parallelism of hvbem is the contiguous row-block
partition (partition_rows, src/assembly.py:362-373) over a thread pool;
PAPER.md:203 distributes the same row blocks over GPUs.  Here block b of
``partition_rows(N, world)`` lives on rank b:

* assembly: each rank assembles its rows (no communication -- panels,
  rules and the column tiling are replicated);
* GMRES: every rank applies its row block to the replicated Krylov vector
  and the block results are all-gathered -- the only data-path exchange.
  On the device path the GEMV's epilogue stores every row result straight
  into all ranks' replicated vectors through CUDA-IPC-mapped peer memory
  (PeerGather, csrc/peer.cu: NVLink stores + an epoch flag barrier); the
  NCCL all-gather (RowGather) remains for the one-off row scans, for
  HVB_PEER_GATHER=0, and when IPC is unavailable (gloo CPU tests).  Krylov basis, Hessenberg and
  Givens state are replicated and updated identically on every rank, so the
  solve needs no other communication and all ranks return the same u;
* fields / tracing: targets split per rank, no communication.
"""

from __future__ import annotations

import ctypes
import logging
import os

import numpy as np

from .assembly import DeviceStore, _rowmax_diag, assemble_rows, device_matvec, partition_rows

__all__ = ["DistributedMatrix", "assemble_distributed", "RowGather", "PeerGather", "split_range"]

logger = logging.getLogger(__name__)
LAST_GATHER = None  # "peer" or "nccl": the data-path exchange of the last distributed operator


def split_range(total: int, world: int, rank: int):
    return partition_rows(total, world)[rank]


class RowGather:
    """All-gather of row-block vectors whose block sizes differ by <= 1."""

    def __init__(self, total: int, group=None):
        import torch
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.ranges = partition_rows(total, self.world)
        self.maxlen = max(b - a for a, b in self.ranges)
        idx = np.concatenate([r * self.maxlen + np.arange(b - a) for r, (a, b) in enumerate(self.ranges)])
        self._idx_np = idx
        self._idx = {}
        self.total = total
        del torch

    def __call__(self, local):
        import torch
        import torch.distributed as dist

        dev = local.device
        # gloo (CPU tests, or several ranks sharing one GPU) gathers host copies
        host = local.is_cuda and dist.get_backend(self.group) == "gloo"
        gdev = torch.device("cpu") if host else dev
        pad = torch.zeros(self.maxlen, dtype=local.dtype, device=gdev)
        pad[: local.shape[0]] = local
        buf = torch.empty(self.world * self.maxlen, dtype=local.dtype, device=gdev)
        dist.all_gather_into_tensor(buf, pad, group=self.group)
        if host:
            buf = buf.to(dev)
        key = str(dev)
        if key not in self._idx:
            self._idx[key] = torch.as_tensor(self._idx_np, device=dev)
        return buf[self._idx[key]]


class _CudaArray:
    """Zero-copy torch view of raw device memory (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}


def _release_region(base, opened):
    """Finalizer of a PeerGather: unmap the peers' regions, free ours."""
    from . import _lib

    for p in opened:
        try:
            _lib.call("hvb_ipc_close", ctypes.c_void_p(p))
        except Exception:  # noqa: BLE001 - interpreter teardown
            pass
    try:
        _lib.call("hvb_ipc_free", ctypes.c_void_p(base))
    except Exception:  # noqa: BLE001
        pass


def _agree(ok: bool, group, device) -> bool:
    """True on every rank iff ``ok`` on every rank (all_reduce MIN)."""
    import torch
    import torch.distributed as dist

    on_dev = dist.get_backend(group) == "nccl"
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=device if on_dev else "cpu")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    return bool(flag.item())


class PeerGather:
    """Fused GEMV + all-gather over CUDA IPC peer memory (csrc/peer.cu).

    Every rank owns a cudaMalloc'd region -- two replicated N-vectors
    (alternating by epoch parity), a row of `world` epoch flags and the GEMV's
    CTA completion counter -- and maps every peer's region.  One matvec =
    hvb_gemv_bcast (each row result stored into all replicas over NVLink,
    the last CTA release-stores the epoch into every rank's flag row) +
    hvb_peer_wait (acquire); no NCCL call and no separate gather launch on
    the data path.  Build with ``PeerGather.create``: every rank takes the
    peer path or none does (the IPC setup outcome is agreed by all_reduce
    before anyone uses it); the region is released by a finalizer."""

    @classmethod
    def create(cls, total: int, group=None, device=None):
        import torch.distributed as dist

        from . import _lib

        self = cls.__new__(cls)
        self.group, self.device, self.total = group, device, total
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        vec_bytes = 8 * total
        self._vec_bytes = vec_bytes
        region = 2 * vec_bytes + 8 * self.world + 64
        base = ctypes.c_void_p()
        handle = None
        try:
            _lib.call("hvb_ipc_alloc", region, ctypes.byref(base))
            hb = _lib.lib().hvb_ipc_handle_bytes()
            handle = (ctypes.c_ubyte * hb)()
            _lib.call("hvb_ipc_handle", base, handle)
            ok = True
        except Exception as exc:  # noqa: BLE001 - reported, then agreed across ranks
            logger.warning("peer-memory region unavailable on rank %d (%s)", self.rank, exc)
            ok = False
        if not _agree(ok, group, device):
            if base.value:
                _release_region(base.value, [])
            return None
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(handle), group=group)
        bases, opened = [], []
        ok = True
        for r, hd in enumerate(handles):
            if r == self.rank:
                bases.append(base.value)
                continue
            buf = (ctypes.c_ubyte * len(hd)).from_buffer_copy(hd)
            p = ctypes.c_void_p()
            try:
                _lib.call("hvb_ipc_open", buf, ctypes.byref(p))
            except Exception as exc:  # noqa: BLE001
                logger.warning("rank %d cannot map rank %d's region (%s)", self.rank, r, exc)
                ok = False
                break
            bases.append(p.value)
            opened.append(p.value)
        if not _agree(ok, group, device):
            _release_region(base.value, opened)
            return None
        self._init_views(base.value, bases, opened)
        dist.barrier(group=group)  # every peer has mapped every region
        return self

    def _init_views(self, base, bases, opened):
        import weakref

        import torch

        vb = self._vec_bytes
        self._base = base
        i64 = dict(dtype=torch.int64, device=self.device)
        self.vec_ptrs = [torch.tensor([b + par * vb for b in bases], **i64) for par in (0, 1)]
        self.flag_ptrs = torch.tensor([b + 2 * vb for b in bases], **i64)
        self.my_flags = base + 2 * vb
        self.done_ptr = base + 2 * vb + 8 * self.world
        self.local = [torch.as_tensor(_CudaArray(base + par * vb, self.total), device=self.device) for par in (0, 1)]
        self.epoch = 0
        self._finalizer = weakref.finalize(self, _release_region, base, list(opened))

    def close(self):
        self._finalizer()

    def matvec(self, store, row0: int, z, right, left_local):
        """Full y = left .* A (z ./ right) from this rank's row block."""
        from . import _lib
        from .assembly import gather_operand

        xp = gather_operand(store, z, right)
        self.epoch += 1
        par = self.epoch & 1
        s = _lib.stream_ptr(self.device)
        _lib.call("hvb_gemv_bcast", _lib.ptr(store.A), store.lda, int(store.A.shape[0]), store.size, _lib.ptr(xp),
                  _lib.ptr(left_local), _lib.ptr(self.vec_ptrs[par]), self.world, row0, _lib.ptr(self.flag_ptrs),
                  self.rank, self.epoch, ctypes.c_void_p(self.done_ptr), s)
        _lib.call("hvb_peer_wait", ctypes.c_void_p(self.my_flags), self.world, self.epoch, s)
        return self.local[par].clone()


def _peer_gather_enabled() -> bool:
    return os.environ.get("HVB_PEER_GATHER", "1") != "0"


class _DistOperator:
    def __init__(self, dmat):
        self.dm = dmat
        self.device = dmat.device
        self.size = dmat.size
        self.gather = RowGather(dmat.size, dmat.group)
        self.peer = dmat.peer_gather()
        global LAST_GATHER
        LAST_GATHER = "peer" if self.peer is not None else "collective"

    def apply(self, z, right=None, left=None):
        a, b = self.dm.start, self.dm.stop
        loc_left = None if left is None else left[a:b]
        if self.peer is not None:
            return self.peer.matvec(self.dm.store, a, z, right, loc_left)
        y = self.dm.local_apply(z, right, loc_left)
        return self.gather(y)

    def rowmax_diag(self):
        rm, dg = self.dm.local_rowmax_diag()
        return self.gather(rm), self.gather(dg)


class DistributedMatrix:
    """This rank's row block of the system plus the collective plumbing.
    Quacks like a SystemMatrix for solver.solve (``operator()``)."""

    def __init__(self, n, n_floating, start, stop, group=None, store: DeviceStore | None = None,
                 local_apply=None, local_rowmax_diag=None, device=None):
        self.n = n
        self.n_floating = n_floating
        self.start = start
        self.stop = stop
        self.group = group
        self.store = store
        self.device = store.A.device if store is not None else device
        self._apply = local_apply
        self._rowmax = local_rowmax_diag
        self.diagnostics: dict = {}

    @property
    def size(self) -> int:
        return self.n + self.n_floating

    @property
    def shape(self):
        return (self.size, self.size)

    def local_apply(self, z, right, left):
        if self._apply is not None:
            return self._apply(z, right, left)
        return device_matvec(self.store, z, right=right, left=left)

    def local_rowmax_diag(self):
        if self._rowmax is not None:
            return self._rowmax()
        return _rowmax_diag(self.store)

    def peer_gather(self):
        """The matrix's PeerGather (built once, on the first solve), or None
        when every rank agreed on the NCCL all-gather (HVB_PEER_GATHER=0,
        float32 storage, CPU operator, or IPC setup failed on some rank)."""
        if not hasattr(self, "_peer"):
            st = self.store
            usable = (_peer_gather_enabled() and st is not None and not st.is_f32 and self._apply is None
                      and self.device is not None and self.device.type == "cuda")
            # every rank evaluates the same conditions; create() agrees on IPC itself
            self._peer = PeerGather.create(self.size, self.group, self.device) if usable else None
        return self._peer

    def operator(self):
        return _DistOperator(self)


def _distributed_neutrality(mesh, dm, group, start: int, stop: int):
    """Neutrality rows n+k of floating surfaces (reference _row_equation
    src/assembly.py:441-468) with their member ADL rows spread over the
    ranks: member chunk c of surface k goes to rank c mod world, the chunk
    partials are all-gathered and the owner of row n+k adds them in chunk
    order -- bitwise the single-process row (assembly._weighted_adl_sum)."""
    import torch
    import torch.distributed as dist

    from .assembly import NEUTRALITY_CHUNK, _neutrality_scales, adl_chunk_sum

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = mesh.n_collocation
    out = {}
    for k in range(mesh.n_floating):
        members = mesh.floating_collocation(k)
        adl, ids = _neutrality_scales(mesh, k)
        chunks = [members[c0:c0 + NEUTRALITY_CHUNK] for c0 in range(0, len(members), NEUTRALITY_CHUNK)]
        per = -(-len(chunks) // world)
        mine = torch.zeros((per, n), dtype=torch.float64, device=dm.device)
        for j, c in enumerate(range(rank, len(chunks), world)):
            mine[j] = adl_chunk_sum(mesh, dm, chunks[c], adl, ids)
        host = dist.get_backend(group) == "gloo"
        send = mine.cpu() if host else mine
        buf = torch.empty((world * per, n), dtype=torch.float64, device=send.device)
        dist.all_gather_into_tensor(buf, send, group=group)
        if start <= n + k < stop:
            buf = buf.to(dm.device)
            acc = torch.zeros(n, dtype=torch.float64, device=dm.device)
            for c in range(len(chunks)):  # chunk order: rank c % world, slot c // world
                acc += buf[(c % world) * per + c // world]
            out[k] = acc
    return out


def assemble_distributed(mesh, cfg=None, group=None, precision: str = "double", device=None):
    """Assemble this rank's row block (rank r owns partition_rows(N, world)[r]);
    neutrality rows are computed across all ranks (_distributed_neutrality)."""
    import torch.distributed as dist

    from .assembly import _device_mesh
    from .quadrature import QuadConfig

    cfg = cfg or QuadConfig()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = mesh.n_collocation
    size = n + mesh.n_floating
    start, stop = split_range(size, world, rank)
    dm = _device_mesh(mesh, cfg, device)
    neutrality = _distributed_neutrality(mesh, dm, group, start, stop) if mesh.n_floating else None
    A, counts = assemble_rows(mesh, dm, start, stop, precision, neutrality=neutrality)
    store = DeviceStore(A, n, size, dm.perm, dm.tiling.perm, row0=start)
    mat = DistributedMatrix(n, mesh.n_floating, start, stop, group=group, store=store)
    mat.diagnostics = {"rows": (start, stop), "pairs_near_singular_local": counts["near"]}
    rhs = np.concatenate([np.where(mesh.row_kind_code == 0, mesh.row_v0, 0.0), np.zeros(mesh.n_floating)])
    return mat, rhs
