"""Row-block sharding over GPUs (one process per GPU, torch.distributed).

Reference: the only parallelism of hvbem is the contiguous row-block
partition (partition_rows, src/assembly.py:362-373) over a thread pool;
PAPER.md:203 distributes the same row blocks over GPUs.  Here block b of
``partition_rows(N, world)`` lives on rank b:

* assembly: each rank assembles its rows (no communication -- panels,
  rules and the column tiling are replicated);
* GMRES: every rank applies its row block to the replicated Krylov vector
  and the block results are all-gathered (NCCL over NVLink; gloo in the CPU
  tests) -- the only data-path collective.  Krylov basis, Hessenberg and
  Givens state are replicated and updated identically on every rank, so the
  solve needs no other communication and all ranks return the same u;
* fields / tracing: targets split per rank, no communication.
"""

from __future__ import annotations

import numpy as np

from .assembly import DeviceStore, _rowmax_diag, assemble_rows, device_matvec, partition_rows

__all__ = ["DistributedMatrix", "assemble_distributed", "RowGather", "split_range"]


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


class _DistOperator:
    def __init__(self, dmat):
        self.dm = dmat
        self.device = dmat.device
        self.size = dmat.size
        self.gather = RowGather(dmat.size, dmat.group)

    def apply(self, z, right=None, left=None):
        a, b = self.dm.start, self.dm.stop
        loc_left = None if left is None else left[a:b]
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

    def operator(self):
        return _DistOperator(self)


def assemble_distributed(mesh, cfg=None, group=None, precision: str = "double", device=None):
    """Assemble this rank's row block (rank r owns partition_rows(N, world)[r])."""
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
    A, counts = assemble_rows(mesh, dm, start, stop, precision)
    store = DeviceStore(A, n, size, dm.perm, dm.tiling.perm, row0=start)
    mat = DistributedMatrix(n, mesh.n_floating, start, stop, group=group, store=store)
    mat.diagnostics = {"rows": (start, stop), "pairs_near_singular_local": counts["near"]}
    rhs = np.concatenate([np.where(mesh.row_kind_code == 0, mesh.row_v0, 0.0), np.zeros(mesh.n_floating)])
    return mat, rhs
