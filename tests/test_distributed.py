"""World-size-2 gloo tests (CPU) of the row-sharded solve: the all-gather
plumbing and the replicated GMRES recurrence give the single-process
answer.  The local block operator is a CPU stand-in here (the product path
uses hvb_gemv on CUDA)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, A, b, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2003_12663_b200.parallel import DistributedMatrix, RowGather, split_range
        from paper_2003_12663_b200.solver import SolverConfig, solve

        N = A.shape[0]
        a, e = split_range(N, world, rank)
        loc = torch.as_tensor(A[a:e])

        def apply(z, right, left):
            x = z / right if right is not None else z
            y = loc @ x
            return left * y if left is not None else y

        def rowmax_diag():
            rm = loc.abs().max(dim=1).values
            dg = torch.as_tensor(np.array([A[i, i] for i in range(a, e)]))
            return rm, dg

        g = RowGather(N)
        full = g(torch.arange(a, e, dtype=torch.float64))
        assert torch.equal(full, torch.arange(N, dtype=torch.float64))
        m = DistributedMatrix(N, 0, a, e, local_apply=apply, local_rowmax_diag=rowmax_diag,
                              device=torch.device("cpu"))
        sol = solve(m, b, SolverConfig(rel_tol=1e-12, restart=7, max_iters=400))
        out_q.put((rank, sol.u, sol.iterations))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N", [9, 40])
def test_distributed_gmres_matches_single(N):
    from oracle import hvb_oracle as ora

    rng = np.random.default_rng(N)
    A = rng.standard_normal((N, N)) + N * np.eye(N)
    A[::3] *= 1e-3  # badly row-scaled rows exercise equilibration
    b = rng.standard_normal(N)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, A, b, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    u0, it0 = res[0][1], res[0][2]
    np.testing.assert_array_equal(u0, res[1][1])  # replicated recurrence: identical on all ranks
    x, it, _ = ora.gmres(A, b, restart=7, rel_tol=1e-12, max_iters=400)
    assert np.max(np.abs(u0 - x)) <= 1e-10 * np.max(np.abs(x))
    assert abs(it0 - it) <= 1
