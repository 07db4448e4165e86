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


def _gpu_worker(rank, world, port, out_q, peer="1"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["HVB_PEER_GATHER"] = peer
    dist.init_process_group("gloo", rank=rank, world_size=world)  # ranks share cuda:0 here
    try:
        torch.cuda.set_device(0)
        from paper_2003_12663_b200 import fixtures
        from paper_2003_12663_b200.parallel import assemble_distributed, split_range
        from paper_2003_12663_b200.postprocess import eval_efield_batch, trace_fieldlines
        from paper_2003_12663_b200.solver import SolverConfig, solve

        m = fixtures.concentric_mesh(2, [(0.5, "electrode 1.0"), (1.0, "electrode 0.0")])
        A, rhs = assemble_distributed(m)
        sol = solve(A, rhs, SolverConfig(rel_tol=1e-12))
        P = np.array([[0.7, 0.1, 0.05], [0.1, 0.6, 0.2], [0.0, 0.0, 0.8], [0.55, 0.2, -0.3]])
        a, b = split_range(len(P), world, rank)
        E = eval_efield_batch(sol, m, P[a:b])
        starts = np.array([[0.55, 0.0, 0.0], [0.0, 0.6, 0.0], [0.0, 0.0, -0.7]])
        la, lb = split_range(len(starts), world, rank)
        lines = trace_fieldlines(sol, m, starts[la:lb], [1] * (lb - la))
        from paper_2003_12663_b200 import parallel

        out_q.put((rank, sol.u, sol.iterations, E, [ln.points for ln in lines], parallel.LAST_GATHER))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
def test_row_sharded_device_path_matches_single_process():
    """World-size 2 (gloo; both ranks on cuda:0) through the real device
    path: row-block assembly, GMRES with the fused GEMV + peer-memory
    all-gather (CUDA IPC), points and lines split per rank -- the
    single-process results."""
    from paper_2003_12663_b200 import fixtures
    from paper_2003_12663_b200.assembly import assemble
    from paper_2003_12663_b200.postprocess import eval_efield_batch, trace_fieldlines
    from paper_2003_12663_b200.solver import SolverConfig, solve

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    m = fixtures.concentric_mesh(2, [(0.5, "electrode 1.0"), (1.0, "electrode 0.0")])
    A, rhs = assemble(m)
    sol = solve(A, rhs, SolverConfig(rel_tol=1e-12))
    P = np.array([[0.7, 0.1, 0.05], [0.1, 0.6, 0.2], [0.0, 0.0, 0.8], [0.55, 0.2, -0.3]])
    E = eval_efield_batch(sol, m, P)
    starts = np.array([[0.55, 0.0, 0.0], [0.0, 0.6, 0.0], [0.0, 0.0, -0.7]])
    lines = trace_fieldlines(sol, m, starts, [1, 1, 1])
    for r in res:
        assert r[5] == "peer"  # fused GEMV + peer-memory all-gather (csrc/peer.cu)
        np.testing.assert_allclose(r[1], sol.u, rtol=0, atol=1e-13 * np.max(np.abs(sol.u)))
        assert abs(r[2] - sol.iterations) <= 1
    np.testing.assert_allclose(np.vstack([r[3] for r in res]), E, rtol=1e-12, atol=1e-14)
    got = [pts for r in res for pts in r[4]]
    assert len(got) == len(lines)
    for g, ln in zip(got, lines):
        assert g.shape == ln.points.shape
        np.testing.assert_allclose(g, ln.points, rtol=0, atol=1e-10)


def _run_pair(target, *extra):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, 2, port, q, *extra)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
def test_peer_gather_equals_nccl_gather_bitwise():
    """The fused GEMV + peer-memory all-gather (release/acquire epoch flags,
    csrc/peer.cu) and the collective all-gather path (HVB_PEER_GATHER=0)
    give bitwise-identical solves, fields and lines (2 ranks on cuda:0)."""
    peer = _run_pair(_gpu_worker, "1")
    coll = _run_pair(_gpu_worker, "0")
    assert [r[5] for r in peer] == ["peer", "peer"] and [r[5] for r in coll] == ["collective", "collective"]
    for a, b in zip(peer, coll):
        np.testing.assert_array_equal(a[1], b[1])
        assert a[2] == b[2]
        np.testing.assert_array_equal(a[3], b[3])
        for pa, pb in zip(a[4], b[4]):
            np.testing.assert_array_equal(pa, pb)


def _float_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from conftest import build_case
        from paper_2003_12663_b200 import assembly
        from paper_2003_12663_b200.parallel import assemble_distributed

        assembly.NEUTRALITY_CHUNK = 16  # several chunks per surface, spread over both ranks
        m = build_case("cfg3mini")
        A, rhs = assemble_distributed(m)
        n = m.n_collocation
        row = A.store.host_rows(n - A.start, n - A.start + 1)[0] if A.start <= n < A.stop else None
        out_q.put((rank, row))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
def test_distributed_neutrality_row_bitwise():
    """The neutrality row's member ADL rows are split over the ranks and
    recombined in chunk order: bitwise the single-process row."""
    from conftest import build_case
    from paper_2003_12663_b200 import assembly

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_float_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    rows = [r[1] for r in res if r[1] is not None]
    assert len(rows) == 1
    old = assembly.NEUTRALITY_CHUNK
    assembly.NEUTRALITY_CHUNK = 16
    try:
        m = build_case("cfg3mini")
        A, _ = assembly.assemble(m)
        ref = A.row(m.n_collocation)
    finally:
        assembly.NEUTRALITY_CHUNK = old
    np.testing.assert_array_equal(rows[0], ref)
