#!/usr/bin/env python
"""Benchmark of the indirect-BEM hot path on config 4 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU)

Workload (configs[3] of BASELINE.json, the metric's config): the synthetic
disconnector-like rod-plane + insulator mesh, 199,104 curved panels,
N = 99,558 unknowns, dense FP64 system 79 GB (> L2, so no flush needed).
One step = one pass of the hot path: assemble the dense system (this rank's
row block), GMRES solve (reference semantics, rel_tol 1e-8; matvec row-block
sharded + NCCL all-gather), E at M field points (points split per rank),
and config 5 on the step's own solution: surface |E|, the top ``--lines``
seeds, device RK45 field lines with the streamer verdict (lines split per
rank).  Inputs are resident in HBM for the device-timed value; the ``e2e``
leg re-runs the pass through the public API from host buffers (mesh arrays
H2D, u and E D2H inside the timed region).

Prints ONE JSON line (rank 0).  ``value`` = assembly entries/s (N^2 / max
over ranks of the assembly time); GMRES solve seconds and field evals/s are
reported beside it; the full config-5 trace (every collocation vertex seeded,
~1e5 lines) is timed once after the steps (``trace_full``).

``--impl reference`` times the reference's OWN implementation, hvbem 0.1.0
as installed unmodified into baseline/_ref (pip --target), on
the box's host cores: per step, reference ``_row_equation`` on a bounded
sample of evenly spaced config-4 rows over a fork pool of every core
(entries/s = rows x N / time); once, the reference ``matvec`` on a row-block
sample and ``eval_efield`` at one point per core.  When baseline/_ref is
missing it falls back to the oracle port (oracle/, kind "port").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "assembly entries/s; GMRES solve s; field evals/s at N=200k panels, 1-8 B200"
E2E_REPS = 3


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--scale", type=float, default=1.0, help="mesh resolution scale (1.0 = config 4)")
    ap.add_argument("--points", type=int, default=100_000, help="field points per step (whole job)")
    ap.add_argument("--lines", type=int, default=8192, help="cfg5 field lines per step (whole job; 0 = skip)")
    ap.add_argument("--uniform-points", type=int, default=1_000_000,
                    help="SURVEY 8d uniform field workload, timed once (0 = skip)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-full-trace", dest="full_trace", action="store_false",
                    help="skip the once-per-run config-5 trace of every vertex (~1e5 lines)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--cpu-rows", type=int, default=24, help="cpu_baseline sample rows")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.idx)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[5 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_copy_gbs():
    """The driver-measured copy bandwidth (MEASURED_PEAKS.json hbm_gbs)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return None


def measure_peaks(dev, sustained_s: float = 3.0):
    """DFMA throughput and read-stream bandwidth of this GPU (denominators).
    DFMA: the burst figure (a 6 ms launch, best of 3) and the sustained one
    (launches back to back for ``sustained_s`` seconds, the rate of the
    second half: the power cap has engaged) -- the sweep, the field
    workloads and the tracer run inside a multi-second step, so their
    fractions use the sustained figure (MEASURED_PEAKS.json's convention)."""
    import torch

    from paper_2003_12663_b200 import _lib

    st = _lib.stream_ptr(dev)
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    blocks, iters = 148 * 16, 3000
    _lib.call("hvb_bench_dfma", _lib.ptr(out), blocks, 100, st)
    flop = 2.0 * 64 * 256 * blocks
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("hvb_bench_dfma", _lib.ptr(out), blocks, iters, st)
        e1.record()
        torch.cuda.synchronize(dev)
        best = max(best, flop * iters / (e0.elapsed_time(e1) / 1e3))
    sustained = best
    if sustained_s > 0:
        it_long = 10 * iters  # ~65 ms per launch
        n_launch = max(2, int(round(sustained_s / (flop * it_long / best))))
        half = n_launch // 2
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for k in range(n_launch):
            if k == half:
                e0.record()
            _lib.call("hvb_bench_dfma", _lib.ptr(out), blocks, it_long, st)
        e1.record()
        torch.cuda.synchronize(dev)
        sustained = flop * it_long * (n_launch - half) / (e0.elapsed_time(e1) / 1e3)
    best = (best, sustained)
    buf = torch.ones(2 ** 30, dtype=torch.float64, device=dev)  # 8 GiB
    bw = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("hvb_bench_read", _lib.ptr(buf), buf.numel(), _lib.ptr(out), 148 * 64, st)
        e1.record()
        torch.cuda.synchronize(dev)
        bw = max(bw, buf.numel() * 8 / (e0.elapsed_time(e1) / 1e3))
    del buf
    return best[0] / 1e12, best[1] / 1e12, bw / 1e9


def regular_flops(mesh, near_rows_counts, sl_rows, adl_rows):
    """Algorithmic FLOPs of the regular sweep: per row 9*nt for
    the classification + 12 nodes x (17 SL | 23 ADL) per regular pair."""
    nt = mesh.n_triangles
    star = mesh.vc_ptr[1:] - mesh.vc_ptr[:-1]
    reg = nt - star - near_rows_counts
    return float(9.0 * nt * (len(sl_rows) + len(adl_rows)) + 12 * 17 * reg[sl_rows].sum()
                 + 12 * 23 * reg[adl_rows].sum())


# ---------------------------------------------------------------------------
# reference arm / cpu baseline (oracle port on the host cores)
# ---------------------------------------------------------------------------

_CPU_MESH = None


_CPU_TABLES = None


_PARENT_PID = os.getpid()


def _one_thread():
    """Forked sample workers: one BLAS thread each (no oversubscription);
    a no-op in the parent process."""
    if os.getpid() == _PARENT_PID:
        return
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except ImportError:  # pragma: no cover
        pass


def _cpu_rows(rows):
    from oracle import hvb_oracle as ora

    _one_thread()
    t = time.perf_counter()
    ora.row_equations(_CPU_MESH, rows, tables=_CPU_TABLES)
    return time.perf_counter() - t


def cpu_sample(mesh, n_rows: int, processes: int, field_points: int = 4):
    """Time the oracle port on evenly spaced rows (+ a GEMV block and a few
    field points) and extrapolate to the full workload."""
    import multiprocessing as mp

    import numpy as np

    from oracle import hvb_oracle as ora

    global _CPU_MESH, _CPU_TABLES
    if _CPU_MESH is not mesh:
        _CPU_MESH = mesh
        # per-mesh sample tables, built once before forking (the reference
        # caches them per mesh too, src/mesh.py:343-352)
        _CPU_TABLES = ora.Tables(mesh, ora.DEFAULT_CFG["regular_order"])
    N = mesh.n_collocation + mesh.n_floating
    rows = np.linspace(0, mesh.n_collocation - 1, n_rows).astype(int)
    chunks = [rows[i::processes].tolist() for i in range(processes)]
    chunks = [c for c in chunks if c]
    t0 = time.perf_counter()
    if processes > 1:
        with mp.get_context("fork").Pool(len(chunks)) as pool:
            pool.map(_cpu_rows, chunks)
    else:
        _cpu_rows(rows.tolist())
    t_rows = time.perf_counter() - t0
    entries_per_s = n_rows * N / t_rows
    # GEMV: numpy BLAS over a row block (all BLAS threads)
    blk = np.random.default_rng(0).standard_normal((min(4096, N), N))
    v = np.random.default_rng(1).standard_normal(N)
    blk @ v
    t0 = time.perf_counter()
    for _ in range(3):
        blk @ v
    t_mv = (time.perf_counter() - t0) / 3 * (N / blk.shape[0])
    del blk
    # field evaluation: one point per process (embarrassingly parallel)
    rng = np.random.default_rng(0)
    lo, hi = mesh.bounding_box()
    P = 0.5 * (lo + hi) + rng.uniform(-0.6, 0.6, (field_points, 3)) * (hi - lo)
    t0 = time.perf_counter()
    if processes > 1 and field_points > 1:
        with mp.get_context("fork").Pool(min(processes, field_points)) as pool:
            pool.map(_cpu_field, [P[i:i + 1] for i in range(field_points)])
    else:
        _cpu_field(P)
    evals_per_s = field_points / (time.perf_counter() - t0)
    return {
        "entries_per_s": entries_per_s,
        "t_rows": t_rows,
        "matvec_s": t_mv,
        "field_evals_per_s": evals_per_s,
        "sample": (f"oracle port: {n_rows} evenly spaced cfg4 rows (row_equations, {processes} procs) "
                   f"-> entries/s x N; numpy GEMV on a 4096-row block; E at {field_points} points "
                   f"({min(processes, field_points)} procs)"),
    }


def _cpu_field(P):
    import numpy as np

    from oracle import hvb_oracle as ora

    _one_thread()
    ora.efield_points(_CPU_MESH, np.ones(_CPU_MESH.n_collocation), P)


REF_DIR = os.path.join(ROOT, "baseline", "_ref")
_REF = {}


def _ref_rows(rows):
    """Forked worker: the reference's own _row_equation on `rows`."""
    _one_thread()
    ra, cfg, mesh, tab = _REF["assembly"], _REF["cfg"], _REF["mesh"], _REF["tables"]
    t = time.perf_counter()
    for r in rows:
        ra._row_equation(mesh, cfg, tab, int(r))
    return time.perf_counter() - t


def _ref_field(x):
    _one_thread()
    t = time.perf_counter()
    _REF["post"].eval_efield(_REF["solution"], _REF["mesh"], x, _REF["cfg"])
    return time.perf_counter() - t


def _load_reference(scale):
    """The reference package from baseline/_ref and its own parse of the
    config-4 mesh (text written by our generator, parsed by hvbem.mesh)."""
    import importlib

    import numpy as np

    sys.path.insert(0, REF_DIR)
    try:
        rmesh = importlib.import_module("hvbem.mesh")
        ra = importlib.import_module("hvbem.assembly")
        rpost = importlib.import_module("hvbem.postprocess")
        rsol = importlib.import_module("hvbem.solver")
        rq = importlib.import_module("hvbem.quadrature")
    finally:
        sys.path.pop(0)
    if not os.path.dirname(os.path.abspath(rmesh.__file__)).startswith(REF_DIR):
        raise ImportError("hvbem imported from outside baseline/_ref")
    from paper_2003_12663_b200 import fixtures

    v, ids, tags, lines = fixtures.rod_plane_parts(scale)
    t0 = time.perf_counter()
    text = fixtures.mesh_text(v, [(tuple(r), int(g)) for r, g in zip(ids.tolist(), tags.tolist())], lines)
    mesh = rmesh.parse_mesh(text)
    cfg = rq.QuadConfig()
    tab = mesh.tables(cfg.regular_order)
    _REF.update(assembly=ra, post=rpost, mesh=mesh, cfg=cfg, tables=tab,
                solution=rsol.Solution(u=np.ones(mesh.n_collocation), V=np.zeros(0), iterations=0, residual=0.0),
                setup_s=time.perf_counter() - t0, matvec=ra.matvec, RowBlock=ra.RowBlock, SystemMatrix=ra.SystemMatrix)
    return mesh


def reference_sample(mesh, cores: int, warmup: int, steps: int):
    """The reference's own code on the host cores (fork pool, one BLAS
    thread per process): entries/s of _row_equation on 2 x cores evenly
    spaced rows per step (median of `steps` after `warmup`), eval_efield at
    one point per core, and one reference matvec on a row-block sample
    extrapolated to N rows."""
    import multiprocessing as mp

    import numpy as np

    n = mesh.n_collocation
    N = n + mesh.n_floating
    per_step = 2 * cores                       # rows per step: ~0.1 s of CPU work per row at config 4
    vals = []
    with mp.get_context("fork").Pool(cores) as pool:
        for k in range(warmup + steps):
            rows = np.minimum(np.linspace(0, n - 1, per_step).astype(int) + k % 7, n - 1)
            t0 = time.perf_counter()
            pool.map(_ref_rows, [rows[i::cores].tolist() for i in range(cores)])
            dt = time.perf_counter() - t0
            if k >= warmup:
                vals.append(per_step * N / dt)
        # field evaluation: one point per core (reference eval_efield)
        rng = np.random.default_rng(0)
        lo, hi = mesh.vertices.min(axis=0), mesh.vertices.max(axis=0)
        P = 0.5 * (lo + hi) + rng.uniform(-0.6, 0.6, (cores, 3)) * (hi - lo)
        t0 = time.perf_counter()
        pool.map(_ref_field, list(P))
        evals_per_s = cores / (time.perf_counter() - t0)
    # GMRES matvec: the reference's matvec on a row-block sample, blocks over
    # its own thread pool (workers = cores), extrapolated to N rows
    rows_blk = min(N, 64 * cores)
    blocks = [_REF["RowBlock"](a, b, np.random.default_rng(a).standard_normal((b - a, N)))
              for a, b in _partition(rows_blk, cores)]
    mat = _REF["SystemMatrix"](n=N, n_floating=0, blocks=blocks)
    x = np.random.default_rng(1).standard_normal(N)
    _REF["matvec"](mat, x, workers=cores)
    t0 = time.perf_counter()
    _REF["matvec"](mat, x, workers=cores)
    matvec_s = (time.perf_counter() - t0) * N / rows_blk
    del blocks, mat
    return {"entries_per_s": float(np.median(vals)), "field_evals_per_s": evals_per_s, "matvec_s": matvec_s,
            "sample": (f"hvbem 0.1.0 from baseline/_ref: _row_equation on {per_step} evenly spaced cfg4 rows per "
                       f"step over {cores} forked processes (entries/s = rows x N / time, median of {steps}); "
                       f"matvec on a {rows_blk}-row block (workers={cores}) x N/{rows_blk}; eval_efield at "
                       f"{cores} points (one per process)")}


def run_reference(args):
    """--impl reference: the reference's own code (baseline/_ref) on the host
    cores; the oracle port stands in only if baseline/_ref is missing."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    try:
        mesh = _load_reference(args.scale)
    except ImportError as exc:
        sys.stderr.write(f"baseline/_ref unavailable ({exc}); timing the oracle port\n")
        return _run_port_reference(args, cores)
    N = mesh.n_collocation + mesh.n_floating
    smp = reference_sample(mesh, cores, args.warmup, args.steps)
    v = smp["entries_per_s"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "entries/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": N * N / v * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (deterministic rod-plane generator; mesh parsed by the reference's own parse_mesh)",
        "config": {"workload": f"cfg4 rod-plane+insulator: {mesh.n_triangles} panels, N={N}",
                   "panels": mesh.n_triangles, "N": N},
        "gmres_solve_s": None,
        "gmres_matvec_s": smp["matvec_s"],
        "field_evals_per_s": smp["field_evals_per_s"],
        "reference_setup_s": _REF["setup_s"],
        "cpu_baseline": {"value": v, "unit": "entries/s", "cores": cores, "kind": "reference",
                         "sample": smp["sample"]},
        "e2e": {"value": v, "unit": "entries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": ("extrapolated from row samples: the full cfg4 system is 79 GB (no CPU assembly or GMRES solve "
                 "at this size; gmres_matvec_s is one reference matvec, iterations are set by the matrix)"),
    }
    print(json.dumps(line), flush=True)


def _partition(total, parts):
    q, r = divmod(total, parts)
    out, a = [], 0
    for b in range(parts):
        e = a + q + (1 if b < r else 0)
        if e > a:
            out.append((a, e))
        a = e
    return out


def _run_port_reference(args, cores):
    import numpy as np

    from paper_2003_12663_b200 import fixtures

    mesh = fixtures.rod_plane_mesh(args.scale)
    N = mesh.n_collocation + mesh.n_floating
    vals, samp = [], None
    for k in range(args.warmup + args.steps):
        s = cpu_sample(mesh, max(4 * cores, args.cpu_rows), cores, field_points=max(2, cores))
        if k >= args.warmup:
            vals.append(s)
        samp = s
    v = float(np.median([s["entries_per_s"] for s in vals]))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "entries/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": N * N / v * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (deterministic rod-plane generator)",
        "config": {"workload": f"cfg4 rod-plane+insulator: {mesh.n_triangles} panels, N={N}",
                   "panels": mesh.n_triangles, "N": N},
        "gmres_solve_s": None,
        "gmres_matvec_s": float(np.median([s["matvec_s"] for s in vals])),
        "field_evals_per_s": float(np.median([s["field_evals_per_s"] for s in vals])),
        "cpu_baseline": {"value": v, "unit": "entries/s", "cores": cores, "kind": "port", "sample": samp["sample"]},
        "e2e": {"value": v, "unit": "entries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "baseline/_ref missing: the oracle port (oracle/hvb_oracle.py) stands in for the reference",
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------


def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # HVB_DIST_BACKEND=gloo lets several ranks share one GPU (validation of
    # the multi-rank path on a 1-GPU box); production is NCCL, one GPU per rank
    backend = os.environ.get("HVB_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend == "gloo" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    import __graft_entry__

    __graft_entry__.build()
    from paper_2003_12663_b200 import _lib, assembly, device, fixtures, parallel, postprocess, tracer
    from paper_2003_12663_b200.quadrature import QuadConfig
    from paper_2003_12663_b200.assembly import assemble
    from paper_2003_12663_b200.device import device_mesh
    from paper_2003_12663_b200.parallel import assemble_distributed, split_range
    from paper_2003_12663_b200.solver import SolverConfig, solve

    tflops_burst, tflops_peak, read_gbs = measure_peaks(dev)
    copy_gbs = measured_copy_gbs()
    t_mb = time.perf_counter()
    mesh = fixtures.rod_plane_mesh(args.scale)
    mesh_build_s = time.perf_counter() - t_mb
    n, nt = mesh.n_collocation, mesh.n_triangles
    N = n + mesh.n_floating
    rng = np.random.default_rng(1234)
    lo, hi = mesh.bounding_box()
    P_all = 0.5 * (lo + hi) + rng.uniform(-0.6, 0.6, (args.points, 3)) * (hi - lo)
    pa, pb = split_range(args.points, world, rank)
    P_dev = torch.as_tensor(P_all[pa:pb], device=dev)
    cfg_solver = SolverConfig()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    counter = {"n": 0}
    orig_call = _lib.call

    # kernels launched per C-ABI call (1 unless listed)
    per_call = {"hvb_trace_round": 8}  # flag reset, N-body, split reduce, near pass, counter reset, ctrl, SD, ctrl

    def counting_call(name, *a):
        if not name.startswith("hvb_bench"):
            counter["n"] += per_call.get(name, 1)
        return orig_call(name, *a)

    _lib.call = counting_call

    gas = postprocess.load_ionization_model(os.path.join(ROOT, "paper_2003_12663_b200", "data", "air_demo.gas"))
    trace_stats = {}

    def trace_phase(sol):
        """cfg5: seeds = top-k surface |E| (orientation sign(E.n), the CLI's
        rule), lines split per rank, device tracer + streamer verdicts."""
        if args.lines <= 0:
            return
        if world > 1:  # each rank its share of the vertices, all-gathered (n doubles)
            ia, ib = split_range(n, world, rank)
            part = torch.as_tensor(postprocess.surface_field_magnitudes(mesh, sol, indices=np.arange(ia, ib)),
                                   device=dev)
            se = parallel.RowGather(n)(part).cpu().numpy()
        else:
            se = postprocess.surface_field_magnitudes(mesh, sol)
        starts, idx, _ = postprocess.pick_start_points(mesh, sol, args.lines, surface_e=se)
        la, lb = split_range(len(starts), world, rank)
        E0 = postprocess.eval_efield_batch(sol, mesh, starts[la:lb])
        orient = np.where(np.einsum("ij,ij->i", E0, mesh.colloc_normals[idx[la:lb]]) >= 0, 1, -1)
        res = tracer.trace_device(sol, mesh, starts[la:lb], orient, postprocess.TraceParams(), QuadConfig())
        val, ver = tracer.streamer_device(res, gas)
        trace_stats.update(rounds=res.rounds, evals=res.field_points, lines=lb - la,
                           accepted=int((res.info[:, 0] - 1).sum()) if lb > la else 0,
                           inception=int(ver.sum().item()),
                           terms=np.bincount(res.info[:, 1], minlength=4).tolist(),
                           max_points=int(res.info[:, 0].max()) if lb > la else 0)

    def one_step(profile=None):
        assembly.PROFILE = profile
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record()
        if world > 1:
            A, rhs = assemble_distributed(mesh)
        else:
            A, rhs = assemble(mesh)
        ev[1].record()
        assembly.PROFILE = None
        sol = solve(A, rhs, cfg_solver)
        ev[2].record()
        dm = device_mesh(mesh)
        u_dev, key = postprocess._u_device(sol, dm)
        src = postprocess._sources(dm, u_dev, key)
        E = postprocess.field_points_device(dm, u_dev, src, P_dev, False)
        ev[3].record()
        del A, E
        trace_phase(sol)
        ev[4].record()
        torch.cuda.synchronize(dev)
        ph = [ev[i].elapsed_time(ev[i + 1]) / 1e3 for i in range(4)]
        return ph, sol

    device_mesh(mesh)  # per-mesh setup (tables, tiling, panel streams) outside the timed region
    for _ in range(args.warmup):
        one_step()
    barrier()
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    counter["n"] = 0
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    barrier()
    t_start.record()
    phases = []
    step_spans = []  # every timed step's assembly spans (CUDA events on the launching stream)
    iters = 0
    for k in range(args.steps):
        prof = []
        ph, sol = one_step(prof)
        step_spans.append(prof)
        phases.append(ph)
        iters = sol.iterations
    t_end.record()
    barrier()
    if sampler:
        sampler.stop()
    launches = counter["n"]
    total = t_start.elapsed_time(t_end) / 1e3
    ph = np.array(phases).mean(axis=0)
    # the regular sweep's average time per step over the timed region (its
    # SL + ADL launches), for the roofline
    reg_steps = [sum(e0.elapsed_time(e1) for lab, e0, e1 in sp if lab == "regular") / 1e3 for sp in step_spans]
    reg_t = float(np.mean(reg_steps))
    if os.environ.get("HVB_BENCH_SPANS"):  # dev: per-step phases and assembly spans
        for k, sp in enumerate(step_spans):
            print(f"step {k}: phases {[round(x, 4) for x in phases[k]]} spans "
                  f"{[(lab, round(e0.elapsed_time(e1), 2)) for lab, e0, e1 in sp]}", file=sys.stderr)
    vec = torch.tensor([total, ph[0], ph[1], ph[2], ph[3], reg_t], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vec, op=dist.ReduceOp.MAX)
    total, t_asm, t_solve, t_field, t_trace, reg_t = vec.tolist()
    tvec = torch.tensor([trace_stats.get("evals", 0), trace_stats.get("inception", 0)], dtype=torch.float64,
                        device=dev)
    if world > 1:
        dist.all_reduce(tvec)
    trace_evals, trace_inception = tvec.tolist()

    # algorithmic flops of this rank's regular sweep (max-over-ranks time -> rank-0 share x world)
    a, b = split_range(N, world, rank)
    rows = np.arange(a, min(b, n))
    near_rows = np.zeros(n, dtype=np.int64)
    kinds = mesh.row_kind_code[rows]
    sl_rows = rows[kinds != 2]
    adl_rows = rows[kinds == 2]
    near_total = _count_near(mesh, rows)
    near_rows[rows] = near_total
    flops = regular_flops(mesh, near_rows, sl_rows, adl_rows)
    achieved = flops / reg_t / 1e12 if reg_t > 0 else 0.0

    # near-surface field evaluation: every collocation point
    # offset by 0.25 of its local circumradius along the normal -- ~6 deferred
    # near-singular panels per point (composite rules of 512-3,072 nodes)
    na, nb = split_range(n, world, rank)
    _, loc_r = postprocess.surface_distance_batch(mesh, mesh.colloc_points[na:nb])
    P_near = torch.as_tensor(mesh.colloc_points[na:nb] + (0.25 * loc_r)[:, None] * mesh.colloc_normals[na:nb],
                             device=dev)
    dmn = device_mesh(mesh)
    u_dev, key = postprocess._u_device(sol, dmn)
    src = postprocess._sources(dmn, u_dev, key)
    postprocess.field_points_device(dmn, u_dev, src, P_near[:1024], False)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    En = postprocess.field_points_device(dmn, u_dev, src, P_near, False)
    f1.record()
    torch.cuda.synchronize(dev)
    near_pairs_per_point = float(En.near_pairs) / max(1, len(P_near))
    fvec = torch.tensor([f0.elapsed_time(f1) / 1e3], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(fvec, op=dist.ReduceOp.MAX)
    t_near = float(fvec.item())
    del En, P_near

    # SURVEY 8d's uniform field workload at its size: 1e6 points in the 1.2x
    # bounding box (seed 0), split per rank, timed once
    n_uni = args.uniform_points
    field_uniform = None
    if n_uni > 0:
        P_u = 0.5 * (lo + hi) + np.random.default_rng(0).uniform(-0.6, 0.6, (n_uni, 3)) * (hi - lo)
        ua, ub = split_range(n_uni, world, rank)
        P_u = torch.as_tensor(P_u[ua:ub], device=dev)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        f0.record()
        Eu = postprocess.field_points_device(dmn, u_dev, src, P_u, False)
        f1.record()
        barrier()
        fvec = torch.tensor([f0.elapsed_time(f1) / 1e3], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(fvec, op=dist.ReduceOp.MAX)
        t_uni = float(fvec.item())
        fl_u = float(n_uni) * (9.0 + 12 * 17) * nt
        field_uniform = {"points": n_uni, "seconds": t_uni, "evals_per_s": n_uni / t_uni,
                         "achieved_tflops": fl_u / t_uni / 1e12, "frac_of_fp64_peak": fl_u / t_uni / 1e12 / tflops_peak,
                         "note": "SURVEY 8d: uniform points in the 1.2x bbox (seed 0), timed once; flop = "
                                 "(9 + 12 x 17) nt per point (near pairs not counted)"}
        del Eu, P_u

    # GEMV roofline: stream this rank's row block a few times (untimed)
    A, rhs = assemble_distributed(mesh) if world > 1 else assemble(mesh)
    st = A.store
    z = torch.randn(N, dtype=torch.float64, device=dev)
    assembly.device_matvec(st, z)
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record()
    for _ in range(5):
        assembly.device_matvec(st, z)
    g1.record()
    torch.cuda.synchronize(dev)
    t_gemv = g0.elapsed_time(g1) / 5e3
    gemv_bytes = 8.0 * st.A.shape[0] * N
    del A, st
    torch.cuda.empty_cache()

    # full config 5: every collocation vertex seeded (~1e5 lines), traced once
    trace_full = None
    if args.full_trace and args.lines > 0:
        trace_stats.clear()
        t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        t0e.record()
        saved = args.lines
        args.lines = n
        trace_phase(sol)
        args.lines = saved
        t1e.record()
        barrier()
        tf = t0e.elapsed_time(t1e) / 1e3
        vec = torch.tensor([tf, trace_stats.get("evals", 0), trace_stats.get("inception", 0),
                            trace_stats.get("accepted", 0)], dtype=torch.float64, device=dev)
        if world > 1:
            t_only = vec[:1].clone()
            dist.all_reduce(t_only, op=dist.ReduceOp.MAX)
            dist.all_reduce(vec)
            vec[0] = t_only[0]
        tf, evals_f, inc_f, acc_f = vec.tolist()
        # a field evaluation is 9 nt (classification) + 12 x 17 nt
        # (density-contracted E nodes) flop, near pairs and the surface
        # distance on top (not counted)
        fl = evals_f * (9.0 + 12 * 17) * nt
        trace_full = {"lines": n, "seconds": tf, "lines_per_s": n / tf, "field_evals": int(evals_f),
                      "evals_per_line": evals_f / n, "reference_scheme_evals_per_line": (evals_f + acc_f) / n,
                      "inception_lines": int(inc_f), "achieved_tflops": fl / tf / 1e12,
                      "frac_of_fp64_peak": fl / tf / 1e12 / tflops_peak,
                      "rank0_terminations": dict(zip(("SurfaceHit", "WeakField", "MaxLength", "LeftDomain"),
                                                     trace_stats.get("terms", []))),
                      "note": "config 5 at its size: seeds at every collocation vertex (0.25 local R along the "
                              "normal), orientation sign(E.n), device RK45 + streamer; timed once after the steps; "
                              "the reference scheme needs one more evaluation per accepted step"}

    # end to end through the public API from host buffers, E2E_REPS times
    # (median): every mesh-derived product -- the column tiling, the device
    # buffers (H2D), the kd-tree of the coincidence check -- is rebuilt from
    # the host SurfaceMesh inside the timed region, exactly as assemble() on
    # a freshly loaded mesh does; u and E come back to the host.  Building
    # the SurfaceMesh itself (the reference's parse_mesh) is timed apart.
    e2e = None
    if not args.no_e2e:
        from paper_2003_12663_b200.device import mesh_tiling

        reps = []
        for _ in range(E2E_REPS):
            barrier()
            mesh._device_cache.clear()
            t0 = time.perf_counter()
            mesh_tiling(mesh)  # (also done inside assemble; split out for the breakdown)
            t_tile = time.perf_counter()
            device_mesh(mesh)
            torch.cuda.synchronize(dev)
            t_dm = time.perf_counter()
            if world > 1:
                A, rhs = assemble_distributed(mesh)
            else:
                A, rhs = assemble(mesh)
            torch.cuda.synchronize(dev)
            t1 = time.perf_counter()
            sol = solve(A, rhs, cfg_solver)
            del A
            t2 = time.perf_counter()
            E = postprocess.eval_efield_batch(sol, mesh, P_all[pa:pb])
            torch.cuda.synchronize(dev)
            t3 = time.perf_counter()
            reps.append([t1 - t0, t2 - t1, t3 - t2, t_tile - t0, t_dm - t_tile])
        ea, es, ef, et, eu = np.median(np.array(reps), axis=0).tolist()
        dmh = device_mesh(mesh)
        h2d = dmh.h2d_bytes + P_dev.numel() * 8 + N * 8  # mesh + tiling arrays, field points, rhs
        d2h = int(n * 8 + E.size * 8)
        evec = torch.tensor([ea, es, ef, et, eu], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(evec, op=dist.ReduceOp.MAX)
        ea, es, ef, et, eu = evec.tolist()
        e2e = {"value": N * N / ea, "unit": "entries/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "gmres_solve_s": es, "field_evals_per_s": args.points / ef,
               "breakdown_s": {"column_tiling": et, "device_mesh_upload": eu, "assemble": ea - et - eu,
                               "solve": es, "field": ef},
               "mesh_build_s": mesh_build_s, "reps": E2E_REPS,
               "note": "public API from the host SurfaceMesh: column tiling (host C++), device mesh (H2D), "
                       "assembly, solve and E at the field points each rep, u and E read back; median of reps; "
                       "the SurfaceMesh construction (mesh_build_s) is reported apart"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # the reference's own code (baseline/_ref) on every host core; the
        # oracle port stands in if baseline/_ref is missing
        cores = os.cpu_count() or 1
        try:
            _load_reference(args.scale)
            s, kind = reference_sample(_REF["mesh"], cores, 1, 3), "reference"
        except ImportError:
            s, kind = cpu_sample(mesh, max(args.cpu_rows, 2 * cores), cores, field_points=cores), "port"
        epl = trace_full["reference_scheme_evals_per_line"] if trace_full else None
        cpu = {"value": s["entries_per_s"], "unit": "entries/s", "cores": cores, "kind": kind,
               "sample": s["sample"], "matvec_s": s["matvec_s"], "field_evals_per_s": s["field_evals_per_s"],
               "trace_lines_per_s": (s["field_evals_per_s"] / epl) if epl else None,
               "trace_note": "field evals/s / the reference scheme's evaluations per line measured in trace_full"}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": N * N / t_asm,
            "unit": "entries/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": total / args.steps * 1e3,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (deterministic rod-plane + insulator generator, no RNG)",
            "config": {"workload": f"cfg4 rod-plane+insulator: {nt} panels, N={N} (dense {8 * N * N / 1e9:.1f} GB FP64)",
                       "panels": nt, "N": N, "field_points": args.points, "scale": args.scale,
                       "l2": "inputs larger than L2 (matrix streamed every matvec)",
                       "parallelism": f"row-block x{world}",
                       "matvec_exchange": (parallel.LAST_GATHER if world > 1 else None)},
            "gmres_solve_s": t_solve,
            "gmres_iterations": iters,
            "field_evals_per_s": args.points / t_field,
            "field_uniform": field_uniform,
            "field_near_surface": {"points": n, "evals_per_s": n / t_near,
                                   "near_pairs_per_point_rank0": near_pairs_per_point,
                                   "note": "every collocation point + 0.25 local R along its normal (SURVEY 8d)"},
            "phases_s": {"assembly": t_asm, "solve": t_solve, "field": t_field, "trace": t_trace,
                         "assembly_regular_kernel": reg_t},
            "trace_full": trace_full,
            "trace": {"lines": min(args.lines, n), "lines_per_s": min(args.lines, n) / t_trace if t_trace else None,
                      "field_evals": int(trace_evals), "inception_lines": int(trace_inception),
                      "rank0_rounds": trace_stats.get("rounds"), "rank0_terminations": dict(zip(
                          ("SurfaceHit", "WeakField", "MaxLength", "LeftDomain"), trace_stats.get("terms", []))),
                      "rank0_max_points": trace_stats.get("max_points"),
                      "note": "cfg5 on the step's own solution: surface |E|, top-k seeds, sign(E.n) orientation, "
                              "device RK45 tracer + streamer (air_demo.gas)"},
            "roofline": {"bound": "fp64", "kernel": "k_sweep", "achieved": achieved,
                         "peak": tflops_peak, "unit": "TFLOP/s", "frac": achieved / tflops_peak if tflops_peak else None,
                         "traffic": _ncu_traffic("k_sweep")[0], "traffic_detail": _ncu_traffic("k_sweep")[1],
                         "peak_burst": tflops_burst, "frac_of_burst": achieved / tflops_burst if tflops_burst else None,
                         "kernel_s_per_step": [round(x, 5) for x in reg_steps],
                         "peak_source": "measured DFMA kernel on this GPU (hvb_bench_dfma), sustained: launches back "
                                        "to back for 3 s, rate of the second half (the sweep runs inside a multi-second "
                                        "step); burst (one 6 ms launch) beside it"},
            "roofline_gemv": {"bound": "hbm", "kernel": "k_gemv_f64", "traffic": _ncu_traffic("k_gemv_f64_v4")[0],
                              "traffic_detail": _ncu_traffic("k_gemv_f64_v4")[1], "achieved": gemv_bytes / t_gemv / 1e9,
                              "peak": read_gbs, "unit": "GB/s", "frac": gemv_bytes / t_gemv / 1e9 / read_gbs,
                              "frac_of_measured_copy": (gemv_bytes / t_gemv / 1e9 / copy_gbs) if copy_gbs else None,
                              "measured_copy_gbs": copy_gbs,
                              "ms_per_matvec": t_gemv * 1e3,
                              "peak_source": "measured read-stream kernel on this GPU (hvb_bench_read: 256-bit non-allocating loads)"},
            "gpu_launches": launches,
            "clocks": sampler.summary() if sampler else None,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _count_near(mesh, rows):
    """Near pairs per row (from the last assembly on this device)."""
    import numpy as np

    from paper_2003_12663_b200 import assembly

    per = getattr(assembly, "LAST_NEAR_ROWS", None)
    if per is None:
        return np.zeros(len(rows), dtype=np.int64)
    return per[rows]


def _ncu_traffic(kernel):
    """(dram read+write bytes of one launch, detail) from the newest
    committed ncu full capture (profiles/rNN_ncu_traffic.json,
    tools/profile_summary.py); (None, None) if there is none."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_traffic.json")))
    if not files:
        return None, None
    try:
        with open(files[-1]) as fh:
            rec = json.load(fh).get(kernel)
    except (OSError, ValueError):
        return None, None
    if rec is None:
        return None, None
    notes = {"k_sweep": "one SL launch of the regular sweep: the 72 GB matrix write + the exchange slots "
                        "written and read back",
             "k_gemv_f64_v4": "one cfg4 matvec (the 79 GB row-major block is read once)"}
    return rec["bytes_per_launch"], {"dram_read_bytes": rec.get("dram_read_bytes"),
                                     "dram_write_bytes": rec.get("dram_write_bytes"),
                                     "source": os.path.basename(files[-1]), "note": notes.get(kernel, "")}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
