"""Fork-based process pool for the CPU oracle legs of the at-scale parity
tests (test infrastructure).  The parent sets ``STATE`` (mesh, density ...)
before the pool forks, so the workers inherit it copy-on-write; workers run
NumPy only (never CUDA) with one BLAS thread each."""

from __future__ import annotations

import multiprocessing as mp
import os

STATE: dict = {}


def _init():
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:  # pragma: no cover
        pass


def pmap(fn, items, procs: int | None = None):
    items = list(items)
    procs = max(1, min(procs or os.cpu_count() or 1, len(items)))
    if procs == 1:
        return [fn(x) for x in items]
    with mp.get_context("fork").Pool(procs, initializer=_init) as pool:
        return pool.map(fn, items, chunksize=1)


# ---- workers (read STATE; oracle only) ------------------------------------


def oracle_rows(rows):
    """Dense oracle rows (reference _row_equation) of STATE['mesh']."""
    from oracle import hvb_oracle as ora

    return ora.row_equations(STATE["mesh"], list(rows), tables=STATE.get("tables"))


def oracle_charge(members):
    """Partial oracle charge vector over a chunk of members."""
    from oracle import hvb_oracle as ora

    return ora.charge_vector(STATE["mesh"], list(members), STATE["adl"], STATE["ids"], tables=STATE.get("tables"))


def oracle_trace(k):
    """Oracle Dormand-Prince line k of STATE['starts'] / STATE['orient']."""
    from oracle import hvb_oracle as ora

    return ora.trace_line(STATE["mesh"], STATE["u"], STATE["starts"][k], int(STATE["orient"][k]),
                          tables=STATE.get("tables"))


def chunks(seq, n):
    seq = list(seq)
    step = max(1, -(-len(seq) // n))
    return [seq[i:i + step] for i in range(0, len(seq), step)]
