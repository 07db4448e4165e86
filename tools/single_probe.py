"""Dev: single-precision storage (assembly.precision = single) on cfg4:
matvec time and the solve under reference semantics."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__
__graft_entry__.build()
from paper_2003_12663_b200 import assembly as AS, fixtures
from paper_2003_12663_b200.solver import solve

mesh = fixtures.rod_plane_mesh(float(sys.argv[1]) if len(sys.argv) > 1 else 1.0)
for prec in ("single", "double"):
    A, b = AS.assemble(mesh, precision=prec)
    st = A.store
    z = torch.randn(A.size, dtype=torch.float64, device="cuda")
    AS.device_matvec(st, z)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        AS.device_matvec(st, z)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 5
    torch.cuda.synchronize(); t0 = time.time()
    try:
        sol = solve(A, b); it, res = sol.iterations, sol.residual
    except Exception as exc:
        it, res = -1, str(exc)[:80]
    torch.cuda.synchronize()
    bytes_ = st.A.element_size() * st.A.shape[0] * A.size
    print(f"{prec}: matvec {t:.2f} ms ({bytes_ / t / 1e6:.0f} GB/s), solve {time.time() - t0:.3f} s iters {it} res {res}")
    del A, st
    torch.cuda.empty_cache()
