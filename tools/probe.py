"""Dev probe: phase timings of the hot path on one GPU (not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2003_12663_b200 import fixtures as F, _lib
from paper_2003_12663_b200 import assembly as AS
from paper_2003_12663_b200.assembly import assemble
from paper_2003_12663_b200.solver import solve, SolverConfig
from paper_2003_12663_b200.postprocess import eval_efield_batch

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
dev = torch.device("cuda", 0)
st = _lib.stream_ptr(dev)
# peaks
out = torch.zeros(1, dtype=torch.float64, device=dev)
for blocks in (148*8, 148*16):
    iters = 4000
    _lib.call("hvb_bench_dfma", _lib.ptr(out), blocks, 200, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); _lib.call("hvb_bench_dfma", _lib.ptr(out), blocks, iters, st); e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    print(f"dfma blocks={blocks}: {2*64*256*blocks*iters/t/1e12:.2f} TFLOP/s")
buf = torch.ones(2**30 // 8 * 8, dtype=torch.float64, device=dev)
_lib.call("hvb_bench_read", _lib.ptr(buf), buf.numel(), _lib.ptr(out), 148*8, st)
e0.record(); _lib.call("hvb_bench_read", _lib.ptr(buf), buf.numel(), _lib.ptr(out), 148*8, st); e1.record(); torch.cuda.synchronize()
print(f"read stream: {buf.numel()*8/(e0.elapsed_time(e1)/1e3)/1e9:.0f} GB/s")
del buf

t = time.time(); mesh = F.rod_plane_mesh(scale); print(f"mesh nt={mesh.n_triangles} n={mesh.n_collocation} {time.time()-t:.1f}s")
t = time.time()
from paper_2003_12663_b200.device import device_mesh
dm = device_mesh(mesh); torch.cuda.synchronize(); print(f"device mesh {time.time()-t:.1f}s tiles={dm.n_tiles} local/n={dm.tiling.redundancy:.3f} stream={dm.stream_for(0).numel()*8/1e6:.0f}MB")
for rep in range(2):
    torch.cuda.synchronize(); t = time.time()
    A, rhs = assemble(mesh); torch.cuda.synchronize(); ta = time.time() - t
    N = A.size
    print(f"assemble {ta:.3f}s  {N*N/ta/1e9:.2f} Gentries/s  near={A.diagnostics['pairs_near_singular']}")
    if rep == 0:
        del A
        torch.cuda.empty_cache()
# profile phases
store = A.store
x = torch.randn(N, dtype=torch.float64, device=dev)
for r in range(3):
    e0.record(); y = AS.device_matvec(store, x); e1.record(); torch.cuda.synchronize()
print(f"gemv {e0.elapsed_time(e1):.2f} ms  {8*N*N/(e0.elapsed_time(e1)/1e3)/1e9:.0f} GB/s")
torch.cuda.synchronize(); t = time.time()
sol = solve(A, rhs); torch.cuda.synchronize(); ts = time.time() - t
print(f"solve {ts:.3f}s iters={sol.iterations} res={sol.residual:.2e}")
rng = np.random.default_rng(0)
lo, hi = mesh.bounding_box(); c = 0.5*(lo+hi); h = 0.6*(hi-lo)
for M in (10000, 100000):
    P = c + rng.uniform(-1, 1, (M, 3)) * h
    torch.cuda.synchronize(); t = time.time()
    E = eval_efield_batch(sol, mesh, P); torch.cuda.synchronize(); tf = time.time()-t
    print(f"field M={M}: {tf:.3f}s {M/tf:.0f} evals/s")
