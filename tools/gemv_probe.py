"""Dev: GEMV variants on a cfg4-width FP64 block (GB/s)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2003_12663_b200 import _lib
N = 99558
lda = -(-N // 32) * 32
rows = 24000
A = torch.randn((rows, lda), dtype=torch.float64, device="cuda")
x = torch.randn(lda, dtype=torch.float64, device="cuda")
y = torch.empty(rows, dtype=torch.float64, device="cuda")
st = _lib.stream_ptr()
ref = None
names = {0: "double2 R8 (prod)", 1: "v4-256b R8", 2: "v4-256b R4", 3: "v4-256b R16", 4: "double2 R4", 5: "double2 R16",
         6: "v4-256b R2", 7: "v4-256b R1"}
for v in range(8):
    _lib.call("hvb_bench_gemv", _lib.ptr(A), lda, rows, N, _lib.ptr(x), _lib.ptr(y), v, st)
    torch.cuda.synchronize()
    if ref is None:
        ref = y.clone()
    err = float((y - ref).abs().max() / ref.abs().max())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        _lib.call("hvb_bench_gemv", _lib.ptr(A), lda, rows, N, _lib.ptr(x), _lib.ptr(y), v, st)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10e3
    print(f"{names[v]:20s} {rows * N * 8 / t / 1e9:8.1f} GB/s  (rel diff vs prod {err:.1e})")

del A
buf = torch.ones(2 ** 30, dtype=torch.float64, device="cuda")  # 8 GiB
out = torch.zeros(1, dtype=torch.float64, device="cuda")
for blocks in (148 * 8, 148 * 16, 148 * 32, 148 * 64):
    _lib.call("hvb_bench_read", _lib.ptr(buf), buf.numel(), _lib.ptr(out), blocks, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        _lib.call("hvb_bench_read", _lib.ptr(buf), buf.numel(), _lib.ptr(out), blocks, st)
    e1.record()
    torch.cuda.synchronize()
    print(f"read stream (256-bit) {blocks} blocks: {buf.numel() * 8 * 5 / (e0.elapsed_time(e1) / 1e3) / 1e9:8.1f} GB/s")
