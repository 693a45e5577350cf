"""Isolated prefill RMSNorm timing (8192 x 4096 f32 -> bf16, L2 flushed): general vs register-lean kernel, vs a torch conversion copy of the same traffic.

    python tools/norm_probe.py
"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2507_11830_b200 import ops
M, h = 8192, 4096
x = torch.randn(M, h, device="cuda")
g = torch.ones(h, device="cuda")
out = torch.empty(M, h, dtype=torch.bfloat16, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(n=20, thr=None):
    if thr: os.environ["SP_NORM_THREADS"] = str(thr)
    else: os.environ.pop("SP_NORM_THREADS", None)
    ts = []
    for i in range(n):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); ops.add_rmsnorm(x, g, 1e-5, out); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort(); return ts[n // 2] * 1e3
ref = None
for lean in ("0", "1"):
    os.environ["SP_NORM_LEAN"] = lean
    us = t()
    o = out.clone()
    if ref is None:
        ref = o
    print(f"rows lean={lean} {us:.1f} us  {M*h*6/us/1e3:.0f} GB/s  bitexact={torch.equal(o, ref)}")
# the same traffic as a plain conversion copy (torch), for reference
ts = []
for i in range(20):
    flush.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); out.copy_(x); e.record(); torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
ts.sort()
us = ts[10] * 1e3
print(f"rows torch f32->bf16 copy {us:.1f} us  {M*h*6/us/1e3:.0f} GB/s")
