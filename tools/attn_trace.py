"""Timeline of the tcgen05 prefill attention's pipeline (instrumented build:
nvcc ... -DATTN_TRACE, loaded with SP_LIB_PATH) — clock64 stamps of CTA (0,0)
(the longest causal work tile of an 8K prefill), iterations 0..31.

    SP_LIB_PATH=build_ab/lib_trace.so python tools/attn_trace.py
Prints, per key tile: when the MMA issuer got V and each half/whole P, when it
finished issuing PV+QK per Q tile, and per softmax warpgroup when S arrived,
the max was done, P-half and P-full were published (cycles from iteration 0).
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import runpy  # noqa: E402

from paper_2507_11830_b200 import _lib  # noqa: E402

runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "attn_probe.py"))
lib = _lib.load()
buf = (ctypes.c_ulonglong * 768)()
fn = lib.sp_attn_trace_copy
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert fn(ctypes.addressof(buf), 768) == 0
t = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(3, 32, 8)
t0 = t[0, 0, 0]
rel = t - t0
print("it | MMA: v_wait v_ok  ph0  pf0  ph1  pf1  qk0_done qk1_done | SM0: wait s_ok max ph pf | SM1: wait s_ok max ph pf")
for it in range(2, 20):
    m = rel[0, it]
    a, b = rel[1, it], rel[2, it]
    print(f"{it:2d} | {m[0]:7d} {m[1]:7d} {m[2]:7d} {m[3]:7d} {m[4]:7d} {m[5]:7d} {m[6]:7d} {m[7]:7d} | "
          f"{a[0]:7d} {a[1]:7d} {a[2]:7d} {a[3]:7d} {a[4]:7d} | {b[0]:7d} {b[1]:7d} {b[2]:7d} {b[3]:7d} {b[4]:7d}")
per = np.diff(rel[0, 2:20, 6])
print("period (cycles between consecutive qk0_done):", per.tolist(), "median", int(np.median(per)))
sm = rel[1, 2:20]
print("softmax0 durations: s_ok->max", np.median(sm[:, 2] - sm[:, 1]), " max->p_half",
      np.median(sm[:, 3] - sm[:, 2]), " p_half->p_full", np.median(sm[:, 4] - sm[:, 3]),
      " idle (p_full -> next s_ok)", np.median(rel[1, 3:21, 1] - rel[1, 2:20, 4]))
