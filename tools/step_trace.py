"""Device timeline of one graph-replayed decode step (or eager prefill pass):
every CTA of every kernel stamps globaltimer at entry, at its
griddepcontrol.wait release and at exit (library built with -DSTEP_TRACE,
see csrc/common.cuh).  Prints one line per launch and the per-boundary
latencies: from the predecessor's last CTA exit to this launch's first wait
release, and how much of a launch ran before that release (PDL overlap).

    SP_NVCC_EXTRA=-DSTEP_TRACE python -m paper_2507_11830_b200.build --force
    cp paper_2507_11830_b200/libshiftpar.so paper_2507_11830_b200/libshiftpar_trace.so
    python -m paper_2507_11830_b200.build --force        # production library back
    python tools/step_trace.py [B] [ctx] [--layers N] [--ctas]   # decode step at batch B
                                    # (--ctas: per-launch exit percentiles, entry/exit corr)
"""
import os
import re
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(HERE, "paper_2507_11830_b200")
os.environ.setdefault("SP_LIB_PATH", os.path.join(PKG, "libshiftpar_trace.so"))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, Engine, LoopbackGroup,  # noqa: E402
                                   ParallelMode, ShiftPolicy, llama31_8b)
from paper_2507_11830_b200 import _lib  # noqa: E402
from paper_2507_11830_b200.weights import ModelWeights  # noqa: E402

TU = {1: "attention.cu", 2: "attention_tc.cu", 3: "decode_layer.cu", 4: "gemm_tcgen05.cu",
      5: "peer.cu", 6: "runtime.cu"}


def kernel_names():
    """(tu, line) of a pdl_trigger() call -> the enclosing kernel's name."""
    out = {}
    for tu, fn in TU.items():
        lines = open(os.path.join(PKG, "csrc", fn)).read().split("\n")
        name = "?"
        for i, ln in enumerate(lines):
            m = re.search(r"\b(\w+_kernel)\s*\(", ln)
            if m and any("__global__" in x for x in lines[max(0, i - 3):i + 1]):
                name = m.group(1)
            out[(tu, i + 1)] = name
    return out


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    B = int(args[0]) if args else 1
    ctx = int(args[1]) if len(args) > 1 else 2048
    layers = 32
    if "--layers" in sys.argv:
        layers = int(sys.argv[sys.argv.index("--layers") + 1])
    lib = _lib.load()
    cfg = llama31_8b(max_seq=ctx + 64, n_layers=layers)
    w = ModelWeights.random(cfg, seed=0, world_size=1)
    eng = Engine(w, LoopbackGroup(1), ShiftPolicy.fixed_tp(),
                 num_blocks=B * -(-(ctx + 64) // 64) + 8)
    rng = np.random.default_rng(0)
    seqs = [eng.new_sequence(i, capacity=ctx + 64) for i in range(B)]
    for i in range(0, B, 8):
        eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, [int(t) for t in rng.integers(0, 1000, ctx)])
                                           for s in seqs[i:i + 8]]), mode=ParallelMode.SP)

    def step():
        eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [1]) for s in seqs]), mode=ParallelMode.TP)
        for s in seqs:
            s.cache.truncate(ctx)
    for _ in range(8):
        step()
    cap = 1 << 18
    buf = torch.zeros(cap * 4, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    rc = lib.sp_step_trace_bind(buf.data_ptr(), cnt.data_ptr(), cap)
    if rc != 0:
        raise SystemExit(f"sp_step_trace_bind: {lib.sp_last_error().decode()} (build the trace library)")
    step()
    torch.cuda.synchronize()
    lib.sp_step_trace_bind(None, None, 0)
    n = min(int(cnt.item()), cap)
    rec = buf[:n * 4].view(n, 4).cpu().numpy().astype(np.uint64)
    names = kernel_names()
    launches = []
    cur = None
    for r in rec:
        tag, t0, tw, t1 = (int(x) for x in r)
        blk, tu, line = tag >> 32, (tag >> 16) & 0xffff, tag & 0xffff
        key = (tu, line)
        if cur is None or cur["key"] != key or blk in cur["blocks"]:
            cur = {"key": key, "name": names.get(key, f"tu{tu}:{line}"), "blocks": set(), "entry": [],
                   "wait": [], "exit": []}
            launches.append(cur)
        cur["blocks"].add(blk)
        cur["entry"].append(t0)
        if tw:
            cur["wait"].append(tw)
        cur["exit"].append(t1)
    base = min(min(L["entry"]) for L in launches)
    end = max(max(L["exit"]) for L in launches)
    print(f"B={B} ctx={ctx} layers={layers}: {len(launches)} launches, {n} CTAs, "
          f"step span {(end - base) / 1e3:.1f} us (first CTA entry -> last CTA exit)")
    print(f"{'kernel':34s} {'ctas':>5s} {'entry0':>8s} {'wait0':>8s} {'wait1':>8s} {'exit0':>8s} {'exit1':>8s}"
          f" {'gap':>6s} {'run':>7s}")
    prev_exit = None
    gaps = {}
    runs = {}
    for L in launches:
        e0 = (min(L["entry"]) - base) / 1e3
        w0 = (min(L["wait"]) - base) / 1e3 if L["wait"] else float("nan")
        w1 = (max(L["wait"]) - base) / 1e3 if L["wait"] else float("nan")
        x0 = (min(L["exit"]) - base) / 1e3
        x1 = (max(L["exit"]) - base) / 1e3
        gap = (w0 - prev_exit) if prev_exit is not None and L["wait"] else float("nan")
        run = x1 - (w0 if L["wait"] else e0)
        if not np.isnan(gap):
            gaps.setdefault(L["name"], []).append(gap)
        runs.setdefault(L["name"], []).append(run)
        if layers <= 2 or len(launches) < 40 or "--all" in sys.argv:
            print(f"{L['name'][:34]:34s} {len(L['blocks']):5d} {e0:8.1f} {w0:8.1f} {w1:8.1f} {x0:8.1f} {x1:8.1f}"
                  f" {gap:6.2f} {run:7.1f}")
            if "--ctas" in sys.argv and len(L["exit"]) > 8:
                # tail shape: exit-time percentiles, and whether late exits
                # are the CTAs that entered late (corr of entry vs exit)
                ex = (np.asarray(L["exit"], dtype=np.float64) - base) / 1e3
                en = (np.asarray(L["entry"], dtype=np.float64) - base) / 1e3
                pct = np.percentile(ex, [10, 50, 90])
                corr = float(np.corrcoef(en, ex)[0, 1]) if en.std() > 0 and ex.std() > 0 else 0.0
                print(f"{'':34s} entry {en.min():.1f}..{en.max():.1f}  exit p10/p50/p90 "
                      f"{pct[0]:.1f}/{pct[1]:.1f}/{pct[2]:.1f}  corr(entry, exit) {corr:+.2f}")
        prev_exit = x1
    print("\nper kernel: launches, mean release gap after the predecessor's last exit (us), "
          "mean run from first release to last exit (us), total run")
    for k in runs:
        g = gaps.get(k, [])
        print(f"  {k:34s} {len(runs[k]):4d}  gap {np.mean(g) if g else float('nan'):6.2f}  "
              f"run {np.mean(runs[k]):7.2f}  total {np.sum(runs[k]):8.1f}")


if __name__ == "__main__":
    main()
