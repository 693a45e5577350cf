"""Debug: where do the TP all-reduce paths (two-shot / one-shot / collective)
diverge?  Prints, per variant pair, the first layer whose K/V differ and the
max logit difference of the prefill and decode outputs."""

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

from helpers import c1_prompts, device_weights  # noqa: E402
from oracle.model import init_weights_llama, llama_tiny_config  # noqa: E402
from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, Engine, LoopbackGroup,  # noqa: E402
                                   ParallelMode, ShiftPolicy)


def run(p, env, extra_env=None):
    for k in ("SP_TP_TWO_SHOT_MIN_ROWS", "SP_FUSED_A2A", "SP_FUSE_SPLITK"):
        os.environ.pop(k, None)
    os.environ.update(env)
    os.environ.update(extra_env or {})
    ow = init_weights_llama(llama_tiny_config(max_seq=512, n_kv_heads=4), seed=1)
    eng = Engine(device_weights(ow, p), LoopbackGroup(p), ShiftPolicy.fixed_tp())
    prompts = [c1_prompts()[i] for i in (0, 3, 5)]
    seqs = [eng.new_sequence(i, capacity=200) for i in range(3)]
    lg, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, q) for s, q in zip(seqs, prompts)]),
                     mode=ParallelMode.TP)
    kv = [[t.cpu() for t in seqs[2].cache.read_window(r, l, 0)] for l in range(4) for r in range(p)]
    lg2, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [7]) for s in seqs]), mode=ParallelMode.TP)
    return [x.cpu() for x in lg], [x.cpu() for x in lg2], kv


for p in ():
    for extra in ({}, {"SP_FUSE_SPLITK": "0"}):
        res = {n: run(p, e, extra) for n, e in (("two", {}),
                                                  ("one", {"SP_TP_TWO_SHOT_MIN_ROWS": "100000"}),
                                                  ("coll", {"SP_FUSED_A2A": "0"}))}
        for other in ("one", "coll"):
            a, b = res["two"], res[other]
            pre = max(float((x - y).abs().max()) for x, y in zip(a[0], b[0]))
            dec = max(float((x - y).abs().max()) for x, y in zip(a[1], b[1]))
            first = next((i for i, (x, y) in enumerate(zip(a[2], b[2]))
                          if not (torch.equal(x[0], y[0]) and torch.equal(x[1], y[1]))), None)
            print(f"p={p} {extra} two vs {other}: prefill {pre:.3g} decode {dec:.3g} "
                  f"first KV (layer*p+rank) diff {first}", flush=True)


# ---- x snapshots after every residual update (one-shot vs collective, P=4)
from paper_2507_11830_b200 import ops  # noqa: E402

snaps = []
_orig = {n: getattr(ops, n) for n in ("add_rmsnorm", "peer_allreduce_add_rmsnorm", "add_f32")}


def _wrap(name):
    def f(*a, **k):
        _orig[name](*a, **k)
        x = a[0] if name != "peer_allreduce_add_rmsnorm" else a[2]
        snaps.append((name, x.data_ptr(), x.detach().clone().cpu()))
    return f


for n in _orig:
    setattr(ops, n, _wrap(n))
out = {}
for name, env in (("one", {"SP_TP_TWO_SHOT_MIN_ROWS": "100000"}), ("coll", {"SP_FUSED_A2A": "0"})):
    snaps.clear()
    run(4, env)
    xp = snaps[0][1]  # the residual x of the prefill pass
    out[name] = [(n, x) for n, ptr, x in snaps if ptr == xp]
for i, ((na, xa), (nb, xb)) in enumerate(zip(out["one"], out["coll"])):
    same = xa.shape == xb.shape and torch.equal(xa, xb)
    diff = float((xa - xb).abs().max()) if xa.shape == xb.shape else -1
    print(f"snap {i}: {na} vs {nb} shape {tuple(xa.shape)} vs {tuple(xb.shape)} equal={same} "
          f"maxdiff={diff:.3g} nrows_diff={int(((xa - xb).abs().amax(1) > 0).sum()) if xa.shape == xb.shape else -1}")
print(len(out["one"]), len(out["coll"]))
