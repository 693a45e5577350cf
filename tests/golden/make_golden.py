"""Generate golden fixtures by running the REAL reference (``shiftsim``).

Run in the build container, where ``/root/reference`` is mounted:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``tests/golden/shiftsim_golden.npz`` and ``shiftsim_golden.json``.
The GPU box never reads ``/root/reference``; it only sees these committed
fixtures.  Every case names the reference call that produced it.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from shiftsim.fabric import DeviceGroup  # noqa: E402
from shiftsim.flops import PassShape, flop_count, shard_rows, swiftkv_flop_ratio  # noqa: E402
from shiftsim.model import (  # noqa: E402
    ModelConfig, forward_reference, greedy_token, induction_weights, init_weights,
    partition_heads, reference_greedy,
)
from shiftsim.parallel_engine import (  # noqa: E402
    Batch, BatchItem, BatchKind, Engine, ParallelMode, ShiftPolicy,
)
from shiftsim.swiftkv import SwiftKvConfig  # noqa: E402
from shiftsim.tensor_core import Precision, softmax_rows  # noqa: E402

OUT = Path(__file__).resolve().parent


def seeded_prompt(seed, length, vocab):  # tests/conftest.py:24-27
    rng = np.random.default_rng(seed)
    return [int(x) for x in rng.integers(0, vocab, size=length)]


def weights_digest(w) -> str:
    h = hashlib.sha256()
    h.update(w.embed.tobytes())
    for lw in w.layers:
        for name in ("wq", "wk", "wv", "wo", "w1", "w2"):
            h.update(getattr(lw, name).tobytes())
    h.update(w.head.tobytes())
    return h.hexdigest()


def c1_prompts():
    """C1 workload: default_rng(7), 8 lengths in [32, 129)."""
    rng = np.random.default_rng(7)
    lens = [int(x) for x in rng.integers(32, 129, size=8)]
    return [[int(t) for t in rng.integers(0, 256, size=n)] for n in lens]


def main():
    arrays, meta = {}, {}

    # 1. init draw-order pins (tests/test_model.py:76-81) + full digest
    w0 = init_weights(ModelConfig(), seed=0)
    meta["init_default_seed0"] = {
        "embed_0_0": float(w0.embed[0, 0]), "embed_0_2": float(w0.embed[0, 2]),
        "head_0_0": float(w0.head[0, 0]), "sha256": weights_digest(w0)}
    meta["softmax_1000_999"] = [float(x) for x in softmax_rows(np.array([[1000.0, 999.0]]))[0]]
    meta["partition_heads_8_4"] = [list(x) for x in partition_heads(8, 4)]
    meta["shard_rows"] = {"10_4": shard_rows(10, 4), "1_2": shard_rows(1, 2)}
    meta["swiftkv_ratio_default_256_cut2"] = swiftkv_flop_ratio(ModelConfig(), 256, 2)

    # 2. tiny config (tests/conftest.py:8-17), seed 3, f64
    tiny = ModelConfig(n_layers=2, n_heads=4, head_dim=8, ffn_dim=64, vocab_size=64, max_seq=256)
    wt = init_weights(tiny, seed=3)
    meta["tiny_sha256"] = weights_digest(wt)
    p21 = seeded_prompt(21, 12, 64)
    arrays["tiny_dense_logits_p21"] = forward_reference(wt, p21)[0]
    p23 = seeded_prompt(23, 13, 64)
    for p in (2, 4):
        for mode in (ParallelMode.TP, ParallelMode.SP):
            eng = Engine(wt, DeviceGroup(p), ShiftPolicy.fixed_tp())
            seq = eng.new_sequence(0, capacity=13)
            lg, rec = eng.step(Batch(BatchKind.PREFILL, [BatchItem(seq, list(p23))]),
                               mode=mode, span_logits=True)
            arrays[f"tiny_{mode.value}{p}_span_logits_p23"] = lg[0]
            meta[f"tiny_{mode.value}{p}_record_p23"] = {
                "flops_per_device": list(rec.flops_per_device),
                "comm": [[e.kind, e.bytes] for e in rec.comm]}
            k0, v0 = seq.cache.device_blocks(0)
            arrays[f"tiny_{mode.value}{p}_dev0_k"] = k0
            arrays[f"tiny_{mode.value}{p}_dev0_v"] = v0
            meta[f"tiny_{mode.value}{p}_write_counter"] = seq.cache.write_counter
    meta["tiny_greedy_p24"] = {"prompt": seeded_prompt(24, 10, 64),
                               "tokens": reference_greedy(wt, seeded_prompt(24, 10, 64), 12)}
    # multi-item SP prefill (tests/test_parallel_engine.py:79-92)
    prompts = [seeded_prompt(30 + i, 6 + 3 * i, 64) for i in range(3)]
    eng = Engine(wt, DeviceGroup(2), ShiftPolicy.fixed_tp())
    items = [BatchItem(eng.new_sequence(i, capacity=len(pp)), list(pp)) for i, pp in enumerate(prompts)]
    lg, rec = eng.step(Batch(BatchKind.PREFILL, items), mode=ParallelMode.SP, span_logits=True)
    meta["tiny_multi_prompts"] = prompts
    for i, l in enumerate(lg):
        arrays[f"tiny_multi_sp2_item{i}"] = l
    # decode flops with history (tests/test_parallel_engine.py:147-166)
    for mode in ("tp", "sp"):
        for p in (1, 2, 4):
            shp = PassShape(spans=(9, 5), history=(0, 0))
            shp2 = PassShape(spans=(1, 1), history=(9, 5))
            meta[f"tiny_flops_{mode}{p}"] = [list(flop_count(shp, mode, tiny, p).per_device),
                                             list(flop_count(shp2, mode, tiny, p).per_device)]

    # 3. SwiftKV (tests/test_swiftkv.py:21-27), seed 5, cut 2, P=2
    kvc = ModelConfig(n_layers=4, n_heads=4, head_dim=8, ffn_dim=64, vocab_size=64, max_seq=512)
    wk = init_weights(kvc, seed=5)
    p50 = seeded_prompt(50, 20, 64)
    for mode in (ParallelMode.TP, ParallelMode.SP):
        eng = Engine(wk, DeviceGroup(2), ShiftPolicy.fixed_tp(), swiftkv=SwiftKvConfig(True, 2))
        seq = eng.new_sequence(0, capacity=24)
        lg, rec = eng.step(Batch(BatchKind.PREFILL, [BatchItem(seq, list(p50))]), mode=mode)
        arrays[f"swiftkv_{mode.value}2_logits_p50"] = lg[0]
        meta[f"swiftkv_{mode.value}2_flops"] = list(rec.flops_per_device)
        toks = [greedy_token(lg[0])]
        for _ in range(3):
            lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(seq, [toks[-1]])]), mode=mode)
            toks.append(greedy_token(lg[0]))
        meta[f"swiftkv_{mode.value}2_decode_tokens"] = toks
    # multi-item SwiftKV SP (uneven tail counts per rank)
    mp = [seeded_prompt(60 + i, 3 + 4 * i, 64) for i in range(3)]
    eng = Engine(wk, DeviceGroup(2), ShiftPolicy.fixed_tp(), swiftkv=SwiftKvConfig(True, 2))
    items = [BatchItem(eng.new_sequence(i, capacity=32), list(pp)) for i, pp in enumerate(mp)]
    lg, _ = eng.step(Batch(BatchKind.PREFILL, items), mode=ParallelMode.SP)
    meta["swiftkv_multi_prompts"] = mp
    arrays["swiftkv_multi_sp2_logits"] = np.stack(lg)

    # 4. C1 compat stand-in: L4, h256 (8 MHA heads of 32), f1024, V256, f32, P=2
    c1 = ModelConfig(n_layers=4, n_heads=8, head_dim=32, ffn_dim=1024, vocab_size=256, max_seq=512)
    wc = init_weights(c1, seed=0, precision=Precision.F32)
    pr = c1_prompts()
    meta["c1_prompt_lens"] = [len(x) for x in pr]
    for mode in (ParallelMode.SP, ParallelMode.TP):
        eng = Engine(wc, DeviceGroup(2), ShiftPolicy.fixed_tp())
        seqs = [eng.new_sequence(i, capacity=len(x) + 4) for i, x in enumerate(pr)]
        lg, rec = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, list(x)) for s, x in zip(seqs, pr)]),
                           mode=mode)
        arrays[f"c1_{mode.value}2_prefill_logits"] = np.stack(lg)
        toks = [[greedy_token(l)] for l in lg]
        for _ in range(3):
            lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [t[-1]]) for s, t in zip(seqs, toks)]),
                             mode=mode)
            for t, l in zip(toks, lg):
                t.append(greedy_token(l))
        meta[f"c1_{mode.value}2_decode_tokens"] = toks
        arrays[f"c1_{mode.value}2_decode_last_logits"] = np.stack(lg)

    # 5. induction model greedy replay (tests/test_model.py:152-160)
    wi = induction_weights(max_seq=256)
    meta["induction"] = []
    for tpl in ([3, 14, 7, 9], [1, 2, 3], [5, 30, 11, 2, 19]):
        prompt = (tpl * (48 // len(tpl) + 1))[:48]
        meta["induction"].append({"prompt": prompt, "tokens": reference_greedy(wi, prompt, 12)})

    np.savez_compressed(OUT / "shiftsim_golden.npz", **arrays)
    with open(OUT / "shiftsim_golden.json", "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays,", len(meta), "meta keys")


if __name__ == "__main__":
    main()
