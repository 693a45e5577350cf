"""Where does the bf16 error of the 8B 8K prefill come from?  Per-layer K/V
error of the product vs the fp32 forward and vs the fp32 forward with bf16
rounding at the points the GPU stores bf16 (tests/torch_ref.py emulate_bf16),
plus the fp32-vs-emulated distance itself (inherent storage error).

    python tools/parity_depth.py [--tokens 8192] [--layers 32] > out.json
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch_ref  # noqa: E402
from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, Engine, LoopbackGroup,  # noqa: E402
                                   ParallelMode, ShiftPolicy, llama31_8b)
from paper_2507_11830_b200.weights import ModelWeights  # noqa: E402


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--f64", action="store_true", help="also run an f64 forward")
    a = ap.parse_args()
    cfg = llama31_8b(n_layers=a.layers, max_seq=max(a.tokens, 128))
    w = ModelWeights.random(cfg, seed=a.seed, world_size=1)
    prompt = [int(t) for t in np.random.default_rng(0).integers(0, cfg.vocab_size, size=a.tokens)]
    eng = Engine(w, LoopbackGroup(1), ShiftPolicy.fixed_sp(), num_blocks=a.tokens // 64 + 8)
    s = eng.new_sequence(0, capacity=a.tokens)
    lg, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, prompt)]), mode=ParallelMode.SP)
    rw = torch_ref.RefWeights.from_model(w)
    out = {"tokens": a.tokens, "layers": a.layers}
    refs = {}
    for name, emu in (("fp32", False), ("emu", True), ("emu_p", True)):
        hid = {}
        want, cache = torch_ref.forward(rw, prompt, emulate_bf16=emu, logit_rows=[a.tokens - 1],
                                        hidden_out=hid, round_p=name == "emu_p")
        refs[name] = (want[0], cache, hid["x"][0])
    if a.f64:
        rw64 = torch_ref.RefWeights.from_model(w, dtype=torch.float64)
        want, cache = torch_ref.forward(rw64, prompt, logit_rows=[a.tokens - 1])
        refs["f64"] = (want[0], cache, None)
    got = lg[0]
    for name, (want, cache, _) in refs.items():
        out[f"logits_vs_{name}"] = rel(got, want)
        per = []
        for layer in range(a.layers):
            kg, vg = s.cache.read_window(0, layer, 0)
            per.append((round(rel(kg.float(), cache.k[layer][:, 0]), 5),
                        round(rel(vg.float(), cache.v[layer][:, 0]), 5)))
        out[f"kv_vs_{name}"] = per
    f, e = refs["fp32"], refs["emu"]
    out["fp32_vs_emu_logits"] = rel(e[0], f[0])
    out["fp32_vs_emu_hidden"] = rel(e[2], f[2])
    out["fp32_vs_emu_kv"] = [round(rel(e[1].k[l][:, 0], f[1].k[l][:, 0]), 5) for l in range(a.layers)]
    out["fp32_vs_emu_p_logits"] = rel(refs["emu_p"][0], f[0])
    if "f64" in refs:
        out["fp32_vs_f64_logits"] = rel(f[0], refs["f64"][0])
        out["fp32_vs_f64_kv"] = [round(rel(f[1].k[l][:, 0], refs["f64"][1].k[l][:, 0]), 7)
                                 for l in range(a.layers)]
    out["hidden_absmax"] = float(f[2].abs().max())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
