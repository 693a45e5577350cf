"""Measurements for the BASELINE configs beyond the bench.py headline (1 GPU).

    python tools/configs_bench.py decode-sweep   # configs[2]: decode B=1..256 across the shift threshold
    python tools/configs_bench.py swiftkv        # configs[4]: 8B SwiftKV 32K prefill (cut 16) vs standard
    python tools/configs_bench.py all

One JSON line per measurement.  Timing: CUDA events around K steps after
warm-up, synchronize on both sides.  Weights: random-init bf16 Llama-3.1-8B.
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, Engine, LoopbackGroup,  # noqa: E402
                                   ParallelMode, ShiftPolicy, SwiftKvConfig, llama31_8b, ops)
from paper_2507_11830_b200.flops import causal_attention_flops, gemm_flops_per_token  # noqa: E402
from paper_2507_11830_b200.weights import ModelWeights  # noqa: E402

PEAKS = {"hbm_gbs": 6552.3, "bf16_tflops_sustained": 1366.3}
try:
    PEAKS.update(json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json"))))
except Exception:
    pass


def timed(fn, steps, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def decode_sweep(weights, cfg, ctx=2048, tau=32):
    """configs[2]: one shared paged pool; prefill B requests to ctx, then decode
    under forced TP, forced SP and the shift policy (tau new tokens)."""
    rng = np.random.default_rng(0)
    bmax = 256
    eng = Engine(weights, LoopbackGroup(1), ShiftPolicy(token_threshold=tau),
                 num_blocks=bmax * -(-(ctx + 64) // 64) + 16)
    seqs = [eng.new_sequence(i, capacity=ctx + 64) for i in range(bmax)]
    prompts = [[int(t) for t in rng.integers(0, cfg.vocab_size, size=ctx)] for _ in range(bmax)]
    for i in range(0, bmax, 8):
        eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, p) for s, p in zip(seqs[i:i + 8], prompts[i:i + 8])]))
    wbytes = weights.nbytes() - weights.embed.nbytes  # the embedding is gathered, not streamed
    for B in (1, 2, 4, 8, 16, 32, 64, 128, 256):
        sub = seqs[:B]
        res = {}
        for label, mode in (("tp", ParallelMode.TP), ("sp", ParallelMode.SP), ("shift", None)):
            def step():
                toks = [1] * B
                for s in sub:
                    s.cache.truncate(s.cache.token_count)  # decode at a fixed context
                eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [t]) for s, t in zip(sub, toks)]),
                         mode=mode)
                for s in sub:
                    s.cache.truncate(s.cache.token_count - 1)
            before = sum(s.cache.write_counter for s in sub)
            res[label] = timed(step, 24, warm=12)  # first replays after a capture run slow
            chosen = eng.mode_log[-1].value
        kv_bytes = B * ctx * cfg.n_layers * 2 * cfg.kv_heads * cfg.head_dim * 2
        roof = (wbytes + kv_bytes) / (PEAKS["hbm_gbs"] * 1e9) * 1e3
        print(json.dumps({"config": "decode-sweep (configs[2])", "n_gpus": 1, "batch": B, "ctx": ctx,
                          "tpot_ms_tp": round(res["tp"], 4), "tpot_ms_sp": round(res["sp"], 4),
                          "tpot_ms_shift": round(res["shift"], 4), "shift_mode": chosen,
                          "tau": tau, "hbm_roofline_ms": round(roof, 4),
                          "frac_of_roofline_tp": round(roof / res["tp"], 4),
                          "tokens_per_s": round(B / res["tp"] * 1e3, 1)}), flush=True)


def swiftkv(weights, cfg, seq=32768, cut=16):
    """configs[4]: SwiftKV early-exit prefill of one 32K-token request vs standard."""
    rng = np.random.default_rng(1)
    prompt = [int(t) for t in rng.integers(0, cfg.vocab_size, size=seq)]
    out = {}
    for label, skv in (("standard", None), ("swiftkv", SwiftKvConfig(enabled=True, cut_layer=cut))):
        eng = Engine(weights, LoopbackGroup(1), ShiftPolicy.fixed_sp(), swiftkv=skv,
                     num_blocks=-(-seq // 64) + 8)
        s = eng.new_sequence(0, capacity=seq)
        batch = Batch(BatchKind.PREFILL, [BatchItem(s, prompt)])

        def step():
            s.cache.truncate(0)
            eng.step(batch, mode=ParallelMode.SP)
        ms = timed(step, 3, warm=1)
        rec = eng.step_records[-1]
        out[label] = (ms, rec.flops_total)
        del eng
        torch.cuda.empty_cache()
    gemm_tok = gemm_flops_per_token(cfg)
    std_ms, std_fl = out["standard"]
    skv_ms, skv_fl = out["swiftkv"]
    print(json.dumps({"config": "swiftkv 32K prefill (configs[4])", "n_gpus": 1, "seq_len": seq,
                      "cut_layer": cut, "standard_ms": round(std_ms, 2),
                      "standard_tokens_per_s": round(seq / std_ms * 1e3, 1),
                      "swiftkv_ms": round(skv_ms, 2),
                      "swiftkv_tokens_per_s": round(seq / skv_ms * 1e3, 1),
                      "speedup": round(std_ms / skv_ms, 3),
                      "metered_flop_ratio": round(skv_fl / std_fl, 4),
                      "swiftkv_tflops_metered_fullwindow": round(skv_fl / (skv_ms / 1e3) / 1e12, 1)}),
          flush=True)


def model_70b(seq=8192, dec_b=16, ctx=2048):
    """configs[3] model geometry on ONE B200: Llama-3.3-70B bf16 replica (141 GB):
    8K single-request prefill tok/s and decode TPOT at B=16, ctx 2K."""
    from paper_2507_11830_b200 import llama33_70b
    cfg = llama33_70b(max_seq=max(seq, ctx + 64))
    w = ModelWeights.random(cfg, seed=0, world_size=1)
    rng = np.random.default_rng(2)
    blocks = -(-seq // 64) + dec_b * -(-(ctx + 64) // 64) + 8
    eng = Engine(w, LoopbackGroup(1), ShiftPolicy.fixed_sp(), num_blocks=blocks)
    prompt = [int(t) for t in rng.integers(0, cfg.vocab_size, size=seq)]
    s = eng.new_sequence(0, capacity=seq)
    batch = Batch(BatchKind.PREFILL, [BatchItem(s, prompt)])

    def pre():
        s.cache.truncate(0)
        eng.step(batch, mode=ParallelMode.SP)
    ms = timed(pre, 3, warm=1)
    gemm_fl = gemm_flops_per_token(cfg) * seq
    attn_fl = causal_attention_flops(cfg, [seq], [0])
    seqs = [eng.new_sequence(10 + i, capacity=ctx + 64) for i in range(dec_b)]
    for i in range(0, dec_b, 4):
        eng.step(Batch(BatchKind.PREFILL, [BatchItem(q, [int(t) for t in rng.integers(0, 1000, ctx)])
                                           for q in seqs[i:i + 4]]), mode=ParallelMode.SP)

    def dec():
        for q in seqs:
            q.cache.truncate(ctx)
        eng.step(Batch(BatchKind.DECODE, [BatchItem(q, [1]) for q in seqs]), mode=ParallelMode.TP)
    tpot = timed(dec, 8, warm=3)
    wbytes = w.nbytes() - w.embed.nbytes  # the embedding is gathered, not streamed
    kv = dec_b * ctx * cfg.n_layers * 2 * cfg.kv_heads * cfg.head_dim * 2
    roof = (wbytes + kv) / (PEAKS["hbm_gbs"] * 1e9) * 1e3
    print(json.dumps({"config": "llama-3.3-70b geometry on 1x B200 (configs[3] model)",
                      "weights_gb": round(wbytes / 1e9, 1), "prefill_seq": seq,
                      "prefill_ms": round(ms, 2), "prefill_tokens_per_s": round(seq / ms * 1e3, 1),
                      "prefill_tflops": round((gemm_fl + attn_fl) / (ms / 1e3) / 1e12, 1),
                      "decode_batch": dec_b, "decode_ctx": ctx, "tpot_ms": round(tpot, 3),
                      "decode_hbm_roofline_ms": round(roof, 3),
                      "decode_frac_of_roofline": round(roof / tpot, 4)}), flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    torch.cuda.set_device(0)
    if what == "70b":
        model_70b()
        sys.exit(0)
    cfg = llama31_8b(max_seq=32768 + 64)
    weights = ModelWeights.random(cfg, seed=0, world_size=1)
    if what in ("decode-sweep", "all"):
        decode_sweep(weights, cfg)
    if what in ("swiftkv", "all"):
        swiftkv(weights, cfg)
