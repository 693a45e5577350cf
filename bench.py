#!/usr/bin/env python
"""Shift-Parallel forward benchmark on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1, one rank per GPU)

Workload (BASELINE.json configs[1]): Llama-3.1-8B geometry, random-init bf16
weights, one 8192-token request prefilled in Ulysses SP mode over N GPUs
(strong scaling: the same request at every N).  A "step" is one full prefill
pass (32 layers + LM head of the last token) on a logically truncated KV
cache.  Also measured (second number of the metric): decode TPOT for a batch
of 64 requests at 2K context in TP mode.

`value` = tokens/s with inputs resident (device-timed with CUDA events,
barrier + synchronize around the K steps, max over ranks); `e2e` = the same
through Engine.step with host token lists, pinned H2D of the step metadata and
a D2H of the logits inside the timed region (wall clock, synchronised).
`--impl reference` times the reference algorithm (the oracle port of shiftsim,
f32 numpy einsum, simulated SP ranks on host threads) on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "prefill tokens/s and decode TPOT (ms) at 1/2/4/8 B200, SP vs TP mode"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seq", type=int, default=8192)
    ap.add_argument("--layers", type=int, default=None, help="debug: truncate depth (invalid for bench)")
    ap.add_argument("--decode-batch", type=int, default=64)
    ap.add_argument("--decode-ctx", type=int, default=2048)
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def peaks():
    p = {"hbm_gbs": 6552.3, "bf16_tflops": 1634.7, "bf16_tflops_sustained": 1366.3, "src": "measured"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p.update(json.load(f))
    except OSError:
        p.update({"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                  "src": "fallback"})
    return p


def workload_config(args, world: int) -> dict:
    """The workload both arms report (BASELINE configs[1]); how the reference
    arm samples it is stated in its cpu_baseline.sample."""
    name = "llama-3.1-8b-geometry single-request 8K-token prefill, Ulysses SP"
    if args.layers:
        name += f" (TRUNCATED to {args.layers} layers: debug only, not a bench value)"
    return {"workload": name, "seq_len": args.seq, "requests": 1, "parallelism": f"sp{world}",
            "l2": "inputs larger than L2 (16 GB of weights streamed per step)"}


def traffic_per_launch(kernel: str):
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu
    capture of this workload (profiles/r01_traffic.json, tools/ncu_traffic.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_traffic.json")) as f:
            return round(json.load(f)["kernels"][kernel]["dram_bytes_per_launch"])
    except (OSError, KeyError, ValueError):
        return None


# ----------------------------------------------------------------- clocks
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                c = [x.strip() for x in line.split(",")]
                if len(c) < 9:
                    continue
                try:
                    sm.append(float(c[1]))
                    mx = max(mx, float(c[2]))
                except ValueError:
                    continue
                for n, v in zip(names, c[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ CPU baseline
class CpuSample:
    """The reference algorithm (oracle port of shiftsim, f32 np.einsum) on one
    Llama-3.1-8B-width layer over `tokens` prompt tokens, SP over simulated
    ranks on host threads (the reference's own threading, fabric.py:57-80);
    tokens/s extrapolated x32 layers."""

    def __init__(self, threads: int, tokens: int = 128, layers_model: int = 32):
        import numpy as np

        from oracle.model import init_weights_llama, llama_tiny_config

        self.p = threads if threads in (1, 2, 4, 8) else 1
        self.tokens, self.layers_model = tokens, layers_model
        cfg = llama_tiny_config(n_layers=1, n_heads=32, n_kv_heads=8, head_dim=128,
                                ffn_dim=14336, vocab_size=256, max_seq=max(tokens, 256))
        self.w = init_weights_llama(cfg, seed=0, bf16=True)
        self.rng = np.random.default_rng(0)

    def run(self) -> float:
        import oracle
        toks = [int(t) for t in self.rng.integers(0, 256, size=self.tokens)]
        eng = oracle.OracleEngine(self.w, self.p, kind="fixed_sp", threaded=self.p > 1)
        s = eng.new_sequence(0, capacity=self.tokens)
        t0 = time.perf_counter()
        eng.step([(s, toks)], mode="sp")
        dt = time.perf_counter() - t0
        eng.group.close()
        self.last_ms = dt * 1e3
        return self.tokens / dt / self.layers_model

    def describe(self, value: float) -> dict:
        return {"value": value, "unit": "tokens/s", "cores": self.p, "kind": "port",
                "sample": (f"oracle port (shiftsim algorithm, f32 np.einsum) of ONE "
                           f"Llama-3.1-8B-width layer (GQA 32q/8kv, SwiGLU 14336) over "
                           f"{self.tokens} prompt tokens, SP over {self.p} simulated ranks on host "
                           f"threads; tokens/s extrapolated x{self.layers_model} layers; vocab-256 "
                           f"stand-in so embedding/LM head are excluded")}


def host_threads() -> int:
    n = min(8, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))
    return max(t for t in (1, 2, 4, 8) if t <= n)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    smp = CpuSample(host_threads())
    vals, ms = [], []
    for i in range(args.warmup + args.steps):
        v = smp.run()
        if i >= args.warmup:
            vals.append(v)
            ms.append(smp.last_ms)
    v = statistics.mean(vals)
    cb = smp.describe(v)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            # a step is the bounded sample (wall clock); the full 8K prefill it stands for
            # would take ms_per_full_step_extrapolated
            "ms_per_step": statistics.mean(ms), "ms_per_full_step_extrapolated": 8192 / v * 1e3,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args, args.gpus),
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- ours
def run_ours(args):
    import numpy as np
    import torch

    from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, Engine, LoopbackGroup,
                                       NcclGroup, ParallelMode, ShiftPolicy, llama31_8b, ops)
    from paper_2507_11830_b200.flops import gemm_flops_per_token
    from paper_2507_11830_b200.weights import ModelWeights

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # SP_BENCH_BACKEND=gloo (test only): several ranks share the GPUs present,
    # collectives staged through host memory — exercises the N>1 plumbing on a
    # 1-GPU box; measured runs use NCCL, one rank per GPU
    backend = os.environ.get("SP_BENCH_BACKEND", "nccl")
    dev_idx = local % torch.cuda.device_count() if backend == "gloo" else local
    torch.cuda.set_device(dev_idx)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ops.device_check()
    pk = peaks()

    ctx_needed = max(args.seq, args.decode_ctx + 64)
    kw = dict(max_seq=ctx_needed)
    if args.layers:
        kw["n_layers"] = args.layers
    cfg = llama31_8b(**kw)
    weights = ModelWeights.random(cfg, seed=0, world_size=world)
    group = NcclGroup() if world > 1 else LoopbackGroup(1)
    bs = 64
    dec_b = 0 if args.no_decode else args.decode_batch
    num_blocks = -(-args.seq // bs) + dec_b * -(-(args.decode_ctx + 64) // bs) + 8
    eng = Engine(weights, group, ShiftPolicy.fixed_sp(), num_blocks=num_blocks, block_size=bs)
    rng = np.random.default_rng(1234)
    prompt = [int(t) for t in rng.integers(0, cfg.vocab_size, size=args.seq)]
    seq = eng.new_sequence(0, capacity=args.seq)
    batch = Batch(BatchKind.PREFILL, [BatchItem(seq, prompt)])

    def prefill():
        seq.cache.truncate(0)
        return eng.step(batch, mode=ParallelMode.SP)[0]

    def sync_barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        prefill()
    # ---------------- timed region: device-resident inputs, CUDA events
    sync_barrier()
    clocks = Clocks(dev_idx)
    clocks.start()
    launches0 = ops.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        prefill()
    ev1.record()
    sync_barrier()
    launches = ops.kernel_launches() - launches0
    clk = clocks.stop()
    elapsed_ms = max_over_ranks(ev0.elapsed_time(ev1))
    ms_step = elapsed_ms / args.steps
    value = args.seq * args.steps / (elapsed_ms / 1e3)
    # per-kernel CUDA events (roofline numerator) in a separate pass of the same
    # K steps: events between launches break the PDL overlap, so they stay out
    # of the timed region above
    ops.PROFILE = {}
    ep0, ep1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ep0.record()
    for _ in range(args.steps):
        prefill()
    ep1.record()
    sync_barrier()
    prof, ops.PROFILE = ops.PROFILE, None
    prof_ms = max_over_ranks(ep0.elapsed_time(ep1))

    def agg(kind):
        recs = prof.get(kind, [])
        if not recs:
            return None
        t = sum(a.elapsed_time(b) for a, b, _, _ in recs)
        return t, sum(f for _, _, f, _ in recs), sum(b for _, _, _, b in recs), len(recs)

    g = agg("gemm")
    a = agg("attn_prefill")
    gemm_ms, gemm_fl, gemm_b, gemm_n = g
    achieved = gemm_fl / (gemm_ms / 1e3) / 1e12
    roofline = {"bound": "tensor", "kernel": "sp_gemm_bf16 (tcgen05)", "achieved": round(achieved, 1),
                "peak": pk["bf16_tflops_sustained"], "unit": "TFLOP/s",
                "frac": round(achieved / pk["bf16_tflops_sustained"], 4),
                "peak_kind": f"{pk['src']} sustained cuBLAS bf16",
                "frac_of_burst": round(achieved / pk["bf16_tflops"], 4),
                "launches": gemm_n, "avg_launch_ms": round(gemm_ms / gemm_n, 4),
                "share_of_step": round(gemm_ms / prof_ms, 4),
                "algorithmic_flops_per_step": gemm_fl // args.steps,
                "algorithmic_bytes_per_launch": gemm_b // max(gemm_n, 1),
                "traffic": traffic_per_launch("sp_gemm_bf16")}
    attn = None
    if a:
        attn = {"kernel": "sp_attention prefill (tcgen05/TMEM, paged, GQA-packed)",
                "achieved_tflops": round(a[1] / (a[0] / 1e3) / 1e12, 1),
                "share_of_step": round(a[0] / prof_ms, 4), "launches": a[3],
                "causal_flops_per_step": a[1] // args.steps}
    step_flops = gemm_flops_per_token(cfg) * args.seq + (a[1] // args.steps if a else 0)
    whole = {"tflops": round(step_flops / (ms_step / 1e3) / 1e12, 1),
             "frac_sustained": round(step_flops / (ms_step / 1e3) / 1e12 / pk["bf16_tflops_sustained"], 4)}

    # ---------------- e2e through the public API (host in, host out)
    e2e_times = []
    h2d = d2h = 0
    for i in range(max(3, args.steps // 2) + 1):
        sync_barrier()
        t0 = time.perf_counter()
        seq.cache.truncate(0)
        lg, rec = eng.step(Batch(BatchKind.PREFILL, [BatchItem(seq, prompt)]), mode=ParallelMode.SP)
        host_logits = lg[0].cpu()
        sync_barrier()
        dt = time.perf_counter() - t0
        if i > 0:
            e2e_times.append(max_over_ranks(dt))
        d2h = host_logits.numel() * host_logits.element_size()
    h2d = eng.last_h2d_bytes
    e2e_val = args.seq / statistics.mean(e2e_times)

    # ---------------- decode TPOT (TP mode, B requests at ctx)
    decode = None
    if dec_b:
        seqs = [eng.new_sequence(100 + i, capacity=args.decode_ctx + 64) for i in range(dec_b)]
        ctx_prompts = [[int(t) for t in rng.integers(0, cfg.vocab_size, size=args.decode_ctx)]
                       for _ in range(dec_b)]
        chunk = max(1, 16384 // args.decode_ctx)
        for i in range(0, dec_b, chunk):  # prefill contexts in SP, 16K tokens per pass
            eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, p) for s, p in
                                               zip(seqs[i:i + chunk], ctx_prompts[i:i + chunk])]),
                     mode=ParallelMode.SP)
        toks = [1] * dec_b

        def dstep():
            return eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [t]) for s, t in zip(seqs, toks)]),
                            mode=ParallelMode.TP)[0]

        n_dec = 16
        for _ in range(3):
            dstep()
        sync_barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n_dec):  # CUDA-graph replays (captured during warm-up)
            dstep()
        e1.record()
        sync_barrier()
        tpot = max_over_ranks(e0.elapsed_time(e1)) / n_dec
        # per-kernel shares from an eager pass (graph replays carry no per-op events)
        eng.cuda_graphs = False
        sync_barrier()
        ops.PROFILE = {}
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record()
        for _ in range(n_dec):
            dstep()
        e3.record()
        sync_barrier()
        dprof, ops.PROFILE = ops.PROFILE, None
        eng.cuda_graphs = True
        tpot_eager = max_over_ranks(e2.elapsed_time(e3)) / n_dec
        ad = dprof.get("attn_decode", [])
        ad_ms = sum(x.elapsed_time(y) for x, y, _, _ in ad)
        ad_b = sum(b for _, _, _, b in ad)
        gd = dprof.get("gemm", [])
        gd_ms = sum(x.elapsed_time(y) for x, y, _, _ in gd)
        gd_b = sum(b for _, _, _, b in gd)
        wbytes = weights.nbytes() // 1  # whole replica (TP views of it at P > 1)
        kv_bytes = dec_b * (args.decode_ctx + 20) * cfg.n_layers * 2 * (cfg.kv_heads // world) * cfg.head_dim * 2
        step_bytes = wbytes // world + kv_bytes
        decode = {"tpot_ms": round(tpot, 4), "tpot_ms_eager": round(tpot_eager, 4),
                  "cuda_graphs": not getattr(group, "_stage", False), "batch": dec_b, "ctx": args.decode_ctx, "mode": "tp",
                  "hbm_roofline_tpot_ms": round(step_bytes / (pk["hbm_gbs"] * 1e9) * 1e3, 4),
                  "frac_of_hbm_roofline": round(step_bytes / (pk["hbm_gbs"] * 1e9) * 1e3 / tpot, 4),
                  "attn_decode": {"achieved_gbs": round(ad_b / (ad_ms / 1e3) / 1e9, 1) if ad_ms else None,
                                  "frac_hbm": round(ad_b / (ad_ms / 1e3) / 1e9 / pk["hbm_gbs"], 4) if ad_ms else None,
                                  "share_of_eager_step": round(ad_ms / (tpot_eager * n_dec), 4)},
                  "gemm": {"achieved_gbs": round(gd_b / (gd_ms / 1e3) / 1e9, 1) if gd_ms else None,
                           "share_of_eager_step": round(gd_ms / (tpot_eager * n_dec), 4)}}

    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            smp = CpuSample(host_threads())
            cpu_base = smp.describe(smp.run())
        except Exception as e:  # keep the GPU line even if the host sample fails
            cpu_base = {"error": repr(e)}

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (random-init N(0,0.02^2) bf16 weights, uniform token ids)",
                "config": workload_config(args, world),
                "roofline": roofline, "attention": attn, "whole_step": whole,
                "decode": decode, "decode_tpot_ms": decode["tpot_ms"] if decode else None,
                "e2e": {"value": round(e2e_val, 1), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h},
                "gpu_launches": launches, "clocks": clk, "cpu_baseline": cpu_base}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
