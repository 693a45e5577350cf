#!/usr/bin/env python
"""Shift-Parallel forward benchmark on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1: run under torchrun (one rank per GPU, NCCL), or let bench.py spawn
``torch.distributed.run`` itself when WORLD_SIZE is unset.

Workload (BASELINE.json configs[1]): Llama-3.1-8B geometry, random-init bf16
weights, one 8192-token request prefilled in Ulysses SP mode over N GPUs
(strong scaling: the same request at every N).  A "step" is one full prefill
pass (32 layers + LM head of the last token) on a logically truncated KV
cache.  The rest of the metric's matrix rides along in the same line: the
same prefill in TP mode, and decode TPOT at B=1 and B=64 (ctx 2K) in TP and
SP mode plus the mode the shift policy picks (configs[2] points), each with
its roofline fraction.

`value` = SP prefill tokens/s with inputs resident (device-timed with CUDA
events, barrier + synchronize around the K steps, max over ranks); `e2e` =
the same through Engine.step with host token lists, pinned H2D of the step
metadata and a D2H of the logits inside the timed region (wall clock,
synchronised, max over ranks).  `--impl reference` times the reference
algorithm (the oracle port of shiftsim, f32 numpy einsum, simulated SP ranks
on host threads) on bounded one-layer samples, extrapolated by a two-point fit.
"""

from __future__ import annotations

import argparse
import glob
import json
import os
import socket
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
    ap.add_argument("--no-tp", action="store_true", help="skip the TP-mode prefill cell")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def peaks():
    p = {"src": "measured (MEASURED_PEAKS.json)"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p.update(json.load(f))
    except OSError:  # B200_PROFILING.md fallback figures
        p.update({"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                  "src": "fallback (B200_PROFILING.md)"})
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
    capture of this workload (tools/ncu_traffic.py)."""
    for name in ("r02_traffic_final.json", "r02_traffic.json", "r01_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                return round(json.load(f)["kernels"][kernel]["dram_bytes_per_launch"])
        except (OSError, KeyError, ValueError):
            continue
    return None


# ------------------------------------------------------------- N>1 launcher
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(args) -> int:
    """`python bench.py --gpus N` without torchrun: launch N ranks through
    torch.distributed.run on this node (rank 0 prints the JSON line)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


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
    """The reference algorithm (oracle port of shiftsim, f32 np.einsum) on ONE
    Llama-3.1-8B-width layer, SP over simulated ranks on host threads (the
    reference's own threading, fabric.py:57-80).  Full-workload tokens/s come
    from a two-point fit of the per-layer time against the
    layer's FLOPs as the reference executes them:

        F(M) = M * G + 4 * d * H * M^2     (projections + full-window attention,
                                            flops.py:116-117)
        T(M) = c + k * F(M)                (fixed overhead + seconds per FLOP)

    through the measured T(512) and T(1024), extrapolated to the 8192-token
    request and x32 layers.  (A free a*M + b*M^2 fit is ill-posed here: at
    M <= 1024 the fixed per-pass overhead hides the quadratic term and b comes
    out <= 0.)  Embedding/LM head of one row excluded — vocab-256 stand-in."""

    POINTS = (512, 1024)

    def __init__(self, threads: int, layers_model: int = 32, seq: int = 8192):
        import numpy as np

        from oracle.model import init_weights_llama, llama_tiny_config

        self.p = threads if threads in (1, 2, 4, 8) else 1
        self.layers_model, self.seq = layers_model, seq
        cfg = llama_tiny_config(n_layers=1, n_heads=32, n_kv_heads=8, head_dim=128,
                                ffn_dim=14336, vocab_size=256, max_seq=max(self.POINTS))
        self.cfg = cfg
        self.w = init_weights_llama(cfg, seed=0, bf16=True)
        self.rng = np.random.default_rng(0)
        self.times = {m: [] for m in self.POINTS}

    def layer_flops(self, m: int) -> int:
        c = self.cfg
        h, d, f = c.hidden, c.head_dim, c.ffn_dim
        g = 2 * h * (c.n_heads + 2 * c.kv_heads) * d + 2 * c.n_heads * d * h + 3 * 2 * h * f
        return m * g + 4 * d * c.n_heads * m * m

    def layer_seconds(self, tokens: int) -> float:
        import oracle
        toks = [int(t) for t in self.rng.integers(0, 256, size=tokens)]
        eng = oracle.OracleEngine(self.w, self.p, kind="fixed_sp", threaded=self.p > 1)
        s = eng.new_sequence(0, capacity=tokens)
        t0 = time.perf_counter()
        eng.step([(s, toks)], mode="sp")
        dt = time.perf_counter() - t0
        eng.group.close()
        self.times[tokens].append(dt)
        return dt

    def fit(self):
        (m1, m2) = self.POINTS
        t1, t2 = statistics.mean(self.times[m1]), statistics.mean(self.times[m2])
        f1, f2 = self.layer_flops(m1), self.layer_flops(m2)
        k = max(t2 - t1, 1e-9) / (f2 - f1)
        c = max(0.0, t1 - k * f1)
        t_full = self.layers_model * (c + k * self.layer_flops(self.seq))
        return c, k, t1, t2, t_full

    def describe(self) -> dict:
        c, k, t1, t2, t_full = self.fit()
        return {"value": self.seq / t_full, "unit": "tokens/s", "cores": self.p, "kind": "port",
                "sample": (f"oracle port (shiftsim algorithm, f32 np.einsum) of ONE Llama-3.1-8B-"
                           f"width layer (GQA 32q/8kv, SwiGLU 14336), SP over {self.p} simulated "
                           f"ranks on host threads, timed at M={self.POINTS[0]} "
                           f"({t1:.2f} s, n={len(self.times[self.POINTS[0]])}) and "
                           f"M={self.POINTS[1]} ({t2:.2f} s, n={len(self.times[self.POINTS[1]])}); "
                           f"T(M) = c + k*F(M), F(M) = M*G + 4dH*M^2 (layer FLOPs as the reference "
                           f"executes them), c={c:.3g} s, 1/k={1 / k / 1e9:.3g} GFLOP/s; full step "
                           f"= {self.layers_model} x T({self.seq}) = {t_full:.0f} s; vocab-256 "
                           f"stand-in, embedding/LM head excluded")}


def host_threads() -> int:
    n = min(8, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))
    return max(t for t in (1, 2, 4, 8) if t <= n)


def run_reference(args):
    """The reference arm: rank 0 only (other torchrun ranks exit without work).
    Each step is ONE bounded one-layer sample, alternating M=512 / M=1024; the
    line's value is the two-point fit over all timed steps."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    smp = CpuSample(host_threads(), seq=args.seq)
    ms = []
    n = args.warmup + args.steps
    for i in range(n):
        m = smp.POINTS[i % 2]
        dt = smp.layer_seconds(m)
        if i < args.warmup:
            smp.times[m].pop()
        else:
            ms.append(dt * 1e3)
    for m in smp.POINTS:  # a fit needs both points even with steps == 1
        if not smp.times[m]:
            smp.layer_seconds(m)
    cb = smp.describe()
    v = cb["value"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            # a step is one bounded sample (wall clock); the full 8K prefill it stands for
            # would take ms_per_full_step_extrapolated
            "ms_per_step": statistics.mean(ms), "ms_per_full_step_extrapolated": args.seq / v * 1e3,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args, args.gpus),
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- NCCL
def nccl_log_setup() -> str:
    """Route NCCL's INIT log to a per-process file (keeps stdout one JSON line)."""
    d = tempfile.mkdtemp(prefix="sp_nccl_")
    if "NCCL_DEBUG" not in os.environ:
        os.environ["NCCL_DEBUG"] = "INFO"
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ["NCCL_DEBUG_FILE"] = os.path.join(d, "nccl.%h.%p.log")
    return d


def nccl_comm_lines(d: str):
    out = []
    for p in glob.glob(os.path.join(d, "*.log")):
        with open(p, errors="replace") as f:
            out += [l.strip() for l in f if "nRanks" in l and "comm 0x" in l]
    return out


# ------------------------------------------------------------------- ours
def run_ours(args):
    import numpy as np
    import torch

    from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, Engine, LoopbackGroup,
                                       NcclGroup, ParallelMode, ShiftPolicy, choose_mode,
                                       default_token_threshold, llama31_8b, ops)
    from paper_2507_11830_b200.flops import causal_attention_flops, gemm_flops_per_token
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
    nccl_dir = None
    if world > 1:
        import torch.distributed as dist
        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            nccl_dir = nccl_log_setup()
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()
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
    num_blocks = -(-args.seq // bs) + (dec_b + 1) * -(-(args.decode_ctx + 64) // bs) + 8
    eng = Engine(weights, group, ShiftPolicy.fixed_sp(), num_blocks=num_blocks, block_size=bs)
    rng = np.random.default_rng(1234)
    prompt = [int(t) for t in rng.integers(0, cfg.vocab_size, size=args.seq)]
    seq = eng.new_sequence(0, capacity=args.seq)
    batch = Batch(BatchKind.PREFILL, [BatchItem(seq, prompt)])

    def prefill(mode=ParallelMode.SP):
        seq.cache.truncate(0)
        return eng.step(batch, mode=mode)[0]

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

    attn_causal = causal_attention_flops(cfg, [args.seq], [0])
    step_flops = gemm_flops_per_token(cfg) * args.seq + attn_causal + 2 * cfg.hidden * cfg.vocab_size

    def timed(fn, k):
        sync_barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            fn()
        e1.record()
        sync_barrier()
        return max_over_ranks(e0.elapsed_time(e1)) / k

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

    def agg(p, kind):
        recs = p.get(kind, [])
        if not recs:
            return None
        t = sum(a.elapsed_time(b) for a, b, _, _ in recs)
        return t, sum(f for _, _, f, _ in recs), sum(b for _, _, _, b in recs), len(recs)

    g = agg(prof, "gemm")
    a = agg(prof, "attn_prefill")
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
                "frac_sustained": round(a[1] / (a[0] / 1e3) / 1e12 / pk["bf16_tflops_sustained"], 4),
                "share_of_step": round(a[0] / prof_ms, 4), "launches": a[3],
                "causal_flops_per_step": a[1] // args.steps}

    def prefill_cell(ms):
        tf = step_flops / world / (ms / 1e3) / 1e12   # per-GPU achieved
        return {"tokens_per_s": round(args.seq / (ms / 1e3), 1), "ms_per_step": round(ms, 3),
                "tflops_per_gpu": round(tf, 1),
                "frac_tensor_sustained": round(tf / pk["bf16_tflops_sustained"], 4)}

    whole = prefill_cell(ms_step)
    matrix = {"prefill": {"sp": whole}}
    if not args.no_tp:
        for _ in range(2):
            prefill(ParallelMode.TP)
        matrix["prefill"]["tp"] = prefill_cell(timed(lambda: prefill(ParallelMode.TP), args.steps))
    if world == 1:
        matrix["prefill"]["note"] = "P=1: TP and SP are the same single-device computation"

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

    # ---------------- decode TPOT: B requests at ctx, TP / SP / shift
    decode = None
    decode_cells = {}
    if dec_b:
        # decode streams the layer weights + LM head (the embedding table is
        # only gathered: B rows) and every request's KV window
        wbytes = weights.nbytes() - weights.embed.nbytes
        tau = default_token_threshold(world, cfg)   # B200 crossover (shift_cost)
        for B in sorted({1, dec_b}):
            seqs = [eng.new_sequence(100 + 1000 * B + i, capacity=args.decode_ctx + 64)
                    for i in range(B)]
            ctx_prompts = [[int(t) for t in rng.integers(0, cfg.vocab_size, size=args.decode_ctx)]
                           for _ in range(B)]
            chunk = max(1, 16384 // args.decode_ctx)
            for i in range(0, B, chunk):  # prefill contexts in SP, 16K tokens per pass
                eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, p) for s, p in
                                                   zip(seqs[i:i + chunk], ctx_prompts[i:i + chunk])]),
                         mode=ParallelMode.SP)
            toks = [1] * B
            dbatch = lambda: Batch(BatchKind.DECODE, [BatchItem(s, [t]) for s, t in zip(seqs, toks)])

            def dstep(mode):
                return eng.step(dbatch(), mode=mode)[0]

            def roll_back():  # keep the context at ctx: every step decodes position ctx
                for s in seqs:
                    s.cache.truncate(args.decode_ctx)

            kv_bytes = B * (args.decode_ctx + 1) * cfg.n_layers * 2 * (cfg.kv_heads // world) \
                * cfg.head_dim * 2
            row = {}
            for mode in (ParallelMode.TP, ParallelMode.SP):
                # eager, capture, then replays until the TPOT is steady (the
                # first replays after a prefill-heavy phase run ~5% slow)
                for _ in range(12):
                    dstep(mode)
                    roll_back()
                n_dec = 32

                def one():
                    dstep(mode)
                    roll_back()
                tpot = timed(one, n_dec)
                wb = wbytes // world if mode is ParallelMode.TP else wbytes
                roof = (wb + kv_bytes) / (pk["hbm_gbs"] * 1e9) * 1e3
                row[mode.value] = {"tpot_ms": round(tpot, 4), "hbm_roofline_ms": round(roof, 4),
                                   "frac_hbm_roofline": round(roof / tpot, 4),
                                   "bytes_per_step": wb + kv_bytes}
            m_shift = choose_mode(ShiftPolicy(token_threshold=tau), dbatch())
            row["shift"] = {"tau": tau, "tau_reference_4P": default_token_threshold(world),
                            "picks": m_shift.value, **row[m_shift.value]}
            if world == 1:
                row["note"] = "P=1: TP and SP are the same single-device computation"
            decode_cells[f"b{B}"] = row
            for s in seqs:
                eng.release(s)
        matrix["decode"] = {"ctx": args.decode_ctx, **decode_cells}
        # per-kernel shares of the B=dec_b TP decode from eager passes (graph
        # replays carry no per-op events)
        seqs = [eng.new_sequence(900000 + i, capacity=args.decode_ctx + 64) for i in range(dec_b)]
        chunk = max(1, 16384 // args.decode_ctx)
        for i in range(0, dec_b, chunk):
            eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, [int(t) for t in rng.integers(
                0, cfg.vocab_size, size=args.decode_ctx)]) for s in seqs[i:i + chunk]]),
                mode=ParallelMode.SP)
        eng.cuda_graphs = False
        ops.PROFILE = {}

        def eager():
            eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [1]) for s in seqs]), mode=ParallelMode.TP)
            for s in seqs:
                s.cache.truncate(args.decode_ctx)
        tpot_eager = timed(eager, 8)
        dprof, ops.PROFILE = ops.PROFILE, None
        eng.cuda_graphs = True
        ad = agg(dprof, "attn_decode")
        gd = agg(dprof, "gemm")
        cell = decode_cells[f"b{dec_b}"]["tp"]
        decode = {"tpot_ms": cell["tpot_ms"], "tpot_ms_eager": round(tpot_eager, 4),
                  "cuda_graphs": not getattr(group, "_stage", False), "batch": dec_b,
                  "ctx": args.decode_ctx, "mode": "tp",
                  "hbm_roofline_tpot_ms": cell["hbm_roofline_ms"],
                  "frac_of_hbm_roofline": cell["frac_hbm_roofline"],
                  "roofline_bytes": "layer weights + LM head (/P in TP) + B x ctx KV; the "
                                    "embedding table (gathered, not streamed) is excluded",
                  "attn_decode": {"achieved_gbs": round(ad[2] / (ad[0] / 1e3) / 1e9, 1),
                                  "frac_hbm": round(ad[2] / (ad[0] / 1e3) / 1e9 / pk["hbm_gbs"], 4),
                                  "share_of_eager_step": round(ad[0] / (tpot_eager * 8), 4)} if ad else None,
                  "gemm": {"achieved_gbs": round(gd[2] / (gd[0] / 1e3) / 1e9, 1),
                           "share_of_eager_step": round(gd[0] / (tpot_eager * 8), 4)} if gd else None}

    cpu_base = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            smp = CpuSample(host_threads(), seq=args.seq)
            for m in smp.POINTS:
                smp.layer_seconds(m)
            cpu_base = smp.describe()
        except Exception as e:  # keep the GPU line even if the host sample fails
            cpu_base = {"error": repr(e)}
    nccl = None
    if nccl_dir is not None:
        lines = nccl_comm_lines(nccl_dir)
        nccl = {"comm_init": lines[:1], "n_comm_lines": len(lines)}
        for l in lines[:1]:
            print(f"[rank {rank}] NCCL {l}", file=sys.stderr, flush=True)

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (random-init N(0,0.02^2) bf16 weights, uniform token ids)",
                "config": workload_config(args, world),
                "roofline": roofline, "attention": attn, "whole_step": whole,
                "matrix": matrix,
                "decode": decode, "decode_tpot_ms": decode["tpot_ms"] if decode else None,
                "e2e": {"value": round(e2e_val, 1), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h},
                "gpu_launches": launches, "clocks": clk, "cpu_baseline": cpu_base,
                "nccl": nccl}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
