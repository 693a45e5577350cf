"""Continuous-batching serving driver over the Shift-Parallel engine (wall clock).

Follows the scheduling semantics of the reference driver
(/root/reference/pkg/src/shiftsim/serving.py:311-517) with the simulated
FLOP/byte clock replaced by real time:

* requests are admitted when their arrival time has passed; a request whose
  prompt plus output budget exceeds ``max_seq`` is rejected up front (:333-344);
* if anything is queued, ONE prefill pass runs over every queued prompt,
  otherwise ONE decode pass over every decoding request — prefill and decode
  are never mixed in a pass (:401-514);
* each pass picks its parallel mode with the engine policy (``choose_mode``,
  the per-pass SP<->TP shift on one KV pool);
* TTFT = first token time - arrival, TPOT = (last - first) / (tokens - 1),
  nearest-rank percentiles (:523-560); finished sequences release their
  paged KV blocks.

With a ``CostModel`` the driver runs on the reference's LOGICAL clock instead
(serving.py:226-244: each pass advances simulated time by
flops_max_device / device_flops_per_s + sum over collectives of
bytes / link_bytes_per_s + latency): arrivals are admitted against simulated
time, an idle driver jumps to the next arrival, and no wall time is read — the
pass schedule is then a deterministic function of the trace, the policy and
the step records, directly comparable with ``run_serving_loop``.

Trace files use the reference's JSON-lines format (arrival_ms, prompt_len,
output_len, corpus), so reference traces replay unchanged.
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from .engine import Batch, BatchItem, BatchKind, Engine, choose_mode, greedy_tokens
from .errors import CacheOverflow, ContractViolation


@dataclass(frozen=True)
class TraceEntry:
    request_id: int
    arrival_ms: int
    prompt_len: int
    output_len: int
    corpus: str = "random"


def bursty_trace(phases: Sequence[Tuple[float, float]], prompt_len: int, output_len: int,
                 seed: int, corpus: str = "random") -> List[TraceEntry]:
    """Seeded Poisson arrivals over (duration_ms, rate_per_s) phases with fixed
    lengths (BASELINE configs[3]: low-traffic then burst, 2K prompts, 256 out)."""
    rng = np.random.default_rng([seed, 0xB0057])
    out: List[TraceEntry] = []
    start = 0.0
    for dur, rate in phases:
        if rate > 0:
            gap = 1000.0 / rate
            t = start + rng.exponential(gap)
            while t < start + dur:
                out.append(TraceEntry(len(out), int(t), prompt_len, output_len, corpus))
                t += rng.exponential(gap)
        start += dur
    return out


def write_trace(path: str, entries: Sequence[TraceEntry]) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        for e in entries:
            fh.write(json.dumps({"arrival_ms": e.arrival_ms, "prompt_len": e.prompt_len,
                                 "output_len": e.output_len, "corpus": e.corpus},
                                sort_keys=True) + "\n")


def read_trace(path: str) -> List[TraceEntry]:
    rows = []
    with open(path, "r", encoding="utf-8") as fh:
        for n, line in enumerate(fh, start=1):
            line = line.strip()
            if not line:
                continue
            try:
                obj = json.loads(line)
                extra = set(obj) - {"arrival_ms", "prompt_len", "output_len", "corpus"}
                if extra:
                    raise ValueError(f"unknown keys {sorted(extra)}")
                row = (int(obj["arrival_ms"]), int(obj["prompt_len"]), int(obj["output_len"]),
                       str(obj.get("corpus", "random")))
                if row[0] < 0 or row[1] < 1 or row[2] < 1 or row[3] not in ("random", "repetitive"):
                    raise ValueError("field out of range")
            except (KeyError, TypeError, ValueError) as exc:
                raise ContractViolation(f"{path}:{n}: bad trace line: {exc}") from exc
            rows.append(row)
    rows.sort(key=lambda r: r[0])
    return [TraceEntry(i, *r) for i, r in enumerate(rows)]


def prompt_tokens(entry: TraceEntry, vocab_size: int, seed: int) -> List[int]:
    """Deterministic prompt for a trace entry (reference serving.py:157-170):
    uniform tokens, or a short seeded template repeated ("repetitive")."""
    rng = np.random.default_rng([seed, entry.request_id, 0x51])
    if entry.corpus == "random":
        return [int(x) for x in rng.integers(0, vocab_size, size=entry.prompt_len)]
    ell = int(rng.integers(4, 13))
    tpl = [int(x) for x in rng.integers(0, vocab_size, size=ell)]
    return (tpl * (-(-entry.prompt_len // ell)))[:entry.prompt_len]


@dataclass(frozen=True)
class CostModel:
    """Deterministic pass-time model (reference serving.py:226-244): the
    logical clock of a replay.  Defaults are the reference's."""

    device_flops_per_s: float = 1.0e10
    link_bytes_per_s: float = 1.0e9
    collective_latency_s: float = 5.0e-5

    def validate(self) -> "CostModel":
        if min(self.device_flops_per_s, self.link_bytes_per_s, self.collective_latency_s) <= 0:
            raise ContractViolation("cost model parameters must be positive")
        return self

    def step_time_s(self, record) -> float:
        compute = record.flops_max_device / self.device_flops_per_s
        comm = sum(e.bytes / self.link_bytes_per_s + self.collective_latency_s for e in record.comm)
        return compute + comm


@dataclass
class RequestMetrics:
    request_id: int
    arrival_ms: float
    ttft_ms: float
    tpot_ms: float
    e2e_ms: float
    tokens_in: int
    tokens_out: int


@dataclass
class PassLog:
    step_id: int
    wall_ms: float
    mode: str
    batch_kind: str
    batch_tokens: int
    n_requests: int
    pass_ms: float
    flops: int = 0          # record.flops_total (reference StepLogEntry.flops)
    comm_bytes: float = 0.0  # record.comm_bytes (reference StepLogEntry.bytes)


@dataclass
class ServingResult:
    metrics: List[RequestMetrics]
    passes: List[PassLog]
    rejected: List[dict]
    outputs: Dict[int, List[int]]


@dataclass
class _Live:
    entry: TraceEntry
    prompt: List[int]
    seq: object = None
    tokens: List[int] = field(default_factory=list)
    first_ms: float = 0.0
    last_ms: float = 0.0


def run_serving(engine: Engine, trace: Sequence[TraceEntry], seed: int = 0,
                time_scale: float = 1.0, max_prefill_tokens: Optional[int] = None,
                cost_model: Optional[CostModel] = None) -> ServingResult:
    """Serve a trace to completion on the wall clock, or on the logical clock
    of ``cost_model`` (reference run_serving_loop semantics, serving.py:311-517).

    ``time_scale`` stretches (>1) or compresses (<1) the trace's arrival times;
    ``max_prefill_tokens`` optionally caps the tokens of one prefill pass
    (the reference prefills every queued prompt at once, the default here).
    """
    cfg = engine.config
    arrivals: List[_Live] = []
    rejected: List[dict] = []
    for e in sorted(trace, key=lambda x: (x.arrival_ms, x.request_id)):
        need = e.prompt_len + e.output_len - 1
        if need > cfg.max_seq:
            rejected.append({"request_id": e.request_id, "arrival_ms": e.arrival_ms,
                             "error": f"needs {need} cache slots, max_seq is {cfg.max_seq}"})
            continue
        arrivals.append(_Live(e, prompt_tokens(e, cfg.vocab_size, seed)))
    queued: List[_Live] = []
    decoding: List[_Live] = []
    metrics: List[RequestMetrics] = []
    passes: List[PassLog] = []
    outputs: Dict[int, List[int]] = {}
    t0 = time.perf_counter()
    if cost_model is not None:
        cost_model.validate()
    sim = [0.0]  # logical clock (ms), used when cost_model is set
    nxt = 0
    pool_blocks = engine.pool.alloc.num_blocks
    bsz = engine.pool.block_size
    committed = 0  # blocks promised to admitted, unfinished requests

    def _blocks(r: _Live) -> int:
        return -(-(len(r.prompt) + r.entry.output_len - 1) // bsz)

    def now_ms() -> float:
        if cost_model is not None:
            return sim[0]
        return (time.perf_counter() - t0) * 1e3

    def done(r: _Live) -> None:
        nonlocal committed
        n = len(r.tokens)
        metrics.append(RequestMetrics(r.entry.request_id, r.entry.arrival_ms * time_scale,
                                      r.first_ms - r.entry.arrival_ms * time_scale,
                                      (r.last_ms - r.first_ms) / (n - 1) if n > 1 else 0.0,
                                      r.last_ms - r.entry.arrival_ms * time_scale,
                                      len(r.prompt), n))
        outputs[r.entry.request_id] = list(r.tokens)
        engine.release(r.seq)
        committed -= _blocks(r)

    while True:
        t = now_ms()
        while nxt < len(arrivals) and arrivals[nxt].entry.arrival_ms * time_scale <= t:
            r = arrivals[nxt]
            r.seq = engine.new_sequence(r.entry.request_id,
                                        capacity=len(r.prompt) + r.entry.output_len - 1)
            queued.append(r)
            nxt += 1
        if not queued and not decoding:
            if nxt >= len(arrivals):
                break
            wait = arrivals[nxt].entry.arrival_ms * time_scale - now_ms()
            if cost_model is not None:
                sim[0] = max(sim[0], arrivals[nxt].entry.arrival_ms * time_scale)
            elif wait > 0:
                time.sleep(wait / 1e3)
            continue
        take = []
        if queued:
            # admission: a request enters only if the paged pool can hold its whole
            # life (prompt + outputs) next to every live request's; prompts that do
            # not fit wait for finished requests to release their blocks
            budget = max_prefill_tokens
            while queued and (budget is None or not take or len(queued[0].prompt) <= budget):
                need = _blocks(queued[0])
                if committed + need > pool_blocks:
                    break
                r = queued.pop(0)
                committed += need
                take.append(r)
                if budget is not None:
                    budget -= len(r.prompt)
            if not take and not decoding:
                raise CacheOverflow(f"request {queued[0].entry.request_id} needs "
                                    f"{_blocks(queued[0])} KV blocks, the pool has {pool_blocks}")
        if take:
            batch = Batch(BatchKind.PREFILL, [BatchItem(r.seq, list(r.prompt)) for r in take])
            kind = "prefill"
        else:
            take = list(decoding)
            batch = Batch(BatchKind.DECODE, [BatchItem(r.seq, [r.tokens[-1]]) for r in take])
            kind = "decode"
        mode = choose_mode(engine.policy, batch)
        t_pass = now_ms()
        logits, rec = engine.step(batch, mode=mode)
        ids = greedy_tokens(logits)  # one argmax kernel + one D2H: the pass is complete
        if cost_model is not None:
            sim[0] += cost_model.step_time_s(rec) * 1000.0
        t_end = now_ms()
        for r, tok in zip(take, ids):
            r.tokens.append(tok)
            if kind == "prefill":
                r.first_ms = t_end
            r.last_ms = t_end
        still = []
        for r in take:
            if len(r.tokens) >= r.entry.output_len:
                done(r)
            elif kind == "prefill":
                decoding.append(r)
            else:
                still.append(r)
        if kind == "decode":
            decoding = still
        passes.append(PassLog(rec.step_id, t_end, rec.mode.value, kind, rec.new_tokens,
                              rec.n_requests, t_end - t_pass, rec.flops_total, rec.comm_bytes))
    metrics.sort(key=lambda m: m.request_id)
    return ServingResult(metrics, passes, rejected, outputs)


def nearest_rank(values: Sequence[float], q: float) -> float:
    """Nearest-rank percentile (numpy method="higher"), as the reference uses."""
    return float(np.percentile(np.asarray(values, dtype=np.float64), q, method="higher"))


def summarize(res: ServingResult) -> dict:
    kinds = [p.mode for p in res.passes]
    shifts = sum(1 for a, b in zip(kinds, kinds[1:]) if a != b)
    ms = res.metrics
    if not ms:
        return {"empty": True, "requests": 0, "rejected": len(res.rejected),
                "mode_shift_count": shifts, "combined_throughput_tokens_per_s": 0.0}
    span = max(m.arrival_ms + m.e2e_ms for m in ms) - min(m.arrival_ms for m in ms)
    tok = sum(m.tokens_in + m.tokens_out for m in ms)
    return {
        "empty": False, "requests": len(ms), "rejected": len(res.rejected),
        "median_ttft_ms": nearest_rank([m.ttft_ms for m in ms], 50),
        "p99_ttft_ms": nearest_rank([m.ttft_ms for m in ms], 99),
        "median_tpot_ms": nearest_rank([m.tpot_ms for m in ms], 50),
        "p99_tpot_ms": nearest_rank([m.tpot_ms for m in ms], 99),
        "combined_throughput_tokens_per_s": tok / (span / 1e3) if span > 0 else 0.0,
        "mode_shift_count": shifts, "makespan_ms": span,
        "tokens_in_total": sum(m.tokens_in for m in ms),
        "tokens_out_total": sum(m.tokens_out for m in ms),
        "passes": len(res.passes),
        "sp_passes": sum(1 for p in res.passes if p.mode == "sp"),
        "tp_passes": sum(1 for p in res.passes if p.mode == "tp"),
    }


def write_metrics_csv(path: str, metrics: Sequence[RequestMetrics]) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("request_id,arrival_ms,ttft_ms,tpot_ms,e2e_ms,tokens_in,tokens_out\n")
        for m in metrics:
            fh.write(f"{m.request_id},{m.arrival_ms:.3f},{m.ttft_ms:.6f},{m.tpot_ms:.6f},"
                     f"{m.e2e_ms:.6f},{m.tokens_in},{m.tokens_out}\n")


def write_pass_log(path: str, passes: Sequence[PassLog]) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        for p in passes:
            fh.write(json.dumps(p.__dict__, sort_keys=True) + "\n")
