"""Golden fixture for serving parity: the REAL reference's
``run_serving_loop`` (/root/reference/pkg/src/shiftsim/serving.py:311-517)
replaying its own frozen trace (pkg/traces/reference_burst.jsonl) on its
logical clock.

Run in the build container, where ``/root/reference`` is mounted:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_serving_golden.py

Writes ``tests/golden/serving_golden.json``:

* ``trace``: the 55 trace rows (the GPU box never reads /root/reference);
* ``model``: the compat-mode model (reference family: MHA, GeLU, sinusoidal
  positions, eps 1e-6; head_dim 32 so the B200 attention kernels take it),
  weights ``init_weights(model, seed=0, F64)`` — the oracle's
  ``init_weights_compat`` restates that draw order bit-exactly;
* ``schedules[policy]``: per pass (kind, mode, batch_tokens, n_requests,
  sim_time_ms) under a COMPUTE-ONLY cost model (link bytes and collective
  latency made negligible), for the shift / fixed_tp / fixed_sp policies —
  pass times are then flops_max_device / 1e10, a quantity both engines
  compute identically (flop_count, flops.py:87-200), so the two drivers must
  produce the same schedule;
* ``outputs`` (shift policy) and, per emitted token, the f64 reference's
  top-2 logit margin and max |logit| recomputed with ``forward_reference``
  over prompt + outputs[:i] (model.py:310-354), so a device token that differs
  can be checked against the margin.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from shiftsim.config import RunConfig  # noqa: E402
from shiftsim.model import ModelConfig, forward_reference  # noqa: E402
from shiftsim.serving import (CostModel, materialize_prompt, read_trace,  # noqa: E402
                              run_serving_loop)

OUT = Path(__file__).resolve().parent / "serving_golden.json"
TRACE = "/root/reference/pkg/traces/reference_burst.jsonl"
MODEL = dict(n_layers=4, n_heads=8, head_dim=32, ffn_dim=512, vocab_size=256, max_seq=4096)
COMPUTE_ONLY = CostModel(device_flops_per_s=1.0e10, link_bytes_per_s=1.0e30,
                         collective_latency_s=1.0e-30)


def main() -> None:
    trace = read_trace(TRACE)
    base = RunConfig(model=ModelConfig(**MODEL), world_size=2, seed=0)
    gold = {"source": "shiftsim run_serving_loop (serving.py:311-517) on "
                      "pkg/traces/reference_burst.jsonl",
            "trace": [{"arrival_ms": e.arrival_ms, "prompt_len": e.prompt_len,
                       "output_len": e.output_len, "corpus": e.corpus} for e in trace],
            "model": MODEL, "world_size": 2, "seed": 0,
            "cost_model": {"device_flops_per_s": COMPUTE_ONLY.device_flops_per_s,
                           "link_bytes_per_s": COMPUTE_ONLY.link_bytes_per_s,
                           "collective_latency_s": COMPUTE_ONLY.collective_latency_s},
            "schedules": {}}
    outputs = None
    for kind in ("shift", "fixed_tp", "fixed_sp"):
        cfg = base.replace(policy_kind=kind)
        eng = cfg.build_engine()
        res = run_serving_loop(eng, trace, cfg.policy(), COMPUTE_ONLY, seed=cfg.seed)
        gold["schedules"][kind] = [
            {"kind": s.batch_kind, "mode": s.mode, "batch_tokens": s.batch_tokens,
             "n_requests": s.n_requests, "sim_time_ms": s.sim_time_ms, "flops": s.flops}
            for s in res.steps]
        if kind == "shift":
            gold["token_threshold"] = cfg.resolved_threshold()
            outputs = res.outputs
            gold["metrics"] = [{"request_id": m.request_id, "ttft_ms": m.ttft_ms,
                                "tpot_ms": m.tpot_ms, "e2e_ms": m.e2e_ms} for m in res.metrics]
            weights = eng.weights
    gold["outputs"] = {str(k): v for k, v in sorted(outputs.items())}
    margins = {}
    for e in trace:
        out = outputs[e.request_id]
        prompt = materialize_prompt(e, MODEL["vocab_size"], 0)
        logits, _ = forward_reference(weights, prompt + out[:-1])
        rows = logits[len(prompt) - 1:]
        assert [int(np.argmax(r)) for r in rows] == out, e.request_id
        srt = np.sort(rows, axis=1)
        margins[str(e.request_id)] = {"margin": [float(x) for x in srt[:, -1] - srt[:, -2]],
                                      "absmax": [float(x) for x in np.abs(rows).max(axis=1)]}
    gold["margins"] = margins
    OUT.write_text(json.dumps(gold, sort_keys=True) + "\n")
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
