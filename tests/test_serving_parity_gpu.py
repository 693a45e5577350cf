"""Serving parity (VERDICT r1 "Next" #10).

The B200 serving driver replays the reference's own frozen trace
(pkg/traces/reference_burst.jsonl, 55 requests, low phase then burst) on the
reference's LOGICAL clock and is compared with ``run_serving_loop``
(/root/reference/pkg/src/shiftsim/serving.py:311-517) as the real reference
ran it (tests/golden/make_serving_golden.py -> serving_golden.json):

1. Schedule: under a compute-only cost model (pass time = flops_max_device /
   1e10, a quantity both engines compute identically) the pass sequence —
   kind, mode, batch tokens, requests, simulated time, FLOPs — is identical for
   the shift, fixed-TP and fixed-SP policies, and so are every request's TTFT /
   TPOT / e2e.
2. Tokens: the device's greedy tokens equal the f64 reference's; where a
   request's tokens first differ, the reference's own top-2 margin there is
   within the bf16 tolerance band (2 x 2e-2 x max|logit|) — a legitimate
   near-tie, not an error.
3. Criterion 6 (tests/test_acceptance.py:290-329), the shift-vs-fixed
   directional check, on the device engine's own step records under the
   reference's DEFAULT cost model: burst-phase median TTFT of shift <= fixed
   TP; low-phase median TPOT of shift <= 1.05 x fixed TP; combined throughput
   of shift >= 0.9 x the best fixed policy.
"""

import json
import os

import numpy as np
import pytest
import torch

from oracle.model import compat_config, init_weights_compat

from helpers import device_weights

pytestmark = pytest.mark.gpu

from paper_2507_11830_b200 import Engine, LoopbackGroup, ShiftPolicy  # noqa: E402
from paper_2507_11830_b200.serving import (CostModel, TraceEntry, nearest_rank,  # noqa: E402
                                           run_serving, summarize)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "serving_golden.json")
TOL = 2e-2


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def gold():
    with open(GOLD) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def weights(gold):
    m = gold["model"]
    ow = init_weights_compat(compat_config(**m), seed=gold["seed"])
    return device_weights(ow, gold["world_size"])


def _trace(gold):
    return [TraceEntry(i, r["arrival_ms"], r["prompt_len"], r["output_len"], r["corpus"])
            for i, r in enumerate(gold["trace"])]


def _policy(kind, tau):
    return {"shift": ShiftPolicy(token_threshold=tau), "fixed_tp": ShiftPolicy.fixed_tp(),
            "fixed_sp": ShiftPolicy.fixed_sp()}[kind]


def _run(gold, weights, kind, cost):
    p = gold["world_size"]
    eng = Engine(weights, LoopbackGroup(p), _policy(kind, gold["token_threshold"]),
                 num_blocks=512, block_size=64)
    return run_serving(eng, _trace(gold), seed=gold["seed"], cost_model=cost)


def _compute_only(gold):
    c = gold["cost_model"]
    return CostModel(c["device_flops_per_s"], c["link_bytes_per_s"], c["collective_latency_s"])


@pytest.mark.parametrize("kind", ["shift", "fixed_tp", "fixed_sp"])
def test_schedule_matches_reference_serving_loop(gold, weights, kind):
    res = _run(gold, weights, kind, _compute_only(gold))
    want = gold["schedules"][kind]
    got = [{"kind": p.batch_kind, "mode": p.mode, "batch_tokens": p.batch_tokens,
            "n_requests": p.n_requests, "flops": p.flops} for p in res.passes]
    assert got == [{k: w[k] for k in ("kind", "mode", "batch_tokens", "n_requests", "flops")}
                   for w in want]
    np.testing.assert_allclose([p.wall_ms for p in res.passes],
                               [w["sim_time_ms"] for w in want], rtol=1e-12)
    assert not res.rejected
    if kind == "shift":
        for m, w in zip(res.metrics, gold["metrics"]):
            assert m.request_id == w["request_id"]
            np.testing.assert_allclose([m.ttft_ms, m.tpot_ms, m.e2e_ms],
                                       [w["ttft_ms"], w["tpot_ms"], w["e2e_ms"]],
                                       rtol=1e-12, atol=1e-9)


def test_tokens_match_reference_up_to_near_ties(gold, weights):
    res = _run(gold, weights, "shift", _compute_only(gold))
    identical, flips = 0, []
    for rid, want in gold["outputs"].items():
        got = res.outputs[int(rid)]
        assert len(got) == len(want)
        i = next((j for j, (a, b) in enumerate(zip(got, want)) if a != b), None)
        if i is None:
            identical += 1
            continue
        mg = gold["margins"][rid]
        rel = mg["margin"][i] / mg["absmax"][i]
        flips.append((int(rid), i, rel))
        assert rel <= 2 * TOL, f"request {rid} token {i}: reference margin {rel:.3g} > {2 * TOL}"
    print(f"serving tokens: {identical}/{len(gold['outputs'])} requests identical; "
          f"near-tie flips (request, index, margin/max|logit|): {flips}")
    # sanity floor only — the bar is the margin check above (measured: 47/55,
    # every flip at a reference margin of ~0.2% of max|logit|)
    assert identical >= 0.8 * len(gold["outputs"])


def test_criterion6_shift_vs_fixed_on_device_records(gold, weights):
    """Reference acceptance criterion 6 on the B200 engine's own records."""
    res = {k: _run(gold, weights, k, CostModel()) for k in ("shift", "fixed_tp", "fixed_sp")}

    def med(v):
        return nearest_rank(v, 50)
    burst_ttft = {k: med([m.ttft_ms for m in r.metrics if m.arrival_ms >= 4000])
                  for k, r in res.items()}
    low_tpot = {k: med([m.tpot_ms for m in r.metrics if m.arrival_ms < 4000])
                for k, r in res.items()}
    thr = {k: summarize(r)["combined_throughput_tokens_per_s"] for k, r in res.items()}
    print("criterion 6 (device records):", burst_ttft, low_tpot, thr)
    assert burst_ttft["shift"] <= burst_ttft["fixed_tp"]
    assert low_tpot["shift"] <= 1.05 * low_tpot["fixed_tp"]
    assert thr["shift"] >= 0.9 * max(thr["fixed_tp"], thr["fixed_sp"])
    assert summarize(res["shift"])["mode_shift_count"] >= 2
