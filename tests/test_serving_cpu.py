"""Serving driver host logic (CPU): traces, prompt materialisation, summaries."""

import os
import sys

import numpy as np
import pytest

from paper_2507_11830_b200.errors import ContractViolation
from paper_2507_11830_b200.serving import (PassLog, RequestMetrics, ServingResult, TraceEntry,
                                           bursty_trace, nearest_rank, prompt_tokens, read_trace,
                                           summarize, write_trace)


def test_bursty_trace_is_deterministic_and_two_phase():
    a = bursty_trace([(4000, 1.5), (2000, 25.0)], 2048, 256, seed=11)
    b = bursty_trace([(4000, 1.5), (2000, 25.0)], 2048, 256, seed=11)
    assert a == b and len(a) > 20
    low = [e for e in a if e.arrival_ms < 4000]
    high = [e for e in a if e.arrival_ms >= 4000]
    assert len(high) > 3 * len(low)
    assert all(e.prompt_len == 2048 and e.output_len == 256 for e in a)
    assert [e.arrival_ms for e in a] == sorted(e.arrival_ms for e in a)


def test_trace_round_trip_and_validation(tmp_path):
    tr = bursty_trace([(1000, 20.0)], 100, 8, seed=3)
    p = tmp_path / "t.jsonl"
    write_trace(str(p), tr)
    assert read_trace(str(p)) == tr
    bad = tmp_path / "bad.jsonl"
    bad.write_text('{"arrival_ms": 1, "prompt_len": 0, "output_len": 3}\n')
    with pytest.raises(ContractViolation):
        read_trace(str(bad))
    bad.write_text('{"arrival_ms": 1, "prompt_len": 2, "output_len": 3, "x": 1}\n')
    with pytest.raises(ContractViolation):
        read_trace(str(bad))


def test_prompt_materialisation_matches_reference_when_available():
    e = TraceEntry(7, 0, 50, 4, "repetitive")
    toks = prompt_tokens(e, 256, seed=5)
    assert len(toks) == 50 and toks == prompt_tokens(e, 256, seed=5)
    ref = "/root/reference/pkg/src"
    if os.path.isdir(ref):
        sys.path.insert(0, ref)
        from shiftsim.serving import TraceEntry as RT, materialize_prompt
        for corpus in ("random", "repetitive"):
            r = RT(7, 0, 50, 4, corpus)
            assert materialize_prompt(r, 256, 5) == prompt_tokens(TraceEntry(7, 0, 50, 4, corpus), 256, 5)


def test_summary_nearest_rank_percentiles():
    ms = [RequestMetrics(i, float(i), float(v), 2.0, 100.0, 10, 5)
          for i, v in enumerate([5.0, 1.0, 3.0, 2.0, 4.0])]
    res = ServingResult(ms, [PassLog(0, 0, "sp", "prefill", 50, 5, 1.0),
                             PassLog(1, 0, "tp", "decode", 5, 5, 1.0)], [], {})
    s = summarize(res)
    assert s["median_ttft_ms"] == 3.0 and s["p99_ttft_ms"] == 5.0
    assert s["mode_shift_count"] == 1 and s["requests"] == 5
    assert nearest_rank([1, 2, 3, 4], 50) == 3.0  # "higher" convention
