"""Suffix drafting and greedy acceptance against golden
vectors produced by the real reference (tests/golden/make_spec_golden.py)."""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2507_11830_b200.errors import ConfigError, ContractViolation
from paper_2507_11830_b200.spec_decode import (DraftResult, SpeculationConfig, SuffixIndex,
                                               accept_greedy, propose)

GOLD = json.loads((Path(__file__).parent / "golden" / "spec_golden.json").read_text())


def test_propose_matches_reference_golden():
    for i, c in enumerate(GOLD["propose"]):
        idx = SuffixIndex(c["history"], c["min_match"], c["max_spec"], c["window"])
        d = propose(idx, limit=c["limit"])
        assert (list(d.tokens), d.match_len) == (c["tokens"], c["match_len"]), i


def test_accept_matches_reference_golden():
    for i, c in enumerate(GOLD["greedy_accept"]):
        rows = np.asarray(c["rows"])
        targets = [int(np.argmax(r)) for r in rows]  # lowest index on ties, as greedy_token
        assert accept_greedy(c["draft"], targets) == c["emitted"], i


def test_contract_errors():
    with pytest.raises(ContractViolation):
        propose(SuffixIndex())
    with pytest.raises(ContractViolation):
        SuffixIndex(min_match=0)
    with pytest.raises(ContractViolation):
        DraftResult((1, 2), 0)
    with pytest.raises(ConfigError):
        SpeculationConfig(max_spec=0).validate()
    assert propose(SuffixIndex([1, 2, 1, 2]), limit=0) == DraftResult((), 0)
    # equal-length matches: the most recent occurrence wins (its continuation
    # runs into the matched suffix itself)
    assert propose(SuffixIndex([7, 8, 7, 8, 7, 8], max_spec=5)) == DraftResult((7, 8), 2)
