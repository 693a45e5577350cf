"""Live pin of the oracle against the REAL reference (shiftsim) — build container only.

Skipped where /root/reference is absent (the GPU box).  Mirrors the
reference's acceptance criterion 1 (tests/test_acceptance.py:73-108): TP/SP
engine outputs at P in {2, 4, 8} over several prompts, plus greedy decode;
here the oracle must be BIT-identical to shiftsim, not merely close.
"""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
if not os.path.isdir(REF):
    pytest.skip("reference not mounted", allow_module_level=True)
sys.path.insert(0, REF)

shiftsim = pytest.importorskip("shiftsim")
from shiftsim.fabric import DeviceGroup  # noqa: E402
from shiftsim.model import ModelConfig, init_weights  # noqa: E402
from shiftsim.parallel_engine import Batch, BatchItem, BatchKind, Engine, ParallelMode, ShiftPolicy  # noqa: E402

import oracle  # noqa: E402
from oracle.model import compat_config, init_weights_compat  # noqa: E402


@pytest.fixture(scope="module")
def weights():
    return init_weights(ModelConfig(), seed=0), init_weights_compat(compat_config(), seed=0)


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("mode", ["tp", "sp"])
def test_engine_bitexact_vs_shiftsim(weights, p, mode):
    rw, ow = weights
    for i in range(4):
        rng = np.random.default_rng([41, i])
        prompt = [int(x) for x in rng.integers(0, 256, size=int(rng.integers(4, 65)))]
        reng = Engine(rw, DeviceGroup(p), ShiftPolicy.fixed_tp())
        oeng = oracle.OracleEngine(ow, p)
        rs = reng.new_sequence(0, capacity=len(prompt) + 3)
        os_ = oeng.new_sequence(0, capacity=len(prompt) + 3)
        rl, rrec = reng.step(Batch(BatchKind.PREFILL, [BatchItem(rs, prompt)]),
                             mode=ParallelMode(mode), span_logits=True)
        ol, orec = oeng.step([(os_, prompt)], mode=mode, span_logits=True)
        assert rl[0].tobytes() == ol[0].tobytes()
        assert tuple(rrec.flops_per_device) == orec["flops_per_device"]
        assert [(e.kind, e.bytes) for e in rrec.comm] == list(orec["comm"])
        tok = int(np.argmax(rl[0][-1]))
        for _ in range(3):
            rl, _ = reng.step(Batch(BatchKind.DECODE, [BatchItem(rs, [tok])]), mode=ParallelMode(mode))
            ol, _ = oeng.step([(os_, [tok])], prefill=False, mode=mode)
            assert rl[0].tobytes() == ol[0].tobytes()
            tok = int(np.argmax(rl[0]))
