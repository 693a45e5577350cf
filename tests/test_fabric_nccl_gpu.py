"""NcclGroup.all_gather_rows on device tensors (the SP logits gather,
fabric.py:173-191): even shards are gathered in place,
uneven ones padded to a common block and compacted by ONE row-gather kernel
(no torch.cat).  NCCL needs one GPU per rank, so the collective is simulated
in-process; the engine paths are covered by the multi-process tests."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("counts", [[3, 3, 3, 3], [2, 1, 0, 2], [0, 4, 1, 1]])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_nccl_all_gather_rows_compaction(counts, dtype):
    """NcclGroup.all_gather_rows on device tensors (the SP logits gather,
    fabric.py:173-191): even shards gathered in place, uneven ones padded and
    compacted by one row-gather kernel.  The collective is simulated in-process
    (each 'rank' is driven with the blocks the others would contribute)."""
    from paper_2507_11830_b200.fabric import _Ledger, NcclGroup
    p, width = len(counts), 24
    blocks = [torch.randn(max(c, 1) + r % 2, width, device="cuda").to(dtype) for r, c in enumerate(counts)]
    mx = max(counts)
    want = torch.cat([blocks[r][:counts[r]] for r in range(p)], 0)

    class FakeDist:
        def __init__(self, me):
            self.me = me

        def all_gather_into_tensor(self, out, inp):
            for r in range(p):
                src = inp if r == self.me else blocks[r]
                if src.shape[0] < mx:  # the other ranks' padded contributions
                    pad = torch.zeros((mx, width), dtype=dtype, device="cuda")
                    pad[:src.shape[0]] = src
                    src = pad
                out[r * mx:(r + 1) * mx].copy_(src[:mx])

    for me in range(p):
        g = NcclGroup.__new__(NcclGroup)
        _Ledger.__init__(g, p)
        g.rank, g.local_ranks, g.device = me, [me], torch.device("cuda")
        g._dist, g._stage, g._compact_idx = FakeDist(me), False, {}
        got = g.all_gather_rows({me: blocks[me]}, counts)
        assert torch.equal(got, want)
