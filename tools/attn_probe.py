"""One 8K causal paged prefill attention call (8B geometry: 32 q / 8 kv heads,
d=128) — for instrumented builds and ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11830_b200 import ops  # noqa: E402

T, d, hq, hk, bs = 8192, 128, 32, 8, 64
nblk = T // bs
kpool = torch.randn(nblk, hk, bs, d, device="cuda").to(torch.bfloat16)
vpool = torch.randn_like(kpool)
q = torch.randn(T, hq * d, device="cuda").to(torch.bfloat16)
bt = torch.arange(nblk, dtype=torch.int32, device="cuda").view(1, -1)
cu = torch.tensor([0, T], dtype=torch.int32, device="cuda")
first = torch.zeros(1, dtype=torch.int32, device="cuda")
kvl = torch.tensor([T], dtype=torch.int32, device="cuda")
tt = ops.attn_tile_tokens(hq, hk, d, bs)
wl = sorted([(0, t0) for t0 in range(0, T, tt)], key=lambda w: -w[1])
work = torch.tensor(wl, dtype=torch.int32, device="cuda").view(-1)
o = torch.empty_like(q)
ops.attention(q, kpool, vpool, bt, cu, first, kvl, o, n_items=1, work=work, n_work=len(wl),
              max_q_len=T, max_kv_len=T, q_heads=hq, kv_heads=hk, head_dim=d, block_size=bs,
              ws=None)
torch.cuda.synchronize()
