"""Prefill attention at the per-GPU shape of Ulysses SP over N GPUs (8B, 8K
tokens): each rank attends 32/N q heads and 8/N kv heads over all tokens."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11830_b200 import ops  # noqa: E402
from paper_2507_11830_b200.engine import attention_split_plan  # noqa: E402

T, d, bs = 8192, 128, 64
for N in [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]:
    hq, hk = 32 // N, 8 // N
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
    ws = torch.empty(ops.attn_workspace_bytes(1, hq, d, T) // 4 + 1, device="cuda")

    def fn():
        ops.attention(q, kpool, vpool, bt, cu, first, kvl, o, n_items=1, work=work,
                      n_work=len(wl), max_q_len=T, max_kv_len=T, q_heads=hq, kv_heads=hk,
                      head_dim=d, block_size=bs, ws=ws)
    # the engine's split-KV plan (Engine._split_plan) when the tiles do not fill the SMs
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    plan = None
    if os.environ.get("SP_ATTN_SPLIT") != "0":
        wl3 = [(i, t0, t0) for i, t0 in wl]
        plan = attention_split_plan(wl3, [T], [0], tt, hk, sms, 1 << 30)
    if plan is not None:
        work_np, split_np, comb_np, slot = plan
        T32 = lambda a: torch.from_numpy(a).to(device="cuda").view(-1)  # noqa: E731
        w2, sp2, cb2 = T32(work_np), T32(split_np), T32(comb_np)
        ent, comb = work_np, comb_np
        ws = torch.empty(slot * hk * ops.SPLIT_SLOT_BYTES // 4 + 1, device="cuda")

        def fn():
            ops.attention_prefill_split(q, kpool, vpool, bt, cu, first, kvl, o, work=w2, split=sp2,
                                        n_work=len(ent), combine=cb2, n_combine=len(comb),
                                        n_slots=slot, q_heads=hq, kv_heads=hk, head_dim=d,
                                        block_size=bs, ws=ws)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    fl = 4 * d * hq * (T * (T + 1) // 2)
    print(json.dumps({"sp": N, "q_heads": hq, "kv_heads": hk, "ctas": len(wl) * hk, "ms": round(ms, 4),
                      "tflops": round(fl / ms / 1e9, 1), "ms_x_N": round(ms * N, 4)}), flush=True)
