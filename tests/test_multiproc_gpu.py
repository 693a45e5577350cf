"""The N>1 engine path with one process per rank (the torchrun/NCCL layout of
bench.py --gpus N), run as 2 processes sharing the one available B200.

NCCL refuses two ranks on one GPU, so the NcclGroup here runs over gloo and
stages its collectives through host memory; everything else — the SPMD
metadata every rank builds, its own head shard of the paged cache, its own
token shard, the split tables of the SP all-to-alls (uneven and empty
shards), the TP all-reduce and the logits all-gather — is the code path the
8-GPU run takes.  The result must be bit-identical to the in-process
LoopbackGroup(2) engine (for two ranks every collective sum is a single
commutative add, so no reduction-order freedom remains).
"""

import os
import socket

import numpy as np
import pytest
import torch

from helpers import c1_prompts, device_weights

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _schedule():
    """C1 prompts (SP prefill), then decode passes alternating TP / SP, the last
    SP decode with ONE request (token shards [1, 0]: an empty shard)."""
    prompts = c1_prompts()[:3]
    return prompts


def _run(engine_factory):
    from paper_2507_11830_b200 import Batch, BatchItem, BatchKind, ParallelMode
    eng = engine_factory()
    prompts = _schedule()
    seqs = [eng.new_sequence(i, capacity=256) for i in range(len(prompts))]
    out = []
    lg, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, p) for s, p in zip(seqs, prompts)]),
                     mode=ParallelMode.SP)
    out.append(np.stack([x.cpu().numpy() for x in lg]))
    # fixed (teacher-forced) tokens: both runs see identical inputs every pass
    for step, mode in enumerate((ParallelMode.TP, ParallelMode.SP, ParallelMode.TP)):
        toks = [(11 * step + 5 * i + 3) % 256 for i in range(len(seqs))]
        lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [t]) for s, t in zip(seqs, toks)]),
                         mode=mode)
        out.append(np.stack([x.cpu().numpy() for x in lg]))
    lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(seqs[0], [toks[0]])]), mode=ParallelMode.SP)
    out.append(np.stack([x.cpu().numpy() for x in lg]))
    fp = seqs[0].cache.fingerprint()
    return out, [s.cache.write_counter for s in seqs], fp


def _tiny(world):
    from oracle.model import init_weights_llama, llama_tiny_config
    if world == 4:  # P | kv_heads
        return init_weights_llama(llama_tiny_config(max_seq=512, n_kv_heads=4), seed=1)
    if world == 8:
        return init_weights_llama(llama_tiny_config(max_seq=512, n_kv_heads=8), seed=2)
    return init_weights_llama(llama_tiny_config(max_seq=512), seed=0)


def _worker(rank, world, port, q, sp_degree=None):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_11830_b200 import Engine, NcclGroup, ShiftPolicy
        ow = _tiny(world)

        def factory():
            # cuda_graphs off: graph capture cannot contain host-staged collectives
            return Engine(device_weights(ow, world), NcclGroup(), ShiftPolicy.fixed_tp(),
                          cuda_graphs=False, sp_degree=sp_degree)

        out, wc, fp = _run(factory)
        q.put((rank, ([o.tolist() for o in out], wc, repr(fp))))
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,sp_degree,fused", [(2, None, False), (4, 2, False),
                                                   (2, None, True), (4, None, True),
                                                   (8, None, True), (8, 4, True)])
def test_multi_process_engine_matches_loopback(world, sp_degree, fused, monkeypatch):
    """(2, None): pure SP/TP over two processes, bit-identical; (4, 2): the
    SP(2) x TP(2) base config over four processes (TP-group all-reduces on
    sub-groups), bit-identical for the mixed prefill, within bf16 tolerance
    for the TP(4) decodes (four-way sums in gloo's order).  fused: the SP
    all-to-alls and TP all-reduces go over CUDA-IPC-mapped peer buffers
    (GEMM epilogue stores into peers, release/acquire flags, one-shot
    ascending-rank all-reduce in the norm kernel) — concurrently running
    processes, bit-identical to the in-process fused path at any P."""
    monkeypatch.setenv("SP_FUSED_A2A", "1" if fused else "0")
    import torch.multiprocessing as mp
    from paper_2507_11830_b200 import Engine, LoopbackGroup, ShiftPolicy

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, sp_degree))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert not isinstance(res[r], str), f"rank {r} failed: {res[r]}"
        assert procs[r].exitcode == 0

    ow = _tiny(world)
    want, want_wc, want_fp = _run(lambda: Engine(device_weights(ow, world), LoopbackGroup(world),
                                                 ShiftPolicy.fixed_tp(), cuda_graphs=False,
                                                 sp_degree=sp_degree))
    for r in range(world):
        got, wc, fp = res[r]
        assert len(got) == len(want)
        for k, (g, w) in enumerate(zip(got, want)):
            g = np.asarray(g, dtype=np.float32)
            if world == 2 or k == 0 or fused:
                # two-member sums (P = 2, and the TP(2) groups of the mixed
                # prefill) leave no reduction-order freedom: bit-identical
                assert np.array_equal(g, w), (r, k)
            else:  # TP(4) all-reduces: gloo's sum order differs from ascending rank
                assert np.max(np.abs(g - w)) <= 2e-2 * np.max(np.abs(w)), (r, k)
        # every rank tracks the global cache cursors (SPMD)
        assert wc == want_wc
        assert fp == repr(want_fp)


@pytest.mark.parametrize("n", [2, 8])
def test_bench_self_spawns_ranks(n):
    """`python bench.py --gpus N` with WORLD_SIZE unset spawns N ranks
    (torch.distributed.run) and rank 0 prints exactly one JSON line carrying
    the SP/TP prefill and decode matrix and the CPU baseline.  Ranks share the
    one GPU through SP_BENCH_BACKEND=gloo (plumbing check, not a number); N=8
    is the driver's largest scaling point (one kv head per rank at 8B)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["SP_BENCH_BACKEND"] = "gloo"
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", str(n),
                          "--steps", "1", "--warmup", "1", "--seq", "1024", "--layers", "2",
                          "--decode-batch", "4", "--decode-ctx", "256"],
                         env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["value"] > 0
    m = d["matrix"]
    assert set(m["prefill"]) >= {"sp", "tp"}
    for b in ("b1", "b4"):
        assert set(m["decode"][b]) >= {"sp", "tp", "shift"}
        assert m["decode"][b]["tp"]["frac_hbm_roofline"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] > 0
