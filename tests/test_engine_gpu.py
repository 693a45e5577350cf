"""Engine parity on a B200: the CUDA path vs the CPU oracle (and the reference's
own golden vectors), mirroring /root/reference/pkg/tests/test_parallel_engine.py.

Tolerances (written here, per BASELINE north star):
* logits / hidden: max |got - want| / max |want| <= 2e-2 against the fp32
  oracle computed from the same bf16-rounded weights (LOGIT_TOL);
* block tables, slot mappings, write counters, fingerprints, FLOP counts,
  comm-event counts: bit-exact / exact;
* SP at P in {1, 2, 4} and TP vs SP at P = 1: bit-identical on the GPU
  (fixed-tile GEMM, M-invariant attention) — the analogue of the reference's
  SP-is-bit-exact test (test_parallel_engine.py:42-50);
* greedy ids: equal wherever the oracle's top-1/top-2 margin exceeds twice the
  measured logit error (random init leaves many near-ties).

P > 1 runs on one GPU through LoopbackGroup (the reference's own simulated-P
execution model); the NCCL group uses the same engine code path.
"""

import numpy as np
import pytest
import torch

import oracle
from oracle.flops import flop_count as oracle_flops
from oracle.model import compat_config, init_weights_compat, init_weights_llama, llama_tiny_config

from helpers import c1_prompts, device_weights, rel_err, top2_margin

pytestmark = pytest.mark.gpu

LOGIT_TOL = 2e-2

sp = pytest.importorskip("paper_2507_11830_b200")
from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, CacheOverflow, ContractViolation,  # noqa: E402
                                   Engine, LoopbackGroup, ParallelMode, ShiftPolicy, SwiftKvConfig,
                                   choose_mode, flop_count, greedy_tokens)
from paper_2507_11830_b200.flops import PassShape  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def c1():
    cfg = llama_tiny_config(max_seq=512)
    return init_weights_llama(cfg, seed=0)


@pytest.fixture(scope="module")
def c1_kv4():
    cfg = llama_tiny_config(max_seq=512, n_kv_heads=4)
    return init_weights_llama(cfg, seed=1)


def make(ow, p, policy=None, swiftkv=None, **kw):
    return Engine(device_weights(ow, p), LoopbackGroup(p), policy or ShiftPolicy.fixed_tp(),
                  swiftkv=swiftkv, **kw)


def to_np(xs):
    return [x.float().cpu().numpy() for x in xs]


@pytest.mark.parametrize("mode", [ParallelMode.TP, ParallelMode.SP])
def test_c1_prefill_and_decode_match_oracle(c1, mode):
    """BASELINE configs[0]: tiny Llama, 8 requests (792 prompt tokens), P=2."""
    prompts = c1_prompts()
    assert sum(map(len, prompts)) == 792
    eng = make(c1, 2)
    oeng = oracle.OracleEngine(c1, 2)
    seqs = [eng.new_sequence(i, capacity=len(p) + 8) for i, p in enumerate(prompts)]
    oseqs = [oeng.new_sequence(i, capacity=len(p) + 8) for i, p in enumerate(prompts)]
    lg, rec = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, p) for s, p in zip(seqs, prompts)]),
                       mode=mode)
    olg, orec = oeng.step(list(zip(oseqs, prompts)), mode=mode.value)
    got, want = np.stack(to_np(lg)), np.stack(olg)
    err = rel_err(got, want)
    assert err <= LOGIT_TOL, err
    assert rec.flops_per_device == orec["flops_per_device"]
    np.testing.assert_array_equal(eng.last_slots, oeng.last_slots)
    np.testing.assert_array_equal(eng.last_block_table, oeng.last_block_table)
    # teacher-forced decode: feed the oracle's greedy tokens to both sides
    toks = [oracle.greedy_token(r) for r in want]
    checked = 0
    for step in range(6):
        lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [t]) for s, t in zip(seqs, toks)]),
                         mode=mode)
        olg, _ = oeng.step([(s, [t]) for s, t in zip(oseqs, toks)], prefill=False, mode=mode.value)
        got, want = np.stack(to_np(lg)), np.stack(olg)
        e = rel_err(got, want)
        assert e <= LOGIT_TOL, (step, e)
        np.testing.assert_array_equal(eng.last_slots, oeng.last_slots)
        abs_err = np.max(np.abs(got - want))
        gids = greedy_tokens(lg)
        for i in range(len(prompts)):
            if top2_margin(want[i]) > 2 * abs_err:
                assert gids[i] == int(np.argmax(want[i]))
                checked += 1
        toks = [int(np.argmax(r)) for r in want]
    assert checked > 0


def test_sp_bitexact_across_world_sizes(c1_kv4, monkeypatch):
    """SP(P) == SP(1) == TP(1) bit-for-bit on the GPU (reference :33-50 analogue).
    Split-K (the decode-size GEMM regime) is pinned off so every shard size runs
    the same GEMM regime; split-K is checked separately (deterministic, within
    tolerance) in test_kernels_gpu.py."""
    monkeypatch.setenv("SP_GEMM_NO_SPLITK", "1")
    prompts = [c1_prompts()[i] for i in (0, 3, 5)]
    outs = {}
    for p, mode in ((1, ParallelMode.SP), (1, ParallelMode.TP), (2, ParallelMode.SP),
                    (4, ParallelMode.SP)):
        eng = make(c1_kv4, p)
        seqs = [eng.new_sequence(i, capacity=200) for i in range(3)]
        lg, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, q) for s, q in zip(seqs, prompts)]),
                         mode=mode, span_logits=True)
        dec, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [7]) for s in seqs]), mode=mode)
        outs[(p, mode)] = [x.cpu() for x in lg] + [x.cpu() for x in dec]
    ref = outs[(1, ParallelMode.SP)]
    for key, val in outs.items():
        for a, b in zip(val, ref):
            assert torch.equal(a, b), key


@pytest.mark.parametrize("p", [2, 4])
def test_tp_matches_oracle_and_sp(c1_kv4, p):
    prompt = c1_prompts()[1]
    res = {}
    for mode in (ParallelMode.TP, ParallelMode.SP):
        eng = make(c1_kv4, p)
        s = eng.new_sequence(0, capacity=len(prompt))
        lg, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, prompt)]), mode=mode,
                         span_logits=True)
        res[mode] = lg[0].cpu().numpy()
    want, _ = oracle.forward_reference(c1_kv4, prompt)
    for mode, got in res.items():
        assert rel_err(got, want) <= LOGIT_TOL, mode


def test_cache_layout_identical_across_modes(c1):
    """Fingerprint equal and layer-0 K/V bit-identical TP vs SP (:130-144)."""
    prompt = c1_prompts()[2]
    caches = {}
    for mode in (ParallelMode.TP, ParallelMode.SP):
        eng = make(c1, 2)
        s = eng.new_sequence(0, capacity=len(prompt))
        eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, prompt)]), mode=mode)
        caches[mode] = s.cache
    a, b = caches[ParallelMode.TP], caches[ParallelMode.SP]
    assert a.fingerprint() == b.fingerprint()
    for dev in range(2):
        ka, va = a.device_blocks(dev)
        kb, vb = b.device_blocks(dev)
        assert torch.equal(ka[0], kb[0]) and torch.equal(va[0], vb[0])


def test_mode_switch_moves_no_cache_bytes(c1):
    """Alternating TP/SP decode writes exactly the new token's rows (:115-127)."""
    cfg = c1.config
    prompt = c1_prompts()[4]
    eng = make(c1, 2)
    s = eng.new_sequence(0, capacity=len(prompt) + 8)
    lg, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, prompt)]), mode=ParallelMode.TP)
    per_token = 2 * cfg.n_layers * cfg.kv_heads * cfg.head_dim * 2  # K,V bf16, all devices
    tok = greedy_tokens(lg)[0]
    for mode in (ParallelMode.SP, ParallelMode.TP, ParallelMode.SP, ParallelMode.TP):
        before = s.cache.write_counter
        lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [tok])]), mode=mode)
        assert s.cache.write_counter - before == per_token
        tok = greedy_tokens(lg)[0]


def test_forced_mode_alternation_matches_fixed_tp(c1):
    """Forced TP/SP schedule decodes like fixed TP where the margin allows (:95-112)."""
    prompt = c1_prompts()[0]

    def run(modes):
        eng = make(c1, 2)
        s = eng.new_sequence(0, capacity=len(prompt) + 12)
        lg, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, prompt)]), mode=ParallelMode.TP)
        out = [lg[0].cpu().numpy()]
        toks = [int(np.argmax(out[-1]))]
        for i in range(10):
            lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [toks[-1]])]), mode=modes(i))
            out.append(lg[0].cpu().numpy())
            toks.append(int(np.argmax(out[-1])))
        return toks, out

    fixed, fl = run(lambda i: ParallelMode.TP)
    mixed, ml = run(lambda i: (ParallelMode.TP, ParallelMode.SP)[i % 2])
    for a, b, la in zip(fixed, mixed, fl):
        if a != b:
            assert top2_margin(la) < 1e-1 * np.max(np.abs(la))
            break  # histories diverge after a near-tie flip
        assert a == b


def test_multi_item_sp_prefill_and_uneven_shards(c1):
    """Multi-item SP (:79-92) with P not dividing M and an empty shard (M=1, P=2)."""
    prompts = [c1_prompts()[i][:n] for i, n in ((0, 5), (1, 9), (2, 13))]
    eng = make(c1, 2)
    items = [BatchItem(eng.new_sequence(i, capacity=len(p) + 2), p) for i, p in enumerate(prompts)]
    lg, _ = eng.step(Batch(BatchKind.PREFILL, items), mode=ParallelMode.SP, span_logits=True)
    for p, got in zip(prompts, lg):
        want, _ = oracle.forward_reference(c1, p)
        assert rel_err(got.cpu().numpy(), want) <= LOGIT_TOL
    # single-token SP decode at P=2 leaves rank 1 with an empty shard
    lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(items[0].seq, [3])]), mode=ParallelMode.SP)
    want, _ = oracle.forward_reference(c1, prompts[0] + [3])
    assert rel_err(lg[0].cpu().numpy(), want[-1]) <= LOGIT_TOL


def test_flops_and_comm_counts(c1):
    cfg = c1.config
    ell = cfg.n_layers
    for mode in (ParallelMode.TP, ParallelMode.SP):
        eng = make(c1, 2)
        items = [BatchItem(eng.new_sequence(i, capacity=20), p)
                 for i, p in enumerate([c1_prompts()[0][:9], c1_prompts()[1][:5]])]
        batch = Batch(BatchKind.PREFILL, items)
        shape = eng.pass_shape(batch)
        _, rec = eng.step(batch, mode=mode)
        assert rec.flops_per_device == flop_count(shape, mode, eng.config, 2)
        assert rec.flops_per_device == oracle_flops((9, 5), (0, 0), mode.value, cfg, 2)
        # TP: 2 all-reduces/layer + logits gather (embedding uses the replica);
        # SP: one fused q|k|v all-to-all + one back all-to-all per layer + gather
        assert len(rec.comm) == 2 * ell + 1
        kinds = {e.kind for e in rec.comm}
        assert kinds == ({"all_reduce", "all_gather"} if mode is ParallelMode.TP
                         else {"all_to_all", "all_gather"})


def test_sp_comm_bytes_follow_gqa_formula(c1):
    """check_comm_ratio (verify_checks.py:177-194) with GQA:
    per device and pass, TP moves 2L f32 all-reduces of [M, h] (ring bytes
    2(P-1)/P each; no embedding all-reduce), SP moves L fused q|k|v
    all-to-alls + L back all-to-alls of bf16 rows ((P-1)/P of what a rank
    sends), so P·SP/TP = L(2H+2Hkv)d·2 / (2L·2h·4) — exact, from the ledger."""
    cfg = c1.config
    L, h, H, Hkv, d, P = cfg.n_layers, cfg.hidden, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, 2
    M = 64
    prompt = (c1_prompts()[0] * 2)[:M]
    by = {}
    for mode in (ParallelMode.TP, ParallelMode.SP):
        eng = make(c1, P)
        s = eng.new_sequence(0, capacity=M)
        eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, prompt)]), mode=mode)
        by[mode] = [eng.group.ledger()[dev] for dev in range(P)]
    frac = (P - 1) / P
    for dev in range(P):
        tp, sp = by[ParallelMode.TP][dev], by[ParallelMode.SP][dev]
        assert tp["all_reduce"] == 2 * L * 2 * frac * M * h * 4
        m_r = M // P
        fwd = frac * m_r * (H + 2 * Hkv) * d * 2   # my tokens' q|k|v, every head block
        back = frac * M * (H // P) * d * 2         # my head block, every token
        assert sp["all_to_all"] == L * (fwd + back)
        ratio = P * sp["all_to_all"] / tp["all_reduce"]
        assert abs(ratio - L * (2 * H + 2 * Hkv) * d * 2 / (2 * L * 2 * h * 4)) < 1e-12
        assert "all_to_all" not in tp and "all_reduce" not in sp


def test_policy_threshold_and_mode_log(c1):
    eng = make(c1, 2, policy=ShiftPolicy(token_threshold=6))
    s = eng.new_sequence(0, capacity=20)
    eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, c1_prompts()[0][:10])]))
    eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [5])]))
    assert eng.mode_log == [ParallelMode.SP, ParallelMode.TP]
    assert [r.step_id for r in eng.step_records] == [0, 1]


def test_capacity_precheck_and_token_range(c1):
    eng = make(c1, 2)
    s = eng.new_sequence(0, capacity=4)
    with pytest.raises(CacheOverflow):
        eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, [1, 2, 3, 4, 5])]))
    assert s.cache.token_count == 0 and s.cache.write_counter == 0
    with pytest.raises(ContractViolation):
        eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, [256])]))
    assert s.cache.write_counter == 0


def test_paged_pool_exhaustion_is_cache_overflow(c1):
    eng = make(c1, 2, num_blocks=2, block_size=16)
    a = eng.new_sequence(0, capacity=64)
    with pytest.raises(CacheOverflow):
        eng.step(Batch(BatchKind.PREFILL, [BatchItem(a, list(range(40)))]))
    assert a.cache.write_counter == 0
    eng.step(Batch(BatchKind.PREFILL, [BatchItem(a, list(range(20)))]))
    eng.release(a)
    b = eng.new_sequence(1, capacity=64)
    eng.step(Batch(BatchKind.PREFILL, [BatchItem(b, list(range(30)))]))


def test_span_logits_and_truncate(c1):
    eng = make(c1, 2)
    prompt = c1_prompts()[3][:20]
    s = eng.new_sequence(0, capacity=32)
    eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, prompt)]), mode=ParallelMode.TP)
    out, rec = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [1, 2, 3])], speculative=True),
                        mode=ParallelMode.TP, span_logits=True)
    assert out[0].shape == (3, 256) and rec.new_tokens == 3
    before = s.cache.write_counter
    s.cache.truncate(21)   # keep 1 of the 3 speculated tokens
    assert s.cache.write_counter == before and s.cache.token_count == 21
    lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [9])]), mode=ParallelMode.SP)
    want, _ = oracle.forward_reference(c1, prompt + [1, 9])
    assert rel_err(lg[0].cpu().numpy(), want[-1]) <= LOGIT_TOL


@pytest.mark.parametrize("mode", [ParallelMode.TP, ParallelMode.SP])
def test_swiftkv_matches_oracle(c1, mode):
    prompts = [c1_prompts()[i][:n] for i, n in ((0, 33), (1, 20), (2, 41))]
    eng = make(c1, 2, swiftkv=SwiftKvConfig(enabled=True, cut_layer=2))
    oeng = oracle.OracleEngine(c1, 2, swiftkv_cut=2)
    seqs = [eng.new_sequence(i, capacity=64) for i in range(3)]
    oseqs = [oeng.new_sequence(i, capacity=64) for i in range(3)]
    lg, rec = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, p) for s, p in zip(seqs, prompts)]),
                       mode=mode)
    olg, orec = oeng.step(list(zip(oseqs, prompts)), mode=mode.value)
    assert rel_err(np.stack(to_np(lg)), np.stack(olg)) <= LOGIT_TOL
    assert rec.flops_per_device == orec["flops_per_device"]
    toks = [int(np.argmax(r)) for r in olg]
    lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [t]) for s, t in zip(seqs, toks)]),
                     mode=mode)
    olg, _ = oeng.step([(s, [t]) for s, t in zip(oseqs, toks)], prefill=False, mode=mode.value)
    assert rel_err(np.stack(to_np(lg)), np.stack(olg)) <= LOGIT_TOL


@pytest.mark.parametrize("mode", [ParallelMode.TP, ParallelMode.SP])
def test_swiftkv_band_and_cache_invariance(c1, mode):
    """check_swiftkv_band (verify_checks.py:197-228): the metered FLOPs equal
    the analytic count, the SwiftKV/standard ratio of a long prefill lies in
    [0.50, 0.62] (cut = L/2), and the cache it leaves (fingerprint, bytes
    written, every layer's K/V present) is the standard one."""
    prompt = (c1_prompts()[0] * 4)[:300]
    res = {}
    for label, skv in (("std", None), ("skv", SwiftKvConfig(enabled=True, cut_layer=2))):
        eng = make(c1, 2, swiftkv=skv)
        s = eng.new_sequence(0, capacity=320)
        batch = Batch(BatchKind.PREFILL, [BatchItem(s, prompt)])
        shape = eng.pass_shape(batch)  # before the step commits the tokens
        _, rec = eng.step(batch, mode=mode)
        cut = None if skv is None else 2
        assert rec.flops_per_device == flop_count(shape, mode, eng.config, 2, swiftkv_cut=cut)
        res[label] = (sum(rec.flops_per_device), s.cache.fingerprint(), s.cache.write_counter)
    ratio = res["skv"][0] / res["std"][0]
    assert 0.50 <= ratio <= 0.62, ratio
    assert res["skv"][1] == res["std"][1] and res["skv"][2] == res["std"][2]


def test_compat_mode_against_reference_golden(golden):
    """The reference's own model family on the GPU vs shiftsim's recorded
    outputs (C1 stand-in: MHA/sinusoidal/GeLU, f32, P=2) — within bf16 tolerance."""
    arrs, meta = golden
    cfg = compat_config(n_layers=4, n_heads=8, head_dim=32, ffn_dim=1024, vocab_size=256,
                        max_seq=512)
    ow = init_weights_compat(cfg, seed=0, dtype=np.float32)
    prompts = c1_prompts()
    for mode in (ParallelMode.SP, ParallelMode.TP):
        eng = make(ow, 2)
        seqs = [eng.new_sequence(i, capacity=len(p) + 4) for i, p in enumerate(prompts)]
        lg, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, p) for s, p in zip(seqs, prompts)]),
                         mode=mode)
        err = rel_err(np.stack(to_np(lg)), arrs[f"c1_{mode.value}2_prefill_logits"])
        assert err <= LOGIT_TOL, (mode, err)


@pytest.fixture(scope="module")
def d128():
    """head_dim 128 (8B-style heads): exercises the tcgen05/TMEM prefill attention."""
    cfg = llama_tiny_config(n_layers=2, n_heads=8, n_kv_heads=2, head_dim=128, ffn_dim=1024,
                            vocab_size=512, max_seq=1024)
    return init_weights_llama(cfg, seed=2)


@pytest.mark.parametrize("mode", [ParallelMode.TP, ParallelMode.SP])
def test_fused_qkv_rope_prefill_bitexact(d128, mode, monkeypatch):
    """Prefill passes (M > 256) run the QKV projection with RoPE + KV write in
    the GEMM epilogue; logits and the cache equal the unfused path bit for bit."""
    prompts = [(c1_prompts()[i] * 3)[:n] for i, n in ((0, 200), (1, 150))]
    res = {}
    for fused in ("1", "0"):
        monkeypatch.setenv("SP_FUSE_ROPE", fused)
        for p in (1, 2):
            eng = make(d128, p)
            seqs = [eng.new_sequence(i, capacity=400) for i in range(2)]
            lg, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, q) for s, q in
                                                       zip(seqs, prompts)]), mode=mode)
            k0 = seqs[0].cache.read_window(0, 1, 0)[0] if p == 1 else None
            res[(fused, p)] = ([x.cpu() for x in lg], k0)
    for p in (1, 2):
        for a, b in zip(res[("1", p)][0], res[("0", p)][0]):
            assert torch.equal(a, b), p
    assert torch.equal(res[("1", 1)][1], res[("0", 1)][1])


@pytest.mark.parametrize("mode", [ParallelMode.TP, ParallelMode.SP])
def test_head_dim_128_tcgen05_attention_matches_oracle(d128, mode):
    rng = np.random.default_rng(5)
    prompts = [[int(t) for t in rng.integers(0, 512, size=n)] for n in (300, 17, 129)]
    eng = make(d128, 2)
    seqs = [eng.new_sequence(i, capacity=400) for i in range(3)]
    lg, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, p) for s, p in zip(seqs, prompts)]),
                     mode=mode, span_logits=True)
    for p, got in zip(prompts, lg):
        want, _ = oracle.forward_reference(d128, p)
        assert rel_err(got.cpu().numpy(), want) <= LOGIT_TOL
    # chunked continuation: a second prefill chunk attends over cached history
    more = [[int(t) for t in rng.integers(0, 512, size=n)] for n in (70, 5, 200)]
    lg, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, p) for s, p in zip(seqs, more)]),
                     mode=mode, span_logits=True)
    for p, q, got in zip(prompts, more, lg):
        want, _ = oracle.forward_reference(d128, p + q)
        assert rel_err(got.cpu().numpy(), want[len(p):]) <= LOGIT_TOL
    # decode steps through the TMA split-KV decode kernel
    hist = [p + q for p, q in zip(prompts, more)]
    for step in range(2):
        toks = [int(x) for x in rng.integers(0, 512, size=3)]
        lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [t]) for s, t in zip(seqs, toks)]),
                         mode=mode)
        for h, t, got in zip(hist, toks, lg):
            h.append(t)
            want, _ = oracle.forward_reference(d128, h)
            assert rel_err(got.cpu().numpy(), want[-1]) <= LOGIT_TOL


@pytest.mark.parametrize("p", [1, 2])
def test_cuda_graph_decode_matches_eager(c1, p):
    """Decode passes replayed from CUDA graphs give bit-identical logits, the
    same cache bookkeeping and the same comm ledger as eager passes."""
    prompts = [c1_prompts()[i][:n] for i, n in ((0, 40), (1, 25), (2, 33))]
    res = {}
    for graphs in (False, True):
        eng = Engine(device_weights(c1, p), LoopbackGroup(p), ShiftPolicy(token_threshold=3),
                     cuda_graphs=graphs)
        seqs = [eng.new_sequence(i, capacity=80) for i in range(3)]
        eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, q) for s, q in zip(seqs, prompts)]))
        outs, recs = [], []
        toks = [1, 2, 3]
        for step in range(9):
            sub = seqs if step % 3 != 2 else seqs[:2]  # batch 3 -> SP, batch 2 -> TP (tau=3)
            lg, rec = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [t]) for s, t in zip(sub, toks)]))
            outs.append([x.cpu() for x in lg])
            recs.append((rec.mode, rec.flops_per_device, rec.comm))
            toks = [int(torch.argmax(x)) for x in lg] + [5]
        res[graphs] = (outs, recs, [s.cache.write_counter for s in seqs],
                       [s.cache.token_count for s in seqs])
        if graphs:
            # both keys captured (second sighting) AND replayed at least once
            by_mode = {k[0]: e for k, e in eng._graphs.items()}
            for mode in (ParallelMode.SP, ParallelMode.TP):
                assert by_mode[mode].graph is not None and by_mode[mode].replays >= 1, mode
    (o0, r0, w0, t0), (o1, r1, w1, t1) = res[False], res[True]
    assert r0 == r1 and w0 == w1 and t0 == t1
    for a, b in zip(o0, o1):
        for x, y in zip(a, b):
            assert torch.equal(x, y)


def test_graphs_survive_a_second_engine(c1):
    """captured decode graphs hold the split-K workspace address; a
    second Engine on the device must not free it.  Replays of engine A after
    engine B exists equal A's eager passes bit for bit."""
    prompt = c1_prompts()[0][:40]

    def run(graphs, interleave):
        eng = Engine(device_weights(c1, 1), LoopbackGroup(1), ShiftPolicy.fixed_tp(),
                     cuda_graphs=graphs)
        s = eng.new_sequence(0, capacity=64)
        eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, prompt)]))
        outs, tok, other = [], 7, None
        for step in range(5):
            if interleave and step == 2:   # after the capture: a second engine appears
                other = Engine(device_weights(c1, 1), LoopbackGroup(1), ShiftPolicy.fixed_tp())
                o = other.new_sequence(0, capacity=64)
                other.step(Batch(BatchKind.PREFILL, [BatchItem(o, prompt[:20])]))
                other.step(Batch(BatchKind.DECODE, [BatchItem(o, [3])]))
                torch.cuda.empty_cache()
            lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [tok])]))
            outs.append(lg[0].cpu())
            tok = int(torch.argmax(lg[0]))
        if graphs:
            assert sum(e.replays for e in eng._graphs.values()) >= 2
        return outs

    want = run(False, False)
    got = run(True, True)
    for a, b in zip(want, got):
        assert torch.equal(a, b)


@pytest.mark.parametrize("p", [2, 4])
def test_fused_peer_all_to_all_matches_collective_path(c1_kv4, p, monkeypatch):
    """The fused SP all-to-all (QKV epilogue storing into peers' receive buffers,
    attention rows scattered to owners, device flags) gives bit-identical logits
    and the same comm ledger as the collective path."""
    prompts = [c1_prompts()[i] for i in (1, 4, 6)]
    res = {}
    for fused in ("1", "0"):
        monkeypatch.setenv("SP_FUSED_A2A", fused)
        eng = make(c1_kv4, p)
        assert (eng._peer is not None) == (fused == "1")
        seqs = [eng.new_sequence(i, capacity=200) for i in range(3)]
        lg, rec = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, q) for s, q in zip(seqs, prompts)]),
                           mode=ParallelMode.SP, span_logits=True)
        out = [x.cpu() for x in lg]
        recs = [rec.comm]
        for step in range(3):  # decode (graph-captured after the first pass)
            lg, rec = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [5 + step]) for s in seqs]),
                               mode=ParallelMode.SP)
            out += [x.cpu() for x in lg]
            recs.append(rec.comm)
        res[fused] = (out, recs)
    for a, b in zip(res["1"][0], res["0"][0]):
        assert torch.equal(a, b)
    assert res["1"][1] == res["0"][1]


@pytest.mark.parametrize("p", [2, 4])
@pytest.mark.parametrize("span", [False, True])
def test_two_shot_tp_allreduce_matches_one_shot_and_collective(c1_kv4, p, span, monkeypatch):
    """Prefill-size TP passes (> SP_TP_TWO_SHOT_MIN_ROWS rows) reduce two-shot:
    each rank sums its row slice (ascending rank), adds the residual, norms and
    pushes bf16 rows to every peer.  Bit-identical logits, KV and ledger to the
    one-shot kernel and to the collective path; uneven row slices (M % P != 0)."""
    prompts = [c1_prompts()[i] for i in (0, 3, 5)]   # 349 tokens
    assert sum(len(q) for q in prompts) % p
    res = {}
    for name, env in (("two", {}), ("one", {"SP_TP_TWO_SHOT_MIN_ROWS": "100000"}),
                      ("coll", {"SP_FUSED_A2A": "0"})):
        for k in ("SP_TP_TWO_SHOT_MIN_ROWS", "SP_FUSED_A2A"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        eng = make(c1_kv4, p)
        seqs = [eng.new_sequence(i, capacity=200) for i in range(3)]
        lg, rec = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, q) for s, q in zip(seqs, prompts)]),
                           mode=ParallelMode.TP, span_logits=span)
        lg2, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [7]) for s in seqs]),
                          mode=ParallelMode.TP)
        k_, v_ = seqs[2].cache.read_window(p - 1, 3, 0)
        res[name] = ([x.cpu() for x in lg + lg2], rec.comm, k_.cpu(), v_.cpu(),
                     [s.cache.write_counter for s in seqs])
    for other in ("one", "coll"):
        for a, b in zip(res["two"][0], res[other][0]):
            assert torch.equal(a, b), other
        assert res["two"][1] == res[other][1]
        assert torch.equal(res["two"][2], res[other][2]) and torch.equal(res["two"][3], res[other][3])
        assert res["two"][4] == res[other][4]


@pytest.mark.parametrize("p", [2, 4])
def test_fused_tp_allreduce_matches_collective_path(c1_kv4, p, monkeypatch):
    """TP with the one-shot all-reduce fused into the add+RMSNorm kernel (partials
    summed from peer buffers in ascending rank order) is bit-identical to the
    collective path, prefill and graph-replayed decode, with the same ledger."""
    prompts = [c1_prompts()[i][:50] for i in (2, 3)]
    res = {}
    for fused in ("1", "0"):
        monkeypatch.setenv("SP_FUSED_A2A", fused)
        eng = make(c1_kv4, p)
        seqs = [eng.new_sequence(i, capacity=100) for i in range(2)]
        lg, rec = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, q) for s, q in zip(seqs, prompts)]),
                           mode=ParallelMode.TP, span_logits=True)
        out, recs = [x.cpu() for x in lg], [rec.comm]
        for step in range(3):
            lg, rec = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [9 + step]) for s in seqs]),
                               mode=ParallelMode.TP)
            out += [x.cpu() for x in lg]
            recs.append(rec.comm)
        res[fused] = (out, recs)
    for a, b in zip(res["1"][0], res["0"][0]):
        assert torch.equal(a, b)
    assert res["1"][1] == res["0"][1]


def test_sp_x_tp_mixed_mode(c1_kv4, monkeypatch):
    """SP(2) x TP(2) and SP(1) x TP(4) on P=4 (PAPER.md:95
    "SP x TP = P"; the reference leaves mixed modes unimplemented,
    SPEC.md:334): logits within the oracle tolerance and within 1e-2 of pure
    SP(4) (the TP all-reduce sums f32 partials where SP accumulates in one
    GEMM); the KV cache the mixed pass writes is bit-identical to SP(4)'s (mode
    invariance: same head block on the same rank, same GEMM K order); a TP(4)
    decode then runs on that cache against the oracle."""
    monkeypatch.setenv("SP_GEMM_NO_SPLITK", "1")
    prompts = [c1_prompts()[i] for i in (0, 3, 5)]
    res = {}
    for label, kw, mode in (("sp4", {}, ParallelMode.SP), ("tp4", {}, ParallelMode.TP),
                            ("sp2xtp2", {"sp_degree": 2}, ParallelMode.SP),
                            ("sp1xtp4", {"sp_degree": 1}, ParallelMode.SP)):
        eng = make(c1_kv4, 4, **kw)
        seqs = [eng.new_sequence(i, capacity=220) for i in range(3)]
        lg, rec = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, q) for s, q in
                                                     zip(seqs, prompts)]), mode=mode)
        res[label] = (eng, seqs, np.stack(to_np(lg)), rec)
    oeng = oracle.OracleEngine(c1_kv4, 1)
    oseqs = [oeng.new_sequence(i, capacity=220) for i in range(3)]
    olg, _ = oeng.step(list(zip(oseqs, prompts)), mode="sp")
    want = np.stack(olg)
    for label, (_, _, got, _) in res.items():
        assert rel_err(got, want) <= LOGIT_TOL, label
    assert rel_err(res["sp2xtp2"][2], res["sp4"][2]) <= 1e-2
    # the mixed pass wrote exactly the cache pure SP(4) writes (head block r on rank r)
    for label in ("sp2xtp2", "sp1xtp4"):
        a, b = res[label][1][0].cache, res["sp4"][1][0].cache
        assert a.fingerprint() == b.fingerprint()
        for dev in range(4):
            ka, va = a.device_blocks(dev)
            kb, vb = b.device_blocks(dev)
            assert torch.equal(ka[0], kb[0]) and torch.equal(va[0], vb[0]), (label, dev)
    # comm: all-to-alls inside SP groups, all-reduces inside TP groups
    kinds = {e.kind for e in res["sp2xtp2"][3].comm}
    assert {"all_to_all", "all_reduce"} <= kinds
    # shift: TP(4) decode on the cache the mixed prefill wrote
    eng, seqs, _, _ = res["sp2xtp2"]
    toks = [oracle.greedy_token(r) for r in want]
    lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [t]) for s, t in zip(seqs, toks)]),
                     mode=ParallelMode.TP)
    olg, _ = oeng.step([(s, [t]) for s, t in zip(oseqs, toks)], prefill=False, mode="sp")
    assert rel_err(np.stack(to_np(lg)), np.stack(olg)) <= LOGIT_TOL


@pytest.mark.parametrize("p", [2, 4])
def test_fused_exchange_tma_store_bitexact(p, monkeypatch):
    """8B-width SP prefill large enough for the 2-CTA GEMM regime (>= 256 rows
    per rank, N = P x W a multiple of 256): the seq->head exchange epilogue
    stages 32x64 boxes and TMA-stores them into each peer's receive rows.
    Logits and K/V are bit-identical to the direct-store epilogue
    (SP_PEER_TMA=0) and to the collective path (SP_FUSED_A2A=0)."""
    ow = init_weights_llama(llama_tiny_config(n_layers=2, n_heads=32, n_kv_heads=8, head_dim=128,
                                              ffn_dim=14336, vocab_size=1024, max_seq=2048), seed=3)
    rng = np.random.default_rng(11)
    prompts = [[int(t) for t in rng.integers(0, 1024, size=n)] for n in (700, 413)]  # uneven
    res = {}
    for name, env in (("tma", {}), ("direct", {"SP_PEER_TMA": "0"}), ("coll", {"SP_FUSED_A2A": "0"})):
        for k in ("SP_PEER_TMA", "SP_FUSED_A2A"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        eng = Engine(device_weights(ow, p), LoopbackGroup(p), ShiftPolicy.fixed_sp())
        seqs = [eng.new_sequence(i, capacity=800) for i in range(2)]
        lg, rec = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, q) for s, q in zip(seqs, prompts)]),
                           mode=ParallelMode.SP, span_logits=True)
        kv = [t.cpu() for r in range(p) for t in seqs[1].cache.read_window(r, 1, 0)]
        res[name] = ([x.cpu() for x in lg], kv, rec.comm)
    for other in ("direct", "coll"):
        for a, b in zip(res["tma"][0], res[other][0]):
            assert torch.equal(a, b), other
        for a, b in zip(res["tma"][1], res[other][1]):
            assert torch.equal(a, b), other
        assert res["tma"][2] == res[other][2]
