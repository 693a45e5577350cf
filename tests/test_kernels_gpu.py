"""Per-kernel numerics of libshiftpar.so on a B200 vs plain fp32 torch references.

Tolerances: the kernels read bf16 operands and accumulate in f32, exactly like
the fp32 reference computed from the same bf16 values, so f32 outputs agree to
accumulation-order noise (<=1e-4 of the output scale) and bf16 outputs to one
bf16 ulp (<=1e-2 relative of the output scale).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ops = pytest.importorskip("paper_2507_11830_b200.ops")


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ops.device_check()


def rnd(*shape, scale=1.0, seed=0, dtype=torch.bfloat16):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(*shape, generator=g, device="cuda") * scale).to(dtype)


def rel(a, b):
    return float((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-30))


GEMM_SHAPES = [(1, 256, 64), (7, 384, 256), (128, 256, 4096), (300, 512, 1024), (1000, 768, 512),
               (257, 6144, 4096), (2048, 1024, 2048), (64, 96, 128)]


@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_gemm_f32_and_bf16(M, N, K):
    a, b = rnd(M, K, seed=1), rnd(N, K, seed=2)
    ref = a.float() @ b.float().t()
    d32 = torch.empty(M, N, device="cuda")
    ops.gemm(a, b, d32, ops.EPI_STORE_F32, M=M, N=N, K=K, lda=K, ldb=K, ldd=N)
    assert rel(d32, ref) < 1e-4
    d16 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ops.gemm(a, b, d16, ops.EPI_STORE_BF16, M=M, N=N, K=K, lda=K, ldb=K, ldd=N)
    assert rel(d16, ref) < 1e-2


def test_gemm_add_f32_residual():
    M, N, K = 333, 512, 768
    a, b = rnd(M, K, seed=3), rnd(N, K, seed=4)
    x = torch.randn(M, N, device="cuda")
    want = x + a.float() @ b.float().t()
    ops.gemm(a, b, x, ops.EPI_ADD_F32, M=M, N=N, K=K, lda=K, ldb=K, ldd=N)
    assert rel(x, want) < 1e-4


def test_gemm_swiglu_interleaved():
    M, f, K = 200, 512, 256
    a = rnd(M, K, seed=5)
    gate, up = rnd(f, K, seed=6), rnd(f, K, seed=7)
    w = torch.empty(2 * f, K, device="cuda", dtype=torch.bfloat16)
    v = w.view(f // 128, 2, 128, K)
    v[:, 0] = gate.view(f // 128, 128, K)
    v[:, 1] = up.view(f // 128, 128, K)
    g = a.float() @ gate.float().t()
    u = a.float() @ up.float().t()
    want = torch.nn.functional.silu(g) * u
    d = torch.empty(M, f, device="cuda", dtype=torch.bfloat16)
    ops.gemm(a, w, d, ops.EPI_SWIGLU, M=M, N=2 * f, K=K, lda=K, ldb=K, ldd=f)
    assert rel(d, want) < 1e-2


def test_gemm_gelu():
    M, N, K = 100, 256, 128
    a, b = rnd(M, K, seed=8), rnd(N, K, seed=9)
    want = torch.nn.functional.gelu(a.float() @ b.float().t(), approximate="tanh")
    d = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ops.gemm(a, b, d, ops.EPI_GELU, M=M, N=N, K=K, lda=K, ldb=K, ldd=N)
    assert rel(d, want) < 1e-2


def test_gemm_peer_layout_and_chunked_a():
    P, rows, W, K = 4, 37, 96, 256
    a, b = rnd(rows, K, seed=10), rnd(P * W, K, seed=11)
    ref = torch.empty(rows, P * W, device="cuda", dtype=torch.bfloat16)
    ops.gemm(a, b, ref, ops.EPI_STORE_BF16, M=rows, N=P * W, K=K, lda=K, ldb=K, ldd=P * W)
    assert rel(ref, a.float() @ b.float().t()) < 1e-2
    send = torch.empty(P * rows, W, device="cuda", dtype=torch.bfloat16)
    ops.gemm(a, b, send, ops.EPI_STORE_BF16, M=rows, N=P * W, K=K, lda=K, ldb=K, ldd=W,
             peer_width=W, peer_stride=rows * W)
    for s in range(P):
        assert torch.equal(send[s * rows:(s + 1) * rows], ref[:, s * W:(s + 1) * W])
    # chunked-K A: back[P][rows][w] acts as A[rows, P*w]
    w = 128
    back = rnd(P * rows, w, seed=12)
    flat = torch.cat([back[s * rows:(s + 1) * rows] for s in range(P)], dim=1)
    wo = rnd(256, P * w, seed=13)
    want = flat.float() @ wo.float().t()
    d = torch.zeros(rows, 256, device="cuda")
    ops.gemm(back, wo, d, ops.EPI_ADD_F32, M=rows, N=256, K=P * w, lda=w, ldb=P * w, ldd=256,
             a_kchunk=w, a_chunk_stride=rows * w)
    assert rel(d, want) < 1e-4


def test_gemm_strided_b_window_is_zero_copy_tp_shard():
    M, N, Kfull, P = 64, 256, 1024, 4
    a_full, b = rnd(M, Kfull, seed=14), rnd(N, Kfull, seed=15)
    kl = Kfull // P
    for r in range(P):
        a = a_full[:, r * kl:(r + 1) * kl].contiguous()
        want = a.float() @ b[:, r * kl:(r + 1) * kl].float().t()
        d = torch.empty(M, N, device="cuda")
        ops.gemm(a, b[:, r * kl:], d, ops.EPI_STORE_F32, M=M, N=N, K=kl, lda=kl, ldb=Kfull, ldd=N)
        assert rel(d, want) < 1e-4


def test_gemm_row_and_column_splits_bitexact(monkeypatch):
    """tensor_core.py:1-28 property on the GPU: fixed tiles, no split-K (the
    split-K regime for decode-size M is pinned off here)."""
    monkeypatch.setenv("SP_GEMM_NO_SPLITK", "1")
    M, N, K = 700, 1024, 512
    a, b = rnd(M, K, seed=16), rnd(N, K, seed=17)
    full = torch.empty(M, N, device="cuda")
    ops.gemm(a, b, full, ops.EPI_STORE_F32, M=M, N=N, K=K, lda=K, ldb=K, ldd=N)
    for lo, hi in ((0, 1), (1, 300), (300, 700)):
        part = torch.empty(hi - lo, N, device="cuda")
        ops.gemm(a[lo:hi], b, part, ops.EPI_STORE_F32, M=hi - lo, N=N, K=K, lda=K, ldb=K, ldd=N)
        assert torch.equal(part, full[lo:hi])
    for lo, hi in ((0, 256), (256, 768), (768, 1024)):
        part = torch.empty(M, hi - lo, device="cuda")
        ops.gemm(a, b[lo:hi], part, ops.EPI_STORE_F32, M=M, N=hi - lo, K=K, lda=K, ldb=K,
                 ldd=hi - lo)
        assert torch.equal(part, full[:, lo:hi])


def test_embed_and_rmsnorm():
    V, h, rows = 1000, 512, 77
    table = rnd(V, h, seed=18)
    ids = torch.randint(0, V, (rows,), device="cuda", dtype=torch.int32)
    x = torch.empty(rows, h, device="cuda")
    ops.embed(ids, table, x)
    assert torch.equal(x, table[ids.long()].float())
    gain = torch.rand(h, device="cuda") + 0.5
    add = torch.randn(rows, h, device="cuda")
    x0 = x.clone()
    out = torch.empty(rows, h, device="cuda", dtype=torch.bfloat16)
    ops.add_rmsnorm(x, gain, 1e-5, out, add=add)
    xs = x0 + add
    assert torch.allclose(x, xs)
    want = gain * (xs / torch.sqrt((xs * xs).mean(-1, keepdim=True) + 1e-5))
    assert rel(out, want) < 1e-2
    idx = torch.tensor([3, 0, 76], device="cuda", dtype=torch.int32)
    o2 = torch.empty(3, h, device="cuda", dtype=torch.bfloat16)
    ops.add_rmsnorm(x, gain, 1e-5, o2, row_idx=idx)
    assert torch.equal(o2, out[idx.long()])


def _rope_ref(x, pos, tab):
    d = x.shape[-1]
    c = tab[pos.long(), :, 0][:, None, :]
    s = tab[pos.long(), :, 1][:, None, :]
    lo, hi = x[..., :d // 2], x[..., d // 2:]
    return torch.cat([lo * c - hi * s, hi * c + lo * s], dim=-1)


def test_rope_kv_write_paged():
    from paper_2507_11830_b200.weights import rope_table
    hq, hk, d, bs, nblk, rows = 4, 2, 64, 16, 10, 40
    tab = torch.as_tensor(rope_table(256, d, 500000.0, None), device="cuda")
    qkv = rnd(rows, (hq + 2 * hk) * d, seed=19)
    pos = torch.arange(5, 5 + rows, device="cuda", dtype=torch.int32)
    perm = torch.randperm(nblk * bs, device="cuda")[:rows].to(torch.int32)
    kpool = torch.zeros(nblk, hk, bs, d, device="cuda", dtype=torch.bfloat16)
    vpool = torch.zeros_like(kpool)
    q = torch.empty(rows, hq * d, device="cuda", dtype=torch.bfloat16)
    ops.rope_kv_write(qkv, pos, perm, tab, q, kpool, vpool, rows=rows, q_heads=hq, kv_heads=hk,
                      head_dim=d, block_size=bs)
    x = qkv.float().view(rows, hq + 2 * hk, d)
    q_ref = _rope_ref(x[:, :hq], pos, tab)
    k_ref = _rope_ref(x[:, hq:hq + hk], pos, tab)
    assert rel(q.view(rows, hq, d), q_ref) < 1e-2
    blk, off = (perm // bs).long(), (perm % bs).long()
    got_k = kpool[blk, :, off]  # [rows, hk, d]
    got_v = vpool[blk, :, off]
    assert rel(got_k, k_ref) < 1e-2
    assert torch.equal(got_v, qkv.view(rows, hq + 2 * hk, d)[:, hq + hk:])


def _attn_ref(q, k, v, first_pos):
    """q [m, H, d], k/v [T, Hkv, d] -> [m, H, d] with causal window semantics."""
    m, H, d = q.shape
    T, Hk, _ = k.shape
    G = H // Hk
    out = torch.empty(m, H, d, device=q.device)
    for hh in range(H):
        s = q[:, hh].float() @ k[:, hh // G].float().t() / d ** 0.5
        ok = torch.arange(T, device=q.device)[None] <= (first_pos + torch.arange(m, device=q.device))[:, None]
        s = s.masked_fill(~ok, float("-inf"))
        out[:, hh] = torch.softmax(s, -1) @ v[:, hh // G].float()
    return out


def _paged(kv_list, hk, d, bs):
    """Scatter per-item [T, hk, d] into a pool with a shuffled block table."""
    nblk = sum(-(-t.shape[0] // bs) for t in kv_list) + 3
    order = torch.randperm(nblk).tolist()
    pool = torch.zeros(nblk, hk, bs, d, device="cuda", dtype=torch.bfloat16)
    tables, nxt = [], 0
    for t in kv_list:
        nb = -(-t.shape[0] // bs)
        tab = order[nxt:nxt + nb]
        nxt += nb
        for j in range(t.shape[0]):
            pool[tab[j // bs], :, j % bs] = t[j]
        tables.append(tab)
    width = max(len(t) for t in tables)
    bt = torch.zeros(len(tables), width, dtype=torch.int32, device="cuda")
    for i, t in enumerate(tables):
        bt[i, :len(t)] = torch.tensor(t, dtype=torch.int32)
    return pool, bt


@pytest.mark.parametrize("d,hq,hk,bs", [(128, 8, 2, 64), (64, 4, 4, 16), (32, 8, 2, 32),
                                        (128, 32, 8, 64)])
def test_attention_prefill_paged_causal(d, hq, hk, bs):
    torch.manual_seed(0)
    spans = [37, 130, 1, 64]
    hist = [0, 20, 70, 5]
    ks, vs, qs = [], [], []
    for m, t0 in zip(spans, hist):
        ks.append(rnd(t0 + m, hk, d, seed=20 + m))
        vs.append(rnd(t0 + m, hk, d, seed=40 + m))
        qs.append(rnd(m, hq, d, seed=60 + m))
    kpool, bt = _paged(ks, hk, d, bs)
    vpool, bt2 = _paged(vs, hk, d, bs)
    # same table for k and v: rebuild v with k's table
    vpool = torch.zeros_like(kpool)
    for i, t in enumerate(vs):
        tab = bt[i].tolist()
        for j in range(t.shape[0]):
            vpool[tab[j // bs], :, j % bs] = t[j]
    q = torch.cat(qs).view(-1, hq * d)
    M = q.shape[0]
    cu = torch.tensor([0] + list(np.cumsum(spans)), dtype=torch.int32, device="cuda")
    first = torch.tensor(hist, dtype=torch.int32, device="cuda")
    kvl = torch.tensor([a + b for a, b in zip(spans, hist)], dtype=torch.int32, device="cuda")
    tt = ops.attn_tile_tokens(hq, hk, d, bs)
    work = [(i, t0) for i, m in enumerate(spans) for t0 in range(0, m, tt)]
    work_t = torch.tensor(work, dtype=torch.int32, device="cuda").view(-1)
    out = torch.empty(M, hq * d, device="cuda", dtype=torch.bfloat16)
    ops.attention(q, kpool, vpool, bt, cu, first, kvl, out, n_items=len(spans), work=work_t,
                  n_work=len(work), max_q_len=max(spans), max_kv_len=int(kvl.max()), q_heads=hq,
                  kv_heads=hk, head_dim=d, block_size=bs, ws=None)
    lo = 0
    for i, (m, t0) in enumerate(zip(spans, hist)):
        want = _attn_ref(qs[i], ks[i], vs[i], t0)
        assert rel(out[lo:lo + m].view(m, hq, d), want) < 2e-2, i
        lo += m


@pytest.mark.parametrize("d,hq,hk,ctx", [(128, 32, 8, 2048), (128, 8, 2, 100), (64, 4, 4, 5000),
                                         (32, 8, 2, 1), (128, 8, 2, 5000), (128, 32, 2, 700),
                                         (128, 64, 8, 300)])
@pytest.mark.parametrize("tc", ["0", "1"])
def test_attention_decode_split_kv(d, hq, hk, ctx, tc, monkeypatch):
    """Split-KV decode (TMA kernel with the first ring of old pages streamed
    before the PDL wait; splits merged by the combine kernel) vs the reference,
    with the mma.sync consumers (tc=0) and the tcgen05/TMEM ones (tc=1: Q as
    the TMEM A operand, S and O in TMEM; d=128 only)."""
    monkeypatch.setenv("SP_DECODE_TC", tc)
    n = 5
    bs = 64
    ctxs = [ctx + 7 * i for i in range(n)]
    ks = [rnd(c, hk, d, seed=100 + i) for i, c in enumerate(ctxs)]
    vs = [rnd(c, hk, d, seed=200 + i) for i, c in enumerate(ctxs)]
    qs = [rnd(1, hq, d, seed=300 + i) for i in range(n)]
    kpool, bt = _paged(ks, hk, d, bs)
    vpool = torch.zeros_like(kpool)
    for i, t in enumerate(vs):
        tab = bt[i].tolist()
        for j in range(t.shape[0]):
            vpool[tab[j // bs], :, j % bs] = t[j]
    q = torch.cat(qs).view(n, hq * d)
    cu = torch.arange(n + 1, dtype=torch.int32, device="cuda")
    kvl = torch.tensor(ctxs, dtype=torch.int32, device="cuda")
    first = kvl - 1
    ws = torch.empty(ops.attn_workspace_bytes(n, hq, d, max(ctxs)) // 4, device="cuda")
    out = torch.empty(n, hq * d, device="cuda", dtype=torch.bfloat16)
    ops.attention(q, kpool, vpool, bt, cu, first, kvl, out, n_items=n, work=None, n_work=0,
                  max_q_len=1, max_kv_len=max(ctxs), q_heads=hq, kv_heads=hk, head_dim=d,
                  block_size=bs, ws=ws)
    for i in range(n):
        want = _attn_ref(qs[i], ks[i], vs[i], ctxs[i] - 1)
        assert rel(out[i].view(1, hq, d), want) < 2e-2, i


def test_pack_unpack_roundtrip_and_add_argmax():
    rows, P, w = 33, 4, 64
    src = rnd(rows, P * w, seed=400)
    packed = torch.empty(P * rows, w, device="cuda", dtype=torch.bfloat16)
    ops.a2a_pack(src, packed, rows, P, w)
    for s in range(P):
        assert torch.equal(packed[s * rows:(s + 1) * rows], src[:, s * w:(s + 1) * w])
    back = torch.empty_like(src)
    ops.a2a_unpack(packed, back, rows, P, w)
    assert torch.equal(back, src)
    a, b = torch.randn(1001, device="cuda"), torch.randn(1001, device="cuda")
    c = torch.empty_like(a)
    ops.add_f32(a, b, c)
    assert torch.equal(c, a + b)
    lg = torch.randn(6, 50000, device="cuda")
    lg[2, 7] = lg[2, 9] = 1e4  # tie -> lowest index (model.py:303-307)
    idx = torch.empty(6, dtype=torch.int32, device="cuda")
    ops.argmax(lg, idx)
    want = lg.argmax(-1).to(torch.int32)
    assert torch.equal(idx, want) and int(idx[2]) == 7


def test_gemm_tile_width_variants_are_bitexact(monkeypatch):
    """The N-tile variants (256/128/64/32, picked by M and N) share the K loop, so
    an output element does not depend on which variant computed it."""
    monkeypatch.setenv("SP_GEMM_NO_SPLITK", "1")
    monkeypatch.setenv("SP_GEMM_NO_SPLITK", "1")  # M = 200 would take the swap-AB regime
    M, N, K = 200, 768, 1024
    a, b = rnd(M, K, seed=30), rnd(N, K, seed=31)
    outs = {}
    for bn in ("256", "128", "64", "32"):
        monkeypatch.setenv("SP_GEMM_FORCE_BN", bn)
        d = torch.empty(M, N, device="cuda")
        ops.gemm(a, b, d, ops.EPI_STORE_F32, M=M, N=N, K=K, lda=K, ldb=K, ldd=N)
        x = torch.ones(M, N, device="cuda")
        ops.gemm(a, b, x, ops.EPI_ADD_F32, M=M, N=N, K=K, lda=K, ldb=K, ldd=N)
        outs[bn] = (d, x)
    for bn, (d, x) in outs.items():
        assert torch.equal(d, outs["256"][0]), bn
        assert torch.equal(x, outs["256"][1]), bn
    assert rel(outs["32"][0], a.float() @ b.float().t()) < 1e-4


@pytest.mark.parametrize("N,K", [(1024, 4096), (2560, 512), (384, 192), (128256, 128)])
@pytest.mark.parametrize("M", [1, 48, 100, 200, 256])
@pytest.mark.parametrize("epi", ["f32", "add", "bf16", "swiglu", "gelu", "peer", "chunked"])
def test_gemm_split_k_regime(epi, M, N, K):
    """Decode-size M: swap-AB stream-K (equal weight share per CTA; super tiles
    split across CTAs summed in ascending-K order by their last CTA).  Shapes
    cover many-CTA tiles (2560x512), a half-empty last super tile (384), and
    whole tiles finished in place (128256x128).  Deterministic run to run;
    within f32 accumulation noise of the reference."""
    if epi == "swiglu" and N % 256:
        pytest.skip("SwiGLU needs gate|up pairs of 128 rows")
    if epi == "chunked" and (K // 4) % 64:
        pytest.skip("chunked-K A needs 64-multiple chunks")
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    ops.set_gemm_workspace(ws)
    try:
        a, b = rnd(M, K, seed=40), rnd(N, K, seed=41)
        ref = a.float() @ b.float().t()
        outs = []
        for _ in range(2):
            if epi == "f32":
                d = torch.empty(M, N, device="cuda")
                ops.gemm(a, b, d, ops.EPI_STORE_F32, M=M, N=N, K=K, lda=K, ldb=K, ldd=N)
                want, tol = ref, 1e-4
            elif epi == "add":
                d = torch.ones(M, N, device="cuda")
                ops.gemm(a, b, d, ops.EPI_ADD_F32, M=M, N=N, K=K, lda=K, ldb=K, ldd=N)
                want, tol = ref + 1, 1e-4
            elif epi == "bf16":
                d = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
                ops.gemm(a, b, d, ops.EPI_STORE_BF16, M=M, N=N, K=K, lda=K, ldb=K, ldd=N)
                want, tol = ref, 1e-2
            elif epi == "gelu":
                d = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
                ops.gemm(a, b, d, ops.EPI_GELU, M=M, N=N, K=K, lda=K, ldb=K, ldd=N)
                want, tol = torch.nn.functional.gelu(ref, approximate="tanh"), 1e-2
            elif epi == "swiglu":
                f = N // 2
                d = torch.empty(M, f, device="cuda", dtype=torch.bfloat16)
                ops.gemm(a, b, d, ops.EPI_SWIGLU, M=M, N=N, K=K, lda=K, ldb=K, ldd=f)
                v = ref.view(M, f // 128, 2, 128)
                want = (torch.nn.functional.silu(v[:, :, 0]) * v[:, :, 1]).reshape(M, f)
                tol = 1e-2
            elif epi == "chunked":
                P, w = 4, K // 4  # SP O-proj: A is the [P][rows][w] all-to-all receive
                back = torch.cat([a[:, s * w:(s + 1) * w] for s in range(P)], dim=0).contiguous()
                d = torch.zeros(M, N, device="cuda")
                ops.gemm(back, b, d, ops.EPI_ADD_F32, M=M, N=N, K=K, lda=w, ldb=K, ldd=N,
                         a_kchunk=w, a_chunk_stride=M * w)
                want, tol = ref, 1e-4
            else:
                P, W = 4, N // 4
                d = torch.empty(P * M, W, device="cuda", dtype=torch.bfloat16)
                ops.gemm(a, b, d, ops.EPI_STORE_BF16, M=M, N=N, K=K, lda=K, ldb=K, ldd=W,
                         peer_width=W, peer_stride=M * W)
                d = torch.cat([d[s * M:(s + 1) * M] for s in range(P)], dim=1)
                want, tol = ref, 1e-2
            outs.append(d.clone())
            assert rel(d, want) < tol
        assert torch.equal(outs[0], outs[1])
    finally:
        ops.set_gemm_workspace(None)


@pytest.mark.parametrize("epi", ["f32", "add", "bf16", "swiglu", "chunked"])
def test_gemm_cta_pair_large_tiles(epi, monkeypatch):
    """Large GEMMs run on CTA pairs (tcgen05.mma.cta_group::2, 256x256 tiles);
    results are bit-identical to the single-CTA kernel and match fp32."""
    M, N, K = 1000, 8192, 1024
    a, b = rnd(M, K, seed=50), rnd(N, K, seed=51)
    ref = a.float() @ b.float().t()
    outs = {}
    for pair_on in ("1", "0"):
        monkeypatch.setenv("SP_GEMM_2CTA", pair_on)
        if epi == "f32":
            d = torch.empty(M, N, device="cuda")
            ops.gemm(a, b, d, ops.EPI_STORE_F32, M=M, N=N, K=K, lda=K, ldb=K, ldd=N)
            want, tol = ref, 1e-4
        elif epi == "add":
            d = torch.full((M, N), 0.5, device="cuda")
            ops.gemm(a, b, d, ops.EPI_ADD_F32, M=M, N=N, K=K, lda=K, ldb=K, ldd=N)
            want, tol = ref + 0.5, 1e-4
        elif epi == "bf16":
            d = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            ops.gemm(a, b, d, ops.EPI_STORE_BF16, M=M, N=N, K=K, lda=K, ldb=K, ldd=N)
            want, tol = ref, 1e-2
        elif epi == "swiglu":
            f = N // 2
            d = torch.empty(M, f, device="cuda", dtype=torch.bfloat16)
            ops.gemm(a, b, d, ops.EPI_SWIGLU, M=M, N=N, K=K, lda=K, ldb=K, ldd=f)
            v = ref.view(M, f // 128, 2, 128)
            want, tol = (torch.nn.functional.silu(v[:, :, 0]) * v[:, :, 1]).reshape(M, f), 1e-2
        else:
            P, w = 4, K // 4
            back = torch.cat([a[:, s * w:(s + 1) * w] for s in range(P)], dim=0).contiguous()
            d = torch.zeros(M, N, device="cuda")
            ops.gemm(back, b, d, ops.EPI_ADD_F32, M=M, N=N, K=K, lda=w, ldb=K, ldd=N,
                     a_kchunk=w, a_chunk_stride=M * w)
            want, tol = ref, 1e-4
        assert rel(d, want) < tol, pair_on
        outs[pair_on] = d
    assert torch.equal(outs["1"], outs["0"])


@pytest.mark.parametrize("M", [1, 7, 32])
def test_gemm_vocab_wide_swap_regime(M):
    """Projections with at least one 256-row weight tile per SM (the LM head,
    70B gate/up) run swap-AB up to 32 tokens (items looped per CTA): f32
    logits and the SwiGLU epilogue match fp32."""
    from paper_2507_11830_b200 import _lib
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    assert _lib.load().sp_gemm_plan(M, 128256, 1024, ops.EPI_STORE_F32, sms) == 0
    K = 1024
    a = rnd(M, K, seed=60)
    w = rnd(128256, K, seed=61, scale=0.05)
    d = torch.empty(M, 128256, device="cuda")
    ops.gemm(a, w, d, ops.EPI_STORE_F32, M=M, N=128256, K=K, lda=K, ldb=K, ldd=128256)
    assert rel(d, a.float() @ w.float().t()) < 1e-4
    N = 57344
    g = rnd(N, K, seed=62, scale=0.05)
    act = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
    ops.gemm(a, g, act, ops.EPI_SWIGLU, M=M, N=N, K=K, lda=K, ldb=K, ldd=N // 2)
    v = (a.float() @ g.float().t()).view(M, N // 256, 2, 128)
    want = (torch.nn.functional.silu(v[:, :, 0]) * v[:, :, 1]).reshape(M, N // 2)
    assert rel(act, want) < 1e-2


@pytest.mark.parametrize("M,ldd", [(1000, 4096), (777, 4352), (8192, 4096)])
def test_gemm_pair_residual_add_tma_bitexact(M, ldd, monkeypatch):
    """The pair kernel's residual add through TMA boxes (SP_ADD_TMA, default on)
    is bit-identical to the direct per-row read-modify-write, on ragged row
    counts (OOB rows of the last box neither read nor written) and on a
    residual with a row stride wider than N (columns past N untouched)."""
    N, K = 4096, 1024
    a, b = rnd(M, K, seed=52), rnd(N, K, seed=53)
    base = torch.randn(M, ldd, device="cuda", generator=torch.Generator("cuda").manual_seed(54))
    outs = {}
    for on in ("1", "0"):
        monkeypatch.setenv("SP_ADD_TMA", on)
        d = base.clone()
        ops.gemm(a, b, d, ops.EPI_ADD_F32, M=M, N=N, K=K, lda=K, ldb=K, ldd=ldd)
        torch.cuda.synchronize()
        assert torch.equal(d[:, N:], base[:, N:])
        assert rel(d[:, :N], base[:, :N] + a.float() @ b.float().t()) < 1e-4
        outs[on] = d
    assert torch.equal(outs["1"], outs["0"])


@pytest.mark.parametrize("epi", ["bf16", "swiglu", "gelu"])
@pytest.mark.parametrize("M,pad", [(1000, 0), (777, 64), (4096, 0)])
def test_gemm_pair_bf16_store_tma_bitexact(epi, M, pad, monkeypatch):
    """bf16 epilogues of the pair kernel through TMA boxes (SP_STORE_TMA,
    default on) are bit-identical to the direct row stores, on ragged rows and
    on an output with a row stride wider than its columns (padding untouched)."""
    N, K = 4096, 1024
    a, b = rnd(M, K, seed=55), rnd(N, K, seed=56)
    code = {"bf16": ops.EPI_STORE_BF16, "swiglu": ops.EPI_SWIGLU, "gelu": ops.EPI_GELU}[epi]
    cols = N // 2 if epi == "swiglu" else N
    outs = {}
    for on in ("1", "0"):
        monkeypatch.setenv("SP_STORE_TMA", on)
        d = torch.full((M, cols + pad), 7.0, device="cuda", dtype=torch.bfloat16)
        ops.gemm(a, b, d, code, M=M, N=N, K=K, lda=K, ldb=K, ldd=cols + pad)
        torch.cuda.synchronize()
        assert bool((d[:, cols:] == 7.0).all())
        outs[on] = d
    ref = a.float() @ b.float().t()
    if epi == "swiglu":
        v = ref.view(M, N // 256, 2, 128)
        ref = (torch.nn.functional.silu(v[:, :, 0]) * v[:, :, 1]).reshape(M, cols)
    elif epi == "gelu":
        ref = torch.nn.functional.gelu(ref, approximate="tanh")
    assert rel(outs["1"][:, :cols], ref) < 1e-2
    assert torch.equal(outs["1"], outs["0"])


@pytest.mark.parametrize("M,N,K", [(64, 4096, 4096), (1, 4096, 14336), (100, 1024, 4096),
                                   (200, 4096, 4096), (300, 512, 1024)])
def test_gemm_partials_fused_into_rmsnorm_bitexact(M, N, K):
    """EPI_PARTIAL_F32 + add_rmsnorm(n_add) (the split-K reduction fused into
    the next norm) is bit-identical to EPI_ADD_F32 + add_rmsnorm; outside the
    split-K (decode, M <= 256) regime one 'partial' is the plain result."""
    ops.set_gemm_workspace(torch.empty(64 << 20, dtype=torch.uint8, device="cuda"))
    try:
        a, b = rnd(M, K, seed=60), rnd(N, K, seed=61)
        x0 = torch.randn(M, N, device="cuda")
        gain = torch.rand(N, device="cuda") + 0.5
        n = ops.gemm_partials(M, N, K)
        assert n >= 1 and (M <= 256 or n == 1)
        x1 = x0.clone()
        ops.gemm(a, b, x1, ops.EPI_ADD_F32, M=M, N=N, K=K, lda=K, ldb=K, ldd=N)
        o1 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        ops.add_rmsnorm(x1, gain, 1e-5, o1)
        parts = torch.full((n, M, N), float("nan"), device="cuda")
        ops.gemm(a, b, parts, ops.EPI_PARTIAL_F32, M=M, N=N, K=K, lda=K, ldb=K, ldd=N)
        x2 = x0.clone()
        o2 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        ops.add_rmsnorm(x2, gain, 1e-5, o2, add=parts, n_add=n)
        assert torch.equal(x1, x2)
        assert torch.equal(o1, o2)
        assert rel(parts.sum(0), a.float() @ b.float().t()) < 1e-4
    finally:
        ops.set_gemm_workspace(None)


@pytest.mark.parametrize("P,M,N,K", [(2, 16, 4096, 4096), (4, 3, 4096, 3584), (2, 200, 1024, 2048)])
def test_peer_allreduce_from_partial_slabs_bitexact(P, M, N, K):
    """The one-shot TP all-reduce reading each rank's K-split slabs (the O/down
    GEMM's EPI_PARTIAL_F32 output, no reduce kernel) equals the all-reduce of
    the GEMM-reduced partials (EPI_STORE_F32), x and the normed output alike."""
    ops.set_gemm_workspace(torch.empty(64 << 20, dtype=torch.uint8, device="cuda"))
    try:
        n = ops.gemm_partials(M, N, K)
        x0 = torch.randn(M, N, device="cuda")
        gain = torch.rand(N, device="cuda") + 0.5
        slabs, whole = [], []
        for r in range(P):
            a, b = rnd(M, K, seed=70 + r), rnd(N, K, seed=80 + r)
            s = torch.full((n, M, N), float("nan"), device="cuda")
            ops.gemm(a, b, s, ops.EPI_PARTIAL_F32, M=M, N=N, K=K, lda=K, ldb=K, ldd=N)
            w = torch.empty(M, N, device="cuda")
            ops.gemm(a, b, w, ops.EPI_STORE_F32, M=M, N=N, K=K, lda=K, ldb=K, ldd=N)
            slabs.append(s)
            whole.append(w)
        outs = []
        for bufs, k in ((slabs, n), (whole, 1)):
            ptrs = torch.tensor([t.data_ptr() for t in bufs], dtype=torch.int64, device="cuda")
            x = x0.clone()
            o = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            ops.peer_allreduce_add_rmsnorm(ptrs, P, x, gain, 1e-5, o, M, slabs=k)
            outs.append((x, o))
        assert torch.equal(outs[0][0], outs[1][0])
        assert torch.equal(outs[0][1], outs[1][1])
        want = x0 + sum(w for w in whole)
        assert rel(outs[0][0], want) < 1e-5
    finally:
        ops.set_gemm_workspace(None)


@pytest.mark.parametrize("M,hq,hk,pair", [(300, 32, 8, "1"), (1000, 4, 1, "1"), (1000, 4, 1, "0"),
                                         (200, 8, 2, "1"), (2048, 16, 4, "1")])
def test_gemm_qkv_rope_fused_bitexact(M, hq, hk, pair, monkeypatch):
    """QKV GEMM with RoPE + paged KV write in its epilogue (2-CTA pairs or the
    1-CTA 128x256 tile) == GEMM(bf16) then rope_kv_write, bit for bit; rows
    with slot -1 write no K/V."""
    monkeypatch.setenv("SP_GEMM_2CTA", pair)
    from paper_2507_11830_b200.weights import rope_table
    d, bs, K = 128, 64, 1024
    W = (hq + 2 * hk) * d
    a, w = rnd(M, K, seed=90), rnd(W, K, seed=91, scale=0.05)
    pos = (torch.arange(M, dtype=torch.int32, device="cuda") * 7) % 4000
    nblk = -(-M // bs) + 4
    slot = torch.randperm(nblk * bs, device="cuda")[:M].to(torch.int32)
    slot[::17] = -1
    tab = torch.from_numpy(rope_table(4096, d, 500000.0, None)).cuda()
    res = []
    for fused in (True, False):
        kp = torch.zeros(nblk, hk, bs, d, device="cuda", dtype=torch.bfloat16)
        vp = torch.zeros_like(kp)
        q = torch.zeros(M, hq * d, device="cuda", dtype=torch.bfloat16)
        if fused:
            ops.gemm_qkv_rope(a, w, M=M, K=K, lda=K, ldb=K, pos=pos, slot=slot, rope=tab, q_out=q,
                              k_pool=kp, v_pool=vp, q_heads=hq, kv_heads=hk, block_size=bs)
        else:
            qkv = torch.empty(M, W, device="cuda", dtype=torch.bfloat16)
            monkeypatch.setenv("SP_GEMM_NO_SPLITK", "1")  # the same (non-swap) GEMM regime
            ops.gemm(a, w, qkv, ops.EPI_STORE_BF16, M=M, N=W, K=K, lda=K, ldb=K, ldd=W)
            monkeypatch.delenv("SP_GEMM_NO_SPLITK")
            ops.rope_kv_write(qkv, pos, slot, tab, q, kp, vp, rows=M, q_heads=hq, kv_heads=hk,
                              head_dim=d, block_size=bs)
        res.append((q, kp, vp))
    for x, y in zip(res[0], res[1]):
        assert torch.equal(x, y)
    assert res[0][1].abs().sum() > 0 and res[0][2].abs().sum() > 0


def test_rope_kv_write_from_partials_bitexact():
    """QKV projection left as K-split partials, reduced inside RoPE + KV write,
    equals the bf16 projection (reduced by the GEMM) fed to RoPE + KV write."""
    ops.set_gemm_workspace(torch.empty(64 << 20, dtype=torch.uint8, device="cuda"))
    try:
        M, hq, hk, d, bs, K = 48, 32, 8, 128, 64, 4096
        W = (hq + 2 * hk) * d
        a, w = rnd(M, K, seed=70), rnd(W, K, seed=71, scale=0.02)
        n = ops.gemm_partials(M, W, K)
        assert n > 1
        qkv = torch.empty(M, W, device="cuda", dtype=torch.bfloat16)
        ops.gemm(a, w, qkv, ops.EPI_STORE_BF16, M=M, N=W, K=K, lda=K, ldb=K, ldd=W)
        parts = torch.empty(n, M, W, device="cuda")
        ops.gemm(a, w, parts, ops.EPI_PARTIAL_F32, M=M, N=W, K=K, lda=K, ldb=K, ldd=W)
        pos = torch.arange(M, dtype=torch.int32, device="cuda") * 3
        slot = torch.randperm(4 * bs, device="cuda")[:M].to(torch.int32)
        from paper_2507_11830_b200.weights import rope_table
        tab = torch.from_numpy(rope_table(4096, d, 500000.0, None)).cuda()
        outs = []
        for use_parts in (False, True):
            q = torch.empty(M, hq * d, device="cuda", dtype=torch.bfloat16)
            kp = torch.zeros(4, hk, bs, d, device="cuda", dtype=torch.bfloat16)
            vp = torch.zeros_like(kp)
            kw = dict(rows=M, q_heads=hq, kv_heads=hk, head_dim=d, block_size=bs)
            if use_parts:
                ops.rope_kv_write_partials(parts, n, pos, slot, tab, q, kp, vp, **kw)
            else:
                ops.rope_kv_write(qkv, pos, slot, tab, q, kp, vp, **kw)
            outs.append((q, kp, vp))
        for x, y in zip(*outs):
            assert torch.equal(x, y)
    finally:
        ops.set_gemm_workspace(None)


@pytest.mark.parametrize("h", [256, 4096, 8192])
def test_rmsnorm_block_size_invariant(h):
    """add_rmsnorm picks wide blocks for few rows (decode) and 256-thread blocks
    for many (prefill); its reduction order is defined on chunks, so a row's
    result is bit-identical whichever block size processed it."""
    rows = 400
    x = torch.randn(rows, h, device="cuda") * 3
    add = torch.randn(2, rows, h, device="cuda")
    gain = torch.rand(h, device="cuda") + 0.5
    big_x = x.clone()
    big = torch.empty(rows, h, device="cuda", dtype=torch.bfloat16)
    ops.add_rmsnorm(big_x, gain, 1e-5, big, add=add, n_add=2)  # 400 rows: narrow blocks
    few = 37
    small_x = x[:few].clone()
    small = torch.empty(few, h, device="cuda", dtype=torch.bfloat16)
    ops.add_rmsnorm(small_x, gain, 1e-5, small, add=add[:, :few].contiguous(), n_add=2)  # wide
    assert torch.equal(small_x, big_x[:few])
    assert torch.equal(small, big[:few])


@pytest.mark.parametrize("rows", [297, 1000, 8192])
def test_rmsnorm_lean_kernel_bitexact(rows, monkeypatch):
    """The prefill norm (no residual add, hidden 4096, many rows) runs on the
    register-lean kernel; it must equal the general add+RMSNorm kernel bit for
    bit, and the few-row (decode) norm of the same rows as well."""
    h = 4096
    x = torch.randn(rows, h, device="cuda") * 2
    gain = torch.rand(h, device="cuda") + 0.5
    outs = []
    for lean in ("0", "1"):
        monkeypatch.setenv("SP_NORM_LEAN", lean)
        o = torch.empty(rows, h, device="cuda", dtype=torch.bfloat16)
        ops.add_rmsnorm(x, gain, 1e-5, o)
        outs.append(o)
    assert torch.equal(outs[0], outs[1])
    few = torch.empty(5, h, device="cuda", dtype=torch.bfloat16)
    ops.add_rmsnorm(x[:5].clone(), gain, 1e-5, few)  # wide-block decode path
    assert torch.equal(few, outs[1][:5])


@pytest.mark.parametrize("chunk", [1, 2, 3])
def test_attention_prefill_split_kv(chunk):
    """Split-KV tcgen05 prefill: each work tile's key tiles cut into ranges of
    `chunk`, partials merged by the combine kernel; equals the reference (and
    the unsplit kernel) within bf16 tolerance, deterministic run to run."""
    d, hq, hk, bs = 128, 8, 2, 64
    spans, hist = [300, 129, 1], [0, 200, 700]
    ks, vs, qs = [], [], []
    for m, t0 in zip(spans, hist):
        ks.append(rnd(t0 + m, hk, d, seed=120 + m))
        vs.append(rnd(t0 + m, hk, d, seed=140 + m))
        qs.append(rnd(m, hq, d, seed=160 + m))
    kpool, bt = _paged(ks, hk, d, bs)
    vpool = torch.zeros_like(kpool)
    for i, t in enumerate(vs):
        tab = bt[i].tolist()
        for j in range(t.shape[0]):
            vpool[tab[j // bs], :, j % bs] = t[j]
    q = torch.cat(qs).view(-1, hq * d)
    M = q.shape[0]
    cu = torch.tensor([0] + list(np.cumsum(spans)), dtype=torch.int32, device="cuda")
    first = torch.tensor(hist, dtype=torch.int32, device="cuda")
    kvl = torch.tensor([a + b for a, b in zip(spans, hist)], dtype=torch.int32, device="cuda")
    tt = ops.attn_tile_tokens(hq, hk, d, bs)
    work, split, combine, slot = [], [], [], 0
    for i, m in enumerate(spans):
        for t0 in range(0, m, tt):
            n_kt = -(-(hist[i] + min(t0 + tt, m)) // 128)
            ns = -(-n_kt // chunk)
            if ns == 1:
                work.append((i, t0)); split.append((0, n_kt, -1, 0))
                continue
            for k in range(ns):
                work.append((i, t0)); split.append((k * chunk, min(n_kt, (k + 1) * chunk), slot + k, 0))
            combine.append((i, t0, slot, ns))
            slot += ns
    T = lambda a: torch.tensor(a, dtype=torch.int32, device="cuda").view(-1)
    ws = torch.empty(max(1, slot) * hk * ops.SPLIT_SLOT_BYTES // 4, device="cuda")
    outs = []
    for _ in range(2):
        out = torch.empty(M, hq * d, device="cuda", dtype=torch.bfloat16)
        ops.attention_prefill_split(q, kpool, vpool, bt, cu, first, kvl, out, work=T(work),
                                    split=T(split), n_work=len(work), combine=T(combine),
                                    n_combine=len(combine), n_slots=max(1, slot), q_heads=hq,
                                    kv_heads=hk, head_dim=d, block_size=bs, ws=ws)
        outs.append(out)
    assert torch.equal(outs[0], outs[1])
    lo = 0
    for i, (m, t0) in enumerate(zip(spans, hist)):
        want = _attn_ref(qs[i], ks[i], vs[i], t0)
        assert rel(outs[0][lo:lo + m].view(m, hq, d), want) < 2e-2, i
        lo += m
