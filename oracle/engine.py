"""Oracle multi-device engine (test infrastructure only).

Restates ``/root/reference/pkg/src/shiftsim/parallel_engine.py`` over the
simulated group of ``oracle.fabric``:

* ``choose_mode``      — :134-145 (SP iff new tokens >= threshold; fixed kinds)
* ``step``             — :231-282 (validate, mode, capacity precheck before any
                         write, flatten :307-329, dispatch, commit, record)
* ``_forward_tp``      — :333-398 (replicated activations, column/row shards,
                         embedding all-reduce, 2 all-reduces/layer, logits
                         all-gather)
* ``_forward_sp``      — :454-537 (contiguous token shards, q/k/v seq->head
                         all-to-alls, head->seq all-to-all, full replicas)
* ``_swiftkv_tail_tp`` — :400-450, ``_swiftkv_tail_sp`` — :544-647

In compat mode every result is bit-identical to the reference.  Llama mode
adds GQA (kv heads partitioned like q heads), RoPE and SwiGLU.  The engine also
drives the oracle ``PagedAllocator`` so tests can compare block tables and slot
mappings with the product bit-exactly.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

from .fabric import SimGroup
from .flops import FlopMeter, shard_bounds
from .kvcache import OracleCacheOverflow, OracleKvCache, PagedAllocator
from .model import OracleWeights, Rounder, embed_rows, mlp_block, partition_heads, qkv_heads
from .prims import OracleContractError, attend_cached, matmul, rms_norm


@dataclass
class OracleSeq:
    seq_id: int
    cache: OracleKvCache


class OracleEngine:
    def __init__(self, weights: OracleWeights, world_size: int, kind: str = "fixed_tp",
                 threshold: Optional[int] = None, swiftkv_cut: Optional[int] = None,
                 emulate_bf16: bool = False, threaded: bool = False,
                 block_size: int = 64, num_blocks: int = 4096):
        cfg = weights.config
        self.w = weights
        self.cfg = cfg
        self.p = world_size
        self.group = SimGroup(world_size, threaded=threaded)
        self.kind = kind
        self.threshold = threshold
        self.cut = swiftkv_cut
        self.rnd = Rounder(emulate_bf16)
        self.q_part = partition_heads(cfg.n_heads, world_size)
        self.kv_part = partition_heads(cfg.kv_heads, world_size)
        if cfg.ffn_dim % world_size or cfg.vocab_size % world_size:
            raise OracleContractError("ffn/vocab must split over world_size")
        self.alloc = PagedAllocator(num_blocks, block_size)
        self.mode_log: List[str] = []
        self.records: List[dict] = []
        self.last_slots: Optional[np.ndarray] = None
        self._steps = 0

    # ------------------------------------------------------------ sequences
    def new_sequence(self, seq_id: int, capacity: Optional[int] = None) -> OracleSeq:
        cap = self.cfg.max_seq if capacity is None else capacity
        if cap > self.cfg.max_seq:
            raise OracleContractError("capacity exceeds max_seq")
        return OracleSeq(seq_id, OracleKvCache(self.cfg.n_layers, self.kv_part,
                                               self.cfg.head_dim, cap, self.w.dtype))

    def choose_mode(self, n_tokens: int) -> str:
        if self.kind == "fixed_tp":
            return "tp"
        if self.kind == "fixed_sp":
            return "sp"
        return "sp" if n_tokens >= self.threshold else "tp"

    # ------------------------------------------------------------------ step
    def step(self, items: List[Tuple[OracleSeq, List[int]]], prefill: bool = True,
             mode: Optional[str] = None, span_logits: bool = False):
        if not items or any(len(t) < 1 for _, t in items):
            raise OracleContractError("empty batch or span")
        n_tok = sum(len(t) for _, t in items)
        mode = mode or self.choose_mode(n_tok)
        for s, t in items:  # precheck before any write (:245-251)
            if s.cache.token_count + len(t) > s.cache.capacity:
                raise OracleCacheOverflow(f"seq {s.seq_id} overflows")
        need = sum(self.alloc.blocks_needed(s.seq_id, s.cache.token_count + len(t))
                   for s, t in items)
        if need > self.alloc.free_blocks:
            raise OracleCacheOverflow("paged pool exhausted")
        cut = self.cut if (prefill and self.cut is not None and self.cut < self.cfg.n_layers) else None
        if cut is not None and span_logits:
            raise OracleContractError("span logits unsupported with early exit")
        toks, pos, bounds, hist = [], [], [], []
        lo = 0
        for s, t in items:
            t0 = s.cache.token_count
            for off, tok in enumerate(t):
                if not 0 <= tok < self.cfg.vocab_size:
                    raise OracleContractError("token id outside vocab")
                toks.append(tok)
                pos.append(t0 + off)
            bounds.append((lo, lo + len(t)))
            hist.append(t0)
            lo += len(t)
        fb = dict(tokens=np.asarray(toks, np.int64), positions=np.asarray(pos, np.int64),
                  bounds=bounds, hist=hist)
        slots = []
        for s, t in items:
            self.alloc.reserve(s.seq_id, s.cache.token_count + len(t))
            slots.append(self.alloc.slots(s.seq_id, np.arange(s.cache.token_count,
                                                               s.cache.token_count + len(t))))
        self.last_slots = np.concatenate(slots)
        self.last_block_table = self.alloc.block_table([s.seq_id for s, _ in items])
        self.group.step_id = self._steps
        rec0 = len(self.group.records)
        meters = [FlopMeter() for _ in range(self.p)]
        if mode == "tp":
            logits = self._forward_tp(fb, items, meters, span_logits, cut)
        else:
            logits = self._forward_sp(fb, items, meters, span_logits, cut)
        for s, t in items:
            s.cache.commit(len(t))
        ev = {}
        for kind, _, nb, _, eid in self.group.records[rec0:]:
            if eid not in ev or nb > ev[eid][1]:
                ev[eid] = (kind, nb)
        rec = dict(step_id=self._steps, mode=mode, new_tokens=n_tok, n_requests=len(items),
                   flops_per_device=tuple(m.flops for m in meters),
                   comm=tuple(ev[e] for e in sorted(ev)))
        self.mode_log.append(mode)
        self.records.append(rec)
        self._steps += 1
        return logits, rec

    # -------------------------------------------------------------- helpers
    def _tp_cols(self, r):
        d = self.cfg.head_dim
        (q0, q1), (k0, k1) = self.q_part[r], self.kv_part[r]
        return slice(q0 * d, q1 * d), slice(k0 * d, k1 * d)

    def _fcols(self, r):
        fs = self.cfg.ffn_dim // self.p
        return slice(r * fs, (r + 1) * fs)

    def _attend_items(self, r, layer, q_all, fb, items, meter, out):
        g = self.cfg.group
        for (lo, hi), t0, (s, _) in zip(fb["bounds"], fb["hist"], items):
            for hl in range(q_all.shape[1]):
                kw, vw = s.cache.read_window(r, layer, hl // g)
                out[lo:hi, hl] = attend_cached(q_all[lo:hi, hl], kw, vw, t0, meter)
        return out

    # ------------------------------------------------------------ TP (:333)
    def _forward_tp(self, fb, items, meters, span_logits, cut):
        cfg, w, g, rnd = self.cfg, self.w, self.group, self.rnd
        eps, d, m_total = cfg.norm_eps, cfg.head_dim, fb["tokens"].shape[0]
        vs = cfg.vocab_size // self.p

        def embed_rank(r):  # vocab-parallel rows + all-reduce (:339-348)
            out = np.zeros((m_total, cfg.hidden), dtype=w.dtype)
            sel = (fb["tokens"] >= r * vs) & (fb["tokens"] < (r + 1) * vs)
            if np.any(sel):
                out[sel] = w.embed[r * vs:(r + 1) * vs][fb["tokens"][sel] - r * vs]
            return out

        x = g.all_reduce_sum(g.map_ranks(embed_rank))[0]
        if cfg.pos == "sinusoidal":
            from .prims import sinusoidal_positions
            x = x + sinusoidal_positions(fb["positions"], cfg.hidden, dtype=w.dtype)
        n_full = cfg.n_layers if cut is None else cut
        for li in range(n_full):
            lw = w.layers[li]
            xn = rnd(rms_norm(x, lw["attn_gain"], eps))

            def attn_rank(r, li=li, lw=lw, xn=xn):
                q, k, v = qkv_heads(w, lw, xn, fb["positions"], rnd, self._tp_cols(r), meters[r])
                for (lo, hi), (s, _) in zip(fb["bounds"], items):
                    s.cache.append(r, li, k[lo:hi], v[lo:hi])
                out = np.empty((m_total, q.shape[1], d), dtype=w.dtype)
                self._attend_items(r, li, q, fb, items, meters[r], out)
                qs, _ = self._tp_cols(r)
                return matmul(rnd(out).reshape(m_total, -1), lw["wo"][qs, :], meters[r])

            x = x + g.all_reduce_sum(g.map_ranks(attn_rank))[0]
            xn2 = rnd(rms_norm(x, lw["mlp_gain"], eps))
            x = x + g.all_reduce_sum(g.map_ranks(
                lambda r, lw=lw, xn2=xn2: mlp_block(w, lw, xn2, rnd, self._fcols(r), meters[r])))[0]
        if cut is not None:
            x = self._tail_tp(fb, items, meters, x, cut)
            xf = rnd(rms_norm(x, w.final_gain, eps))
        else:
            rows = (np.arange(m_total) if span_logits
                    else np.asarray([hi - 1 for _, hi in fb["bounds"]]))
            xf = rnd(rms_norm(x[rows], w.final_gain, eps))
        lt = g.all_gather(g.map_ranks(
            lambda r: np.ascontiguousarray(matmul(xf, w.head[:, r * vs:(r + 1) * vs], meters[r]).T)))
        logits = np.ascontiguousarray(lt.T)
        return self._split(logits, fb, items, span_logits and cut is None)

    def _tail_tp(self, fb, items, meters, x, cut):  # :400-450
        cfg, w, g, rnd = self.cfg, self.w, self.group, self.rnd
        eps, d, m_total = cfg.norm_eps, cfg.head_dim, fb["tokens"].shape[0]
        z = rnd(rms_norm(x, w.layers[cut]["attn_gain"], eps))
        for li in range(cut, cfg.n_layers):
            lw = w.layers[li]

            def proj_rank(r, li=li, lw=lw):
                _, ks = self._tp_cols(r)
                k = rnd(matmul(z, lw["wk"][:, ks], meters[r])).reshape(m_total, -1, d)
                v = rnd(matmul(z, lw["wv"][:, ks], meters[r])).reshape(m_total, -1, d)
                if cfg.pos == "rope":
                    from .prims import rope_apply
                    k = rnd(rope_apply(k, fb["positions"], w.rope))
                for (lo, hi), (s, _) in zip(fb["bounds"], items):
                    s.cache.append(r, li, k[lo:hi], v[lo:hi])

            g.map_ranks(proj_rank)
        ends = [hi - 1 for _, hi in fb["bounds"]]
        xt = np.ascontiguousarray(x[ends])
        n_req = len(items)
        wins = [t0 + (hi - lo) for (lo, hi), t0 in zip(fb["bounds"], fb["hist"])]
        tpos = np.asarray([wv - 1 for wv in wins])
        for li in range(cut, cfg.n_layers):
            lw = w.layers[li]
            xn = rnd(rms_norm(xt, lw["attn_gain"], eps))

            def tail_attn(r, li=li, lw=lw, xn=xn):
                qs, _ = self._tp_cols(r)
                q = rnd(matmul(xn, lw["wq"][:, qs], meters[r])).reshape(n_req, -1, d)
                if cfg.pos == "rope":
                    from .prims import rope_apply
                    q = rnd(rope_apply(q, tpos, w.rope))
                out = np.empty((n_req, q.shape[1], d), dtype=w.dtype)
                for i, ((s, _), win) in enumerate(zip(items, wins)):
                    for hl in range(q.shape[1]):
                        kw, vw = s.cache.read_window(r, li, hl // cfg.group)
                        out[i:i + 1, hl] = attend_cached(q[i:i + 1, hl], kw, vw, win - 1, meters[r])
                return matmul(rnd(out).reshape(n_req, -1), lw["wo"][qs, :], meters[r])

            xt = xt + g.all_reduce_sum(g.map_ranks(tail_attn))[0]
            xn2 = rnd(rms_norm(xt, lw["mlp_gain"], eps))
            xt = xt + g.all_reduce_sum(g.map_ranks(
                lambda r, lw=lw, xn2=xn2: mlp_block(w, lw, xn2, rnd, self._fcols(r), meters[r])))[0]
        return xt

    # ------------------------------------------------------------ SP (:454)
    def _head_blocks(self, t, part):
        return [np.ascontiguousarray(t[:, lo:hi, :]) for lo, hi in part]

    def _forward_sp(self, fb, items, meters, span_logits, cut):
        cfg, w, g, rnd, P = self.cfg, self.w, self.group, self.rnd, self.p
        eps, d, m_total = cfg.norm_eps, cfg.head_dim, fb["tokens"].shape[0]
        sb = shard_bounds(m_total, P)
        xs = g.map_ranks(lambda r: embed_rows(w, fb["tokens"][sb[r][0]:sb[r][1]],
                                              fb["positions"][sb[r][0]:sb[r][1]]))
        n_full = cfg.n_layers if cut is None else cut
        for li in range(n_full):
            lw = w.layers[li]

            def qkv_rank(r, lw=lw):
                xn = rnd(rms_norm(xs[r], lw["attn_gain"], eps))
                return qkv_heads(w, lw, xn, fb["positions"][sb[r][0]:sb[r][1]], rnd,
                                 None, meters[r])

            qkv = g.map_ranks(qkv_rank)
            q_rx = g.all_to_all([self._head_blocks(qkv[r][0], self.q_part) for r in range(P)])
            k_rx = g.all_to_all([self._head_blocks(qkv[r][1], self.kv_part) for r in range(P)])
            v_rx = g.all_to_all([self._head_blocks(qkv[r][2], self.kv_part) for r in range(P)])

            def attn_rank(r, li=li):
                q_all = np.concatenate(q_rx[r], axis=0)
                k_all = np.concatenate(k_rx[r], axis=0)
                v_all = np.concatenate(v_rx[r], axis=0)
                for (lo, hi), (s, _) in zip(fb["bounds"], items):
                    s.cache.append(r, li, k_all[lo:hi], v_all[lo:hi])
                out = np.empty((m_total, q_all.shape[1], d), dtype=w.dtype)
                return rnd(self._attend_items(r, li, q_all, fb, items, meters[r], out))

            att = g.map_ranks(attn_rank)
            back = g.all_to_all([[np.ascontiguousarray(att[r][lo:hi]) for lo, hi in sb]
                                 for r in range(P)])

            def post_rank(r, lw=lw):
                rows = xs[r].shape[0]
                a = np.concatenate(back[r], axis=1).reshape(rows, cfg.hidden)
                xn_ = xs[r] + matmul(a, lw["wo"], meters[r])
                xn2 = rnd(rms_norm(xn_, lw["mlp_gain"], eps))
                return xn_ + mlp_block(w, lw, xn2, rnd, None, meters[r])

            xs = g.map_ranks(post_rank)
        if cut is not None:
            return self._tail_sp(fb, items, meters, xs, sb, cut)
        ends = [hi - 1 for _, hi in fb["bounds"]]

        def logits_rank(r):
            lo, hi = sb[r]
            rows = xs[r] if span_logits else xs[r][[e - lo for e in ends if lo <= e < hi]]
            return matmul(rnd(rms_norm(rows, w.final_gain, eps)), w.head, meters[r])

        logits = g.all_gather(g.map_ranks(logits_rank))
        return self._split(logits, fb, items, span_logits)

    def _tail_sp(self, fb, items, meters, xs, sb, cut):  # :544-647
        cfg, w, g, rnd, P = self.cfg, self.w, self.group, self.rnd, self.p
        eps, d = cfg.norm_eps, cfg.head_dim
        gain = w.layers[cut]["attn_gain"]
        zs = g.map_ranks(lambda r: rnd(rms_norm(xs[r], gain, eps)))
        for li in range(cut, cfg.n_layers):
            lw = w.layers[li]

            def kv_rank(r, lw=lw):
                rows = zs[r].shape[0]
                k = rnd(matmul(zs[r], lw["wk"], meters[r])).reshape(rows, cfg.kv_heads, d)
                v = rnd(matmul(zs[r], lw["wv"], meters[r])).reshape(rows, cfg.kv_heads, d)
                if cfg.pos == "rope":
                    from .prims import rope_apply
                    k = rnd(rope_apply(k, fb["positions"][sb[r][0]:sb[r][1]], w.rope))
                return k, v

            kv = g.map_ranks(kv_rank)
            k_rx = g.all_to_all([self._head_blocks(kv[r][0], self.kv_part) for r in range(P)])
            v_rx = g.all_to_all([self._head_blocks(kv[r][1], self.kv_part) for r in range(P)])

            def append_rank(r, li=li):
                k_all = np.concatenate(k_rx[r], axis=0)
                v_all = np.concatenate(v_rx[r], axis=0)
                for (lo, hi), (s, _) in zip(fb["bounds"], items):
                    s.cache.append(r, li, k_all[lo:hi], v_all[lo:hi])

            g.map_ranks(append_rank)
        ends = [hi - 1 for _, hi in fb["bounds"]]
        wins = [t0 + (hi - lo) for (lo, hi), t0 in zip(fb["bounds"], fb["hist"])]
        owner_rows = [[e - lo for e in ends if lo <= e < hi] for lo, hi in sb]
        owner_of_end = [next(r for r, (lo, hi) in enumerate(sb) if lo <= e < hi) for e in ends]
        tails = [np.ascontiguousarray(xs[r][owner_rows[r]]) for r in range(P)]
        tpos = [np.asarray([wins[i] - 1 for i, e in enumerate(ends) if sb[r][0] <= e < sb[r][1]],
                           dtype=np.int64) for r in range(P)]
        n_req = len(items)
        seen, tail_sl = 0, []
        for r in range(P):
            tail_sl.append((seen, seen + len(owner_rows[r])))
            seen += len(owner_rows[r])
        for li in range(cut, cfg.n_layers):
            lw = w.layers[li]

            def tail_q(r, lw=lw):
                xn = rnd(rms_norm(tails[r], lw["attn_gain"], eps))
                q = rnd(matmul(xn, lw["wq"], meters[r])).reshape(xn.shape[0], cfg.n_heads, d)
                if cfg.pos == "rope":
                    from .prims import rope_apply
                    q = rnd(rope_apply(q, tpos[r], w.rope))
                return q

            qs = g.map_ranks(tail_q)
            q_rx = g.all_to_all([self._head_blocks(qs[r], self.q_part) for r in range(P)])

            def tail_attn(r, li=li):
                q_all = np.concatenate(q_rx[r], axis=0)
                out = np.empty((n_req, q_all.shape[1], d), dtype=w.dtype)
                for i, ((s, _), win) in enumerate(zip(items, wins)):
                    for hl in range(q_all.shape[1]):
                        kw, vw = s.cache.read_window(r, li, hl // cfg.group)
                        out[i:i + 1, hl] = attend_cached(q_all[i:i + 1, hl], kw, vw, win - 1,
                                                         meters[r])
                return rnd(out)

            att = g.map_ranks(tail_attn)
            back = g.all_to_all([[np.ascontiguousarray(att[r][lo:hi]) for lo, hi in tail_sl]
                                 for r in range(P)])

            def tail_post(r, lw=lw):
                rows = tails[r].shape[0]
                a = np.concatenate(back[r], axis=1).reshape(rows, cfg.hidden)
                xn_ = tails[r] + matmul(a, lw["wo"], meters[r])
                xn2 = rnd(rms_norm(xn_, lw["mlp_gain"], eps))
                return xn_ + mlp_block(w, lw, xn2, rnd, None, meters[r])

            tails = g.map_ranks(tail_post)
        logits = g.all_gather(g.map_ranks(
            lambda r: matmul(rnd(rms_norm(tails[r], w.final_gain, eps)), w.head, meters[r])))
        order = np.argsort(np.asarray(owner_of_end), kind="stable")
        inv = np.empty_like(order)
        inv[order] = np.arange(n_req)
        logits = logits[inv]
        return [logits[i] for i in range(n_req)]

    @staticmethod
    def _split(logits, fb, items, span):
        if span:
            return [np.ascontiguousarray(logits[lo:hi]) for lo, hi in fb["bounds"]]
        return [logits[i] for i in range(len(items))]
