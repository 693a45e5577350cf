"""Shift-Parallel engine on B200: per-pass SP/TP over one head-sharded paged KV pool.

Drop-in for the reference engine API (/root/reference/pkg/src/shiftsim/
parallel_engine.py): ``Engine(weights, group, policy, swiftkv)`` (:194-216),
``new_sequence`` (:220-227), ``step(batch, mode=None, span_logits=False) ->
(logits per item, StepRecord)`` (:231-282), ``choose_mode`` (:134-145) and
the ``Batch`` / ``BatchItem`` / ``Sequence`` / ``ShiftPolicy`` types (:63-127).

What runs where (all arithmetic is libshiftpar.so, sm_100a):

TP pass (:333-398)  x replicated [M, h] f32; per rank r: QKV GEMM on the rank's
    rows of the fused weight -> RoPE + paged KV write -> attention over owned
    heads -> O GEMM on the rank's K window -> NCCL all-reduce -> fused
    add+RMSNorm -> SwiGLU GEMM on owned ffn rows -> down GEMM -> all-reduce.
    The embedding uses the resident replica (no all-reduce, containment
    model.py:257-281); at P = 1 the partials add straight into x in the GEMM
    epilogue.
SP pass (:454-537)  tokens of the flattened batch split contiguously; per rank:
    RMSNorm -> full-replica QKV GEMM whose epilogue writes each peer's head
    block into a contiguous send buffer -> ONE all-to-all (q|k|v fused) ->
    the same RoPE/KV-write and attention kernels as TP (the received layout is
    identical to a TP rank's QKV output) -> all-to-all back -> O GEMM reading
    the per-peer receive layout through a 3-D TMA map, adding into x ->
    RMSNorm -> SwiGLU -> down GEMM adding into x.
Both modes write identical K/V rows to the same per-device blocks, so the
mode can change every pass with zero KV movement (kv_cache.py:1-15).
"""

from __future__ import annotations

import enum
import os
import time
import warnings
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence as Seq, Tuple

import numpy as np
import torch

from . import ops
from .config import ModelConfig
from .errors import CacheOverflow, ConfigError, ContractViolation
from .fabric import CommRecord, DeviceGroup, LoopbackGroup
from .flops import FlopMeter, PassShape, flop_count, shard_bounds, shard_rows
from .kv_cache import KvCache, KvPool
from .peer import PeerLinks, fused_a2a_enabled, two_shot_min_rows
from .weights import ModelWeights


class ParallelMode(enum.Enum):
    TP = "tp"
    SP = "sp"


class BatchKind(enum.Enum):
    PREFILL = "prefill"
    DECODE = "decode"


@dataclass
class Sequence:
    """Engine-side identity of one request: an id plus its KV cache (:63-68)."""

    seq_id: int
    cache: KvCache


@dataclass
class BatchItem:
    seq: Sequence
    tokens: List[int]


@dataclass
class Batch:
    kind: BatchKind
    items: List[BatchItem]
    speculative: bool = False

    @property
    def total_new_tokens(self) -> int:
        return sum(len(it.tokens) for it in self.items)

    def validate(self) -> None:
        """parallel_engine.py:88-99."""
        if not self.items:
            raise ContractViolation("batch must contain at least one item")
        for it in self.items:
            if len(it.tokens) < 1:
                raise ContractViolation("batch item with empty span")
        if self.kind is BatchKind.DECODE and not self.speculative:
            if any(len(it.tokens) != 1 for it in self.items):
                raise ContractViolation("decode batches carry exactly 1 new token per request")
        if len({id(it.seq.cache) for it in self.items}) != len(self.items):
            raise ContractViolation("a sequence may appear at most once per batch")


@dataclass(frozen=True)
class ShiftPolicy:
    """SP at or above ``token_threshold`` new tokens, TP below (:102-127)."""

    token_threshold: Optional[int] = None
    kind: str = "shift"

    def validate(self) -> "ShiftPolicy":
        if self.kind not in ("fixed_tp", "fixed_sp", "shift"):
            raise ConfigError(f"unknown policy kind {self.kind!r}")
        if self.kind == "shift" and (self.token_threshold is None or self.token_threshold < 1):
            raise ConfigError("shift policy needs token_threshold >= 1")
        return self

    @staticmethod
    def fixed_tp() -> "ShiftPolicy":
        return ShiftPolicy(kind="fixed_tp")

    @staticmethod
    def fixed_sp() -> "ShiftPolicy":
        return ShiftPolicy(kind="fixed_sp")


def default_token_threshold(world_size: int, config=None) -> int:
    """Without a model config: the reference default 4·P (:130-131).  With
    one: the B200 crossover of ``shift_cost.crossover`` — the smallest
    batched-token count from which an SP pass is modelled no slower than a TP
    pass on this geometry (calibrated by tools/tau_sweep.py)."""
    if world_size < 1:
        raise ConfigError("world_size must be >= 1")
    if config is None:
        return 4 * world_size
    from .shift_cost import crossover
    return max(1, crossover(config, world_size))


def choose_mode(policy: ShiftPolicy, batch: Batch) -> ParallelMode:
    policy.validate()
    if policy.kind == "fixed_tp":
        return ParallelMode.TP
    if policy.kind == "fixed_sp":
        return ParallelMode.SP
    return ParallelMode.SP if batch.total_new_tokens >= policy.token_threshold else ParallelMode.TP


@dataclass(frozen=True)
class SwiftKvConfig:
    """Early-exit prefill (reference swiftkv.py:26-46)."""

    enabled: bool = False
    cut_layer: Optional[int] = None

    def resolve_cut(self, n_layers: int) -> int:
        if not self.enabled:
            return n_layers
        cut = n_layers // 2 if self.cut_layer is None else self.cut_layer
        if not 1 <= cut <= n_layers:
            raise ConfigError(f"cut_layer {cut} outside [1, {n_layers}]")
        return cut


@dataclass(frozen=True)
class CommEvent:
    kind: str
    bytes: float


@dataclass(frozen=True)
class StepRecord:
    """parallel_engine.py:156-176 (+ host wall time of the enqueue)."""

    step_id: int
    mode: ParallelMode
    kind: BatchKind
    new_tokens: int
    n_requests: int
    flops_per_device: Tuple[int, ...]
    comm: Tuple[CommEvent, ...]
    host_ms: float = 0.0

    @property
    def flops_total(self) -> int:
        return sum(self.flops_per_device)

    @property
    def flops_max_device(self) -> int:
        return max(self.flops_per_device)

    @property
    def comm_bytes(self) -> float:
        return sum(e.bytes for e in self.comm)


def partition_heads(n_heads: int, world_size: int) -> Tuple[Tuple[int, int], ...]:
    """Device d owns heads [d H/P, (d+1) H/P) (model.py:186-193)."""
    if world_size < 1 or n_heads % world_size:
        raise ConfigError(f"n_heads {n_heads} not divisible by world_size {world_size}")
    w = n_heads // world_size
    return tuple((r * w, (r + 1) * w) for r in range(world_size))


class _Meta:
    """Per-pass device metadata, uploaded with ONE host->device copy."""

    pass


class _GraphEntry:
    """A captured decode pass: static metadata buffer, graph, static outputs."""

    def __init__(self):
        self.dev: Optional[torch.Tensor] = None
        self.graph = None
        self.outputs: List[torch.Tensor] = []
        self.charges: list = []
        self.kernels = 0
        self.failed = False  # capture raised: this key stays eager
        self.seen = 0  # eager passes run with this key so far
        self.replays = 0


class _RopedQ:
    """Marker: the QKV epilogue already rotated q (here) and wrote K/V."""
    __slots__ = ("q",)

    def __init__(self, q: torch.Tensor):
        self.q = q


def attention_split_plan(wl, spans, hist, tt: int, hk: int, sms: int, max_slots: int):
    """Split-KV plan for a prefill pass whose work tiles x kv heads do not
    fill the SMs (one long request under SP=8: 128 tiles x 1 kv head with
    causal costs 1..64 key tiles, so the longest tile alone set the kernel
    time).  Tiles longer than total/(SMs/kv heads) key tiles are cut into
    nearly equal key ranges, merged later by the combine kernel; entries are
    ordered longest first so the block scheduler packs them into ~one wave.

    wl: (item, t0, key0) work tiles; returns (work [n,2], split [n,4] =
    (first key tile, end key tile, slot | -1, 0), combine [c,4] = (item, t0,
    first slot, n slots), n_slots) or None when nothing needs splitting."""
    if len(wl) * hk >= sms:
        return None
    kt = 128  # key tile of the tcgen05 kernel
    tiles = []
    for i, t0, _ in wl:
        q_end = min(t0 + tt, spans[i])
        tiles.append((i, t0, -(-(hist[i] + q_end) // kt)))
    total = sum(c for _, _, c in tiles)
    # ~1.5 waves: pieces of at most total/(1.5 SMs) key tiles, longest first
    # (the block scheduler then packs them LPT-style).  SP=8 8K attention
    # (tools/attn_sp_shapes.py): 1 wave 750, 1.25 770, 1.5 800, 1.75 774,
    # 2 673 TFLOP/s — smaller pieces pack better until the per-CTA prologue,
    # Q reload and partial traffic dominate.  SP_ATTN_SPLIT_WAVES overrides.
    waves = float(os.environ.get("SP_ATTN_SPLIT_WAVES", "1.5"))
    chunk = max(2, -(-total // max(1, int(waves * sms) // hk)))
    entries, combine, slot = [], [], 0
    for i, t0, c in tiles:
        ns = -(-c // chunk)
        if ns <= 1:
            entries.append((c, i, t0, 0, c, -1))
            continue
        bounds = [c * k // ns for k in range(ns + 1)]
        for k in range(ns):
            entries.append((bounds[k + 1] - bounds[k], i, t0, bounds[k], bounds[k + 1], slot + k))
        combine.append((i, t0, slot, ns))
        slot += ns
    if slot == 0 or slot > max_slots:
        return None  # nothing long enough to split, or no workspace for it
    entries.sort(key=lambda e: -e[0])
    work = np.asarray([(e[1], e[2]) for e in entries], dtype=np.int32).reshape(-1, 2)
    split = np.asarray([(e[3], e[4], e[5], 0) for e in entries], dtype=np.int32).reshape(-1, 4)
    comb = np.asarray(combine, dtype=np.int32).reshape(-1, 4)
    return work, split, comb, slot


class Engine:
    def __init__(self, weights: ModelWeights, group: DeviceGroup, policy: ShiftPolicy,
                 swiftkv: Optional[SwiftKvConfig] = None, *, num_blocks: Optional[int] = None,
                 block_size: int = 64, cuda_graphs: bool = True, max_pass_tokens: int = 16384,
                 sp_degree: Optional[int] = None):
        cfg = weights.config
        self.weights = weights
        self.config: ModelConfig = cfg
        self.group = group
        self.policy = policy.validate()
        self.swiftkv = swiftkv if swiftkv is not None else SwiftKvConfig()
        self.world_size = group.world_size
        if weights.world_size != self.world_size:
            raise ConfigError("weights were laid out for a different world size")
        cfg.check_world(self.world_size)
        # SP mode runs SP(s) x TP(P/s) when sp_degree = s < P (the paper's
        # "SP x TP = P" base config); s = P is the reference's pure SP
        self.sp_degree = self.world_size if sp_degree is None else sp_degree
        if self.sp_degree < 1 or self.world_size % self.sp_degree:
            raise ConfigError("sp_degree must divide the world size")
        if self.sp_degree < self.world_size:
            t = self.world_size // self.sp_degree
            if cfg.ffn_dim // t % 128 or cfg.kv_heads % self.world_size:
                raise ConfigError("SP x TP needs 128-row SwiGLU shards and P | kv_heads")
            s = self.sp_degree
            group.make_subgroups([[g * s + i for g in range(t)] for i in range(s)])
        self.partition = partition_heads(cfg.n_heads, self.world_size)
        self.kv_partition = partition_heads(cfg.kv_heads, self.world_size)
        self.device = weights.embed.device
        ops.device_check()
        # split-K workspace for decode-size GEMMs: one per device, allocated once and
        # never freed (captured decode graphs hold its address)
        ops.ensure_gemm_workspace(self.device)
        if isinstance(group, LoopbackGroup):
            group._add = ops.add_f32
        if self.swiftkv.enabled:
            cut = self.swiftkv.resolve_cut(cfg.n_layers)
            if cut < cfg.n_layers:
                weights.ensure_swiftkv(cut)
        if num_blocks is None:
            num_blocks = max(16, 4 * -(-cfg.max_seq // block_size))
        self.pool = KvPool(cfg.n_layers, self.kv_partition, cfg.head_dim, num_blocks, block_size,
                           group.local_ranks, self.device)
        # fused SP all-to-all over peer memory (passes up to max_pass_tokens tokens)
        self._peer: Optional[PeerLinks] = None
        if fused_a2a_enabled(group):
            hqw = cfg.n_heads // self.world_size * cfg.head_dim
            try:
                self._peer = PeerLinks(group, max_pass_tokens, weights.qkv_width, hqw, cfg.hidden,
                                       self.device)
            except Exception as e:  # e.g. no IPC/P2P between the ranks' GPUs
                warnings.warn(f"peer-memory exchanges unavailable ({e}); using collectives")
                self._peer = None
        self.mode_log: List[ParallelMode] = []
        self.step_records: List[StepRecord] = []
        self._step_counter = 0
        self._next_key = 0
        self._pinned: List[torch.Tensor] = []
        self._pin_events: List[Optional[torch.cuda.Event]] = []
        self._pin_idx = 0
        # attention split-KV workspace, allocated once (graph replays need static buffers)
        self._ws = torch.empty(16 << 20, dtype=torch.float32, device=self.device)
        self._sms = torch.cuda.get_device_properties(self.device).multi_processor_count
        self.cuda_graphs = cuda_graphs
        self._fuse_splitk = os.environ.get("SP_FUSE_SPLITK", "1") != "0"
        self._fuse_rope = os.environ.get("SP_FUSE_ROPE", "1") != "0"
        self._fuse_attn_rope = os.environ.get("SP_FUSE_ATTN_ROPE", "1") != "0"
        # fused decode layer (one persistent kernel per layer, P = 1 TP decode):
        # opt-in (SP_DECODE_FUSED=1) — measured slower than the kernel chain
        # ("fused decode layer")
        self._decode_fused = os.environ.get("SP_DECODE_FUSED", "0") == "1"
        self._dl_sync = torch.zeros(2, dtype=torch.int32, device=self.device)
        self._dl_ws: Dict[int, int] = {}
        self._graph_after = max(1, int(os.environ.get("SP_GRAPH_AFTER", "2")))
        self._graphs: Dict[tuple, _GraphEntry] = {}
        self._graph_pool = torch.cuda.graph_pool_handle() if cuda_graphs else None
        self._capturing = False

    # ---------------------------------------------------------- sequences
    def new_sequence(self, seq_id: int, capacity: Optional[int] = None) -> Sequence:
        cap = self.config.max_seq if capacity is None else capacity
        if cap > self.config.max_seq:
            raise ContractViolation(f"capacity {cap} exceeds max_seq {self.config.max_seq}")
        key = self._next_key
        self._next_key += 1
        return Sequence(seq_id=seq_id, cache=KvCache(self.pool, key, cap))

    def release(self, seq: Sequence) -> None:
        """Return a finished sequence's blocks to the pool (paged extension)."""
        self.pool.alloc.release(seq.cache.key)
        seq.cache.released = True

    # --------------------------------------------------------------- step
    def step(self, batch: Batch, mode: Optional[ParallelMode] = None,
             span_logits: bool = False) -> Tuple[List[torch.Tensor], StepRecord]:
        t_host = time.perf_counter()
        batch.validate()
        if mode is None:
            mode = choose_mode(self.policy, batch)
        for it in batch.items:
            c = it.seq.cache
            if c.released:
                raise ContractViolation(f"sequence {it.seq.seq_id} was released")
            if c.token_count + len(it.tokens) > c.capacity:
                raise CacheOverflow(f"sequence {it.seq.seq_id}: {c.token_count + len(it.tokens)} "
                                    f"tokens exceed capacity {c.capacity}")
        cut_full = self.swiftkv.resolve_cut(self.config.n_layers)
        use_swiftkv = (self.swiftkv.enabled and batch.kind is BatchKind.PREFILL
                       and cut_full < self.config.n_layers)
        if use_swiftkv and span_logits:
            raise ContractViolation("span logits unsupported with early-exit prefill")
        v = self.config.vocab_size
        for it in batch.items:
            for tok in it.tokens:
                if not 0 <= tok < v:
                    raise ContractViolation(f"token id {tok} outside vocab [0, {v})")
        alloc = self.pool.alloc
        need = sum(alloc.blocks_needed(it.seq.cache.key, it.seq.cache.token_count + len(it.tokens))
                   for it in batch.items)
        if need > alloc.free_blocks:
            raise CacheOverflow(f"paged KV pool exhausted: {need} blocks needed, "
                                f"{alloc.free_blocks} free")
        for it in batch.items:
            alloc.reserve(it.seq.cache.key, it.seq.cache.token_count + len(it.tokens))
        cut = cut_full if use_swiftkv else None
        graph_key = None
        if (self.cuda_graphs and cut is None and not span_logits
                and not getattr(self.group, "_stage", False)  # host-staged collectives
                and not (mode is ParallelMode.SP and self.sp_degree < self.world_size)
                and all(len(it.tokens) == 1 for it in batch.items)):
            graph_key = (mode, len(batch.items), self._bt_width_cap(batch),
                         self._kv_bucket(batch))
        shape = self.pass_shape(batch, span_logits) if graph_key else None
        meta = self._metadata(batch, mode, span_logits, cut, graph_key=graph_key)
        self.group.begin_step(self._step_counter)
        rec_start = len(self.group.records)
        meters = [FlopMeter() for _ in range(self.world_size)]
        entry = self._graphs.get(graph_key) if graph_key else None
        if entry is not None and entry.graph is not None:
            # replay: host bookkeeping + ledger exactly as the eager pass would record
            for layer in range(self.config.n_layers):
                self._stage_all(layer, batch)
            for kind, per_dev in entry.charges:
                self.group.charge(kind, per_dev)
            entry.graph.replay()
            entry.replays += 1
            ops.add_graph_launches(entry.kernels)
            logits = [t.clone() for t in entry.outputs]
            flops = flop_count(shape, mode, self.config, self.world_size)
            for m, f in zip(meters, flops):
                m.flops = f
        else:
            fwd = self._forward_tp if mode is ParallelMode.TP else self._forward_sp
            logits = fwd(meta, batch, meters, span_logits, cut)
            if graph_key is not None and not self._graphs[graph_key].failed:
                # capture once a key recurs: serving sees many one-off batch sizes
                # whose capture (a second host-side forward + sync) would cost more
                # than the eager pass it replaces (SP_GRAPH_AFTER, default 2)
                e = self._graphs[graph_key]
                e.seen += 1
                if e.seen >= self._graph_after:
                    self._capture(graph_key, meta, batch, fwd)
        for it in batch.items:
            it.seq.cache.commit(len(it.tokens))
        record = StepRecord(step_id=self._step_counter, mode=mode, kind=batch.kind,
                            new_tokens=meta.M, n_requests=meta.n,
                            flops_per_device=tuple(m.flops for m in meters),
                            comm=self._comm_events(self.group.records[rec_start:]),
                            host_ms=(time.perf_counter() - t_host) * 1e3)
        self.mode_log.append(mode)
        self.step_records.append(record)
        self._step_counter += 1
        return logits, record

    def _bt_width_cap(self, batch: Batch) -> int:
        """Block-table width for graph keys: covers every item's capacity,
        rounded up to a power of two so the key is stable while sequences grow."""
        bs = self.pool.block_size
        need = max(-(-it.seq.cache.capacity // bs) for it in batch.items)
        w = 1
        while w < need:
            w *= 2
        return w

    def _kv_bucket(self, batch: Batch) -> int:
        """Power-of-two bucket of the longest key window in pages: part of the
        graph key, so the decode attention's KV split count (chosen from the
        host max_kv_len at capture and frozen into the graph) follows the
        context as sequences grow."""
        bs = self.pool.block_size
        pages = max(-(-(it.seq.cache.token_count + len(it.tokens)) // bs) for it in batch.items)
        w = 1
        while w < pages:
            w *= 2
        return w

    def _capture(self, key, meta: "_Meta", batch: Batch, fwd) -> None:
        """Record the decode pass just executed eagerly as a CUDA graph (same
        static metadata buffer); later passes with the same key replay it."""
        entry = self._graphs[key]
        n_rec = len(self.group.records)
        k0 = ops.kernel_launches()
        graph = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        self._capturing = True
        try:
            with torch.cuda.graph(graph, pool=self._graph_pool):
                outs = fwd(meta, batch, [FlopMeter() for _ in range(self.world_size)], False, None)
        except RuntimeError as e:
            # e.g. a collective backend that cannot be captured: run this key eagerly
            del self.group.records[n_rec:]
            entry.failed = True
            warnings.warn(f"CUDA-graph capture of decode pass {key} failed ({e}); running eagerly")
            return
        finally:
            self._capturing = False
        entry.kernels = ops.kernel_launches() - k0
        events = {}
        for r in self.group.records[n_rec:]:
            events.setdefault(r.event_id, [r.kind, [0.0] * self.world_size])[1][r.device] = r.bytes
        entry.charges = [tuple(events[e]) for e in sorted(events)]
        del self.group.records[n_rec:]
        entry.outputs = outs
        entry.graph = graph

    def forward_tp(self, batch: Batch, span_logits: bool = False):
        return self.step(batch, mode=ParallelMode.TP, span_logits=span_logits)

    def forward_sp(self, batch: Batch, span_logits: bool = False):
        return self.step(batch, mode=ParallelMode.SP, span_logits=span_logits)

    def pass_shape(self, batch: Batch, span_logits: bool = False) -> PassShape:
        return PassShape(spans=tuple(len(it.tokens) for it in batch.items),
                         history=tuple(it.seq.cache.token_count for it in batch.items),
                         span_logits=span_logits)

    @staticmethod
    def _comm_events(records: Seq[CommRecord]) -> Tuple[CommEvent, ...]:
        by = {}
        for r in records:
            cur = by.get(r.event_id)
            if cur is None or r.bytes > cur[1]:
                by[r.event_id] = (r.kind, r.bytes)
        return tuple(CommEvent(k, b) for k, b in (by[e] for e in sorted(by)))

    # ----------------------------------------------------------- metadata
    def _pinned_buffer(self, n: int) -> torch.Tensor:
        if not self._pinned:
            self._pinned = [torch.empty(0, dtype=torch.int32).pin_memory() for _ in range(2)]
            self._pin_events = [None, None]
        i = self._pin_idx
        self._pin_idx ^= 1
        ev = self._pin_events[i]
        if ev is not None:
            ev.synchronize()  # the previous copy out of this buffer has finished
        if self._pinned[i].numel() < n:
            self._pinned[i] = torch.empty(max(n, 2 * self._pinned[i].numel()),
                                          dtype=torch.int32).pin_memory()
        return self._pinned[i], i

    def _metadata(self, batch: Batch, mode: ParallelMode, span_logits: bool,
                  cut: Optional[int], graph_key=None) -> _Meta:
        """Flatten the batch (parallel_engine.py:307-329) and build every index
        array the kernels need; one pinned H2D copy."""
        cfg = self.config
        P = self.world_size
        bs = self.pool.block_size
        alloc = self.pool.alloc
        items = batch.items
        n = len(items)
        spans = [len(it.tokens) for it in items]
        hist = [it.seq.cache.token_count for it in items]
        M = sum(spans)
        toks = np.concatenate([np.asarray(it.tokens, dtype=np.int32) for it in items])
        pos = np.concatenate([np.arange(h0, h0 + m, dtype=np.int32) for h0, m in zip(hist, spans)])
        slots = np.concatenate([alloc.slots(it.seq.cache.key, h0, m)
                                for it, h0, m in zip(items, hist, spans)])
        cu = np.zeros(n + 1, dtype=np.int32)
        cu[1:] = np.cumsum(spans)
        first = np.asarray(hist, dtype=np.int32)
        kvlen = first + np.asarray(spans, dtype=np.int32)
        width = max(len(alloc.tables[it.seq.cache.key]) for it in items)
        if graph_key is not None:
            width = graph_key[2]
        bt = np.zeros((n, width), dtype=np.int32)
        for i, it in enumerate(items):
            tab = alloc.tables[it.seq.cache.key]
            bt[i, :len(tab)] = tab
        ends = (cu[1:] - 1).astype(np.int32)
        decode_like = all(m == 1 for m in spans)
        split = combine = None
        n_slots = 0
        if decode_like:
            work = np.zeros((0, 2), dtype=np.int32)
        else:
            tt = ops.attn_tile_tokens(cfg.n_heads // P, cfg.kv_heads // P, cfg.head_dim, bs)
            wl = [(i, t0, hist[i] + t0) for i in range(n) for t0 in range(0, spans[i], tt)]
            wl.sort(key=lambda w: -w[2])  # heaviest causal tiles first
            work = np.asarray([(i, t0) for i, t0, _ in wl], dtype=np.int32).reshape(-1, 2)
            plan = self._split_plan(wl, spans, hist, tt)
            if plan is not None:
                work, split, combine, n_slots = plan
        # SP token shards: P of them, or s under SP(s) x TP(P/s)
        n_shards = self.sp_degree if mode is ParallelMode.SP else P
        bounds = shard_bounds(M, n_shards)
        # SP: per-shard local indices of the rows whose logits are returned
        sp_rows = []
        for lo, hi in bounds:
            if span_logits:
                sp_rows.append(np.arange(0, hi - lo, dtype=np.int32))
            else:
                sp_rows.append(np.asarray([e - lo for e in ends if lo <= e < hi], dtype=np.int32))
        tail_pos = (kvlen - 1).astype(np.int32)
        tail_slot = np.full(n, -1, dtype=np.int32)
        tail_cu = np.arange(n + 1, dtype=np.int32)
        parts = dict(toks=toks, pos=pos, slots=slots, cu=cu, first=first, kvlen=kvlen,
                     bt=bt.reshape(-1), ends=ends, work=work.reshape(-1),
                     tail_pos=tail_pos, tail_slot=tail_slot, tail_cu=tail_cu)
        if split is not None:
            parts["work_split"] = split.reshape(-1)
            parts["work_combine"] = combine.reshape(-1)
        for r in range(n_shards):
            parts[f"sprows{r}"] = sp_rows[r]
        # every array starts on a 16-byte boundary (the kernels read int2 pairs)
        total = sum(-(-a.size // 4) * 4 for a in parts.values())
        host, idx = self._pinned_buffer(total)
        if graph_key is not None:
            entry = self._graphs.setdefault(graph_key, _GraphEntry())
            if entry.dev is None:
                entry.dev = torch.empty(max(total, 1), dtype=torch.int32, device=self.device)
            dev = entry.dev
        else:
            dev = torch.empty(max(total, 1), dtype=torch.int32, device=self.device)
        views = {}
        off = 0
        hv = host.numpy()
        for k, a in parts.items():
            hv[off:off + a.size] = a
            views[k] = (off, a.size)
            off += -(-a.size // 4) * 4
        dev[:total].copy_(host[:total], non_blocking=True)
        self.last_h2d_bytes = total * 4
        ev = torch.cuda.Event()
        ev.record()
        self._pin_events[idx] = ev
        meta = _Meta()
        for k, (o, s) in views.items():
            setattr(meta, k, dev[o:o + s])
        meta.bt = meta.bt.view(n, width)
        meta.work_pairs = meta.work
        meta.n_work = work.shape[0]
        meta.n_combine = None if split is None else combine.shape[0]
        meta.n_slots = n_slots
        meta.M, meta.n, meta.spans, meta.hist = M, n, spans, hist
        meta.ends_host = ends
        meta.bounds = bounds
        meta.rows = [hi - lo for lo, hi in bounds]
        meta.sp_counts = [a.size for a in sp_rows]
        meta.max_q = max(spans)
        meta.max_kv = int(kvlen.max())
        meta.windows = kvlen.tolist()
        meta.decode_like = decode_like
        self.last_slots = slots
        self.last_block_table = bt
        return meta

    def _split_plan(self, wl, spans, hist, tt):
        """Split-KV plan for the tcgen05 prefill (see attention_split_plan);
        None when not needed, not applicable or disabled (SP_ATTN_SPLIT=0)."""
        cfg = self.config
        hk = cfg.kv_heads // self.world_size
        if (os.environ.get("SP_ATTN_SPLIT") == "0" or cfg.head_dim != 128
                or self.pool.block_size % 64):
            return None
        max_slots = self._ws.numel() * self._ws.element_size() // (hk * ops.SPLIT_SLOT_BYTES)
        return attention_split_plan(wl, spans, hist, tt, hk, self._sms, max_slots)

    def _workspace(self, n_items: int, q_heads: int, max_kv: int) -> Optional[torch.Tensor]:
        # fixed 64 MB: the kernel falls back to one split when a pass would need more
        return self._ws

    # ------------------------------------------------------- shared pieces
    def _attend(self, r: int, layer: int, q: Optional[torch.Tensor], out: torch.Tensor,
                meta: _Meta, meter: FlopMeter, *, tails: bool = False, parts=None) -> None:
        """Attention of one rank's heads (attend_cached loops, parallel_engine.py
        :362-368 / :494-500).  ``parts`` = (QKV K-split partials, count) of a
        decode pass: Q and the new token's RoPE + KV write are computed inside
        the decode attention kernel (sp_attention_decode_qkv) instead of a
        separate rope_kv_write_partials launch — bit-identical."""
        cfg = self.config
        P = self.world_size
        hq, hk, d = cfg.n_heads // P, cfg.kv_heads // P, cfg.head_dim
        if tails:
            n_rows, cu, first = meta.n, meta.tail_cu, meta.tail_pos
            decode_like = True
            spans = [1] * meta.n
        else:
            n_rows, cu, first = meta.M, meta.cu, meta.first
            decode_like = meta.decode_like
            spans = meta.spans
        ws = self._workspace(meta.n, hq, meta.max_kv) if decode_like else None
        # algorithmic work: causal half of q·Kᵀ + P·V, and K/V bytes streamed
        hist = [w - m for m, w in zip(spans, meta.windows)]
        causal = sum(m * t0 + m * (m + 1) // 2 for m, t0 in zip(spans, hist))
        kv_bytes = sum(meta.windows) * hk * d * 2 * 2
        if parts is not None:
            ops.attention_decode_qkv(parts[0], parts[1], meta.pos, meta.slots, self.weights.rope,
                                     self.pool.layer_k(r, layer), self.pool.layer_v(r, layer),
                                     meta.bt, cu, meta.kvlen, out, n_items=meta.n,
                                     max_kv_len=meta.max_kv, q_heads=hq, kv_heads=hk,
                                     block_size=self.pool.block_size, ws=ws,
                                     work_flops=4 * d * hq * causal, work_bytes=kv_bytes)
        elif not tails and not decode_like and meta.n_combine is not None:
            ops.attention_prefill_split(
                q, self.pool.layer_k(r, layer), self.pool.layer_v(r, layer), meta.bt, cu, first,
                meta.kvlen, out, work=meta.work_pairs, split=meta.work_split,
                n_work=meta.n_work, combine=meta.work_combine, n_combine=meta.n_combine,
                n_slots=meta.n_slots, q_heads=hq, kv_heads=hk, head_dim=d,
                block_size=self.pool.block_size, ws=self._ws, work_flops=4 * d * hq * causal,
                work_bytes=kv_bytes)
        else:
            ops.attention(q, self.pool.layer_k(r, layer), self.pool.layer_v(r, layer), meta.bt,
                          cu, first, meta.kvlen, out, n_items=meta.n,
                          work=None if decode_like else meta.work_pairs,
                          n_work=0 if decode_like else meta.n_work, max_q_len=max(spans),
                          max_kv_len=meta.max_kv, q_heads=hq, kv_heads=hk, head_dim=d,
                          block_size=self.pool.block_size, ws=ws,
                          work_flops=4 * d * hq * causal, work_bytes=kv_bytes)
        # reference meter: per item per owned head, q·Kᵀ and P·V over the full window
        for m, w in zip(spans, meta.windows):
            meter.add_matmul(hq * m, d, w)
            meter.add_matmul(hq * m, w, d)

    def _kv_write(self, r: int, layer: int, qkv: torch.Tensor, q_out: Optional[torch.Tensor],
                  meta: _Meta, batch: Batch, *, q_heads: Optional[int] = None,
                  pos=None, slots=None, rows=None, parts=None) -> None:
        cfg = self.config
        P = self.world_size
        hq = cfg.n_heads // P if q_heads is None else q_heads
        if parts is not None:
            ops.rope_kv_write_partials(parts[0], parts[1], meta.pos if pos is None else pos,
                                       meta.slots if slots is None else slots, self.weights.rope,
                                       q_out, self.pool.layer_k(r, layer),
                                       self.pool.layer_v(r, layer),
                                       rows=meta.M if rows is None else rows, q_heads=hq,
                                       kv_heads=cfg.kv_heads // P, head_dim=cfg.head_dim,
                                       block_size=self.pool.block_size)
            return
        ops.rope_kv_write(qkv, meta.pos if pos is None else pos,
                          meta.slots if slots is None else slots, self.weights.rope, q_out,
                          self.pool.layer_k(r, layer), self.pool.layer_v(r, layer),
                          rows=meta.M if rows is None else rows, q_heads=hq,
                          kv_heads=cfg.kv_heads // P, head_dim=cfg.head_dim,
                          block_size=self.pool.block_size)

    def _attn_rope_fusable(self, meta) -> bool:
        """Decode pass whose attention runs on the TMA decode kernel (head_dim
        128, pages of a multiple of 64 keys): RoPE + the KV write go into it
        (SP_FUSE_ATTN_ROPE=0 keeps the separate kernel)."""
        return (self._fuse_attn_rope and meta.decode_like and self.config.head_dim == 128
                and self.pool.block_size % 64 == 0)

    def _fused_qkv_rope(self, M: int, hq: int, hk: int) -> bool:
        """QKV GEMM with RoPE + KV write in its epilogue: prefill-size passes
        (the decode regime keeps its K-split partials -> RoPE kernel), head_dim
        128, whole-head 256-column tiles.  SP_FUSE_ROPE=0 disables."""
        return (M > 256 and self.config.head_dim == 128 and (hq + 2 * hk) % 2 == 0
                and self._fuse_rope)

    def _qkv_rope(self, r, layer, xn, wqkv, q, meta, hq, hk, meter) -> None:
        h = self.config.hidden
        ops.gemm_qkv_rope(xn, wqkv, M=meta.M, K=h, lda=h, ldb=h, pos=meta.pos, slot=meta.slots,
                          rope=self.weights.rope, q_out=q, k_pool=self.pool.layer_k(r, layer),
                          v_pool=self.pool.layer_v(r, layer), q_heads=hq, kv_heads=hk,
                          block_size=self.pool.block_size, meter=meter)

    def _stage_all(self, layer: int, batch: Batch) -> None:
        # every process tracks the global cursors: all P devices append this layer
        if self._capturing:
            return  # graph capture re-records a pass whose writes are already counted
        for it in batch.items:
            for dev in range(self.world_size):
                it.seq.cache._stage(dev, layer, len(it.tokens))

    def _split(self, logits: torch.Tensor, meta: _Meta, span: bool) -> List[torch.Tensor]:
        if span:
            out, lo = [], 0
            for m in meta.spans:
                out.append(logits[lo:lo + m])
                lo += m
            return out
        return [logits[i] for i in range(meta.n)]

    # ================================================================= TP
    def _forward_tp(self, meta, batch, meters, span_logits, cut):
        if self._use_fused_decode(meta, span_logits, cut):
            return self._forward_tp_fused_decode(meta, batch, meters)
        peer = self._peer
        if (peer is not None and cut is None and two_shot_min_rows() < meta.M <= peer.max_tokens):
            return self._forward_tp_two_shot(meta, batch, meters, span_logits, peer)
        cfg, w, g = self.config, self.weights, self.group
        P = self.world_size
        M, h, d = meta.M, cfg.hidden, cfg.head_dim
        hq, hk = cfg.n_heads // P, cfg.kv_heads // P
        W = w.qkv_width
        hqw = hq * d
        fl = cfg.ffn_dim // P
        dev = self.device
        eps = cfg.norm_eps
        x = torch.empty((M, h), dtype=torch.float32, device=dev)
        ops.embed(meta.toks, w.embed, x, meta.pos, w.pos_table)
        pending: Optional[torch.Tensor] = None
        n_full = cfg.n_layers if cut is None else cut
        xn = torch.empty((M, h), dtype=torch.bfloat16, device=dev)
        # fused one-shot all-reduce over peer memory (partials -> peers' sum in the norm kernel)
        peer = self._peer if (self._peer is not None and M <= self._peer.max_tokens) else None
        peer_pending = False
        peer_slabs = [1, 1]   # K-split slabs per rank in the peer partial buffers (O, down)
        split_pending = None  # (K-split partials of the last projection, count) -> next norm
        for layer in range(n_full):
            lw = w.layers[layer]
            if peer_pending:
                ops.peer_allreduce_add_rmsnorm(peer.part_ptrs[1], P, x, lw.attn_gain, eps, xn, M,
                                               slabs=peer_slabs[1])
            elif split_pending is not None:
                ops.add_rmsnorm(x, lw.attn_gain, eps, xn, add=split_pending[0],
                                n_add=split_pending[1])
                split_pending = None
            else:
                ops.add_rmsnorm(x, lw.attn_gain, eps, xn, add=pending)
            self._stage_all(layer, batch)
            parts = {}
            for r in g.local_ranks:
                q = torch.empty((M, hqw), dtype=torch.bfloat16, device=dev)
                n_qkv = self._partials(M, W, h)
                fused_parts = None
                if n_qkv > 1:  # decode: K-split partials reduced inside RoPE + KV write
                    qparts = torch.empty((n_qkv, M, W), dtype=torch.float32, device=dev)
                    ops.gemm(xn, lw.wqkv[r * W:(r + 1) * W], qparts, ops.EPI_PARTIAL_F32, M=M,
                             N=W, K=h, lda=h, ldb=h, ldd=W, meter=meters[r])
                    if self._attn_rope_fusable(meta):  # ... or inside the decode attention
                        fused_parts = (qparts, n_qkv)
                    else:
                        self._kv_write(r, layer, None, q, meta, batch, parts=(qparts, n_qkv))
                elif self._fused_qkv_rope(M, hq, hk):
                    self._qkv_rope(r, layer, xn, lw.wqkv[r * W:(r + 1) * W], q, meta, hq, hk,
                                   meters[r])
                else:
                    qkv = torch.empty((M, W), dtype=torch.bfloat16, device=dev)
                    ops.gemm(xn, lw.wqkv[r * W:(r + 1) * W], qkv, ops.EPI_STORE_BF16, M=M, N=W,
                             K=h, lda=h, ldb=h, ldd=W, meter=meters[r])
                    self._kv_write(r, layer, qkv, q, meta, batch)
                o = torch.empty((M, hqw), dtype=torch.bfloat16, device=dev)
                self._attend(r, layer, q, o, meta, meters[r], parts=fused_parts)
                wo = lw.wo[:, r * hqw:]
                if P == 1:
                    split_pending = self._proj_residual(o, wo, x, M, h, hqw, cfg.n_heads * d,
                                                        meters[r], fuse=True)
                else:
                    part, peer_slabs[0] = self._tp_partial(peer, r, 0, o, wo, M, hqw,
                                                           cfg.n_heads * d, meters[r])
                    parts[r] = part
                    if peer is not None:
                        ops.peer_signal(peer.tp_flag_ptrs[0], P, r)
            xn2 = torch.empty((M, h), dtype=torch.bfloat16, device=dev)
            if peer is not None:
                self._peer_reduce_wait(0, parts)
                ops.peer_allreduce_add_rmsnorm(peer.part_ptrs[0], P, x, lw.mlp_gain, eps, xn2, M,
                                               slabs=peer_slabs[0])
            elif split_pending is not None:
                ops.add_rmsnorm(x, lw.mlp_gain, eps, xn2, add=split_pending[0],
                                n_add=split_pending[1])
                split_pending = None
            else:
                red = g.all_reduce_sum(parts)[g.local_ranks[0]] if P > 1 else None
                ops.add_rmsnorm(x, lw.mlp_gain, eps, xn2, add=red)
            parts = {}
            for r in g.local_ranks:
                act = torch.empty((M, fl), dtype=torch.bfloat16, device=dev)
                self._mlp_up(xn2, lw, r, act, M, meters[r])
                wd = lw.wdown[:, r * fl:]
                if P == 1:
                    # the last layer's sum must land in x before the final norm
                    split_pending = self._proj_residual(act, wd, x, M, h, fl, cfg.ffn_dim,
                                                        meters[r], fuse=layer < n_full - 1)
                else:
                    part, peer_slabs[1] = self._tp_partial(peer, r, 1, act, wd, M, fl,
                                                           cfg.ffn_dim, meters[r])
                    parts[r] = part
                    if peer is not None:
                        ops.peer_signal(peer.tp_flag_ptrs[1], P, r)
            if peer is not None:
                self._peer_reduce_wait(1, parts)
                peer_pending = True
            else:
                pending = g.all_reduce_sum(parts)[g.local_ranks[0]] if P > 1 else None
        if peer_pending:
            ops.peer_allreduce_add_rmsnorm(peer.part_ptrs[1], P, x, None, eps, None, M,
                                           slabs=peer_slabs[1])
        elif pending is not None:
            ops.add_f32(x, pending, x)
        if cut is not None:
            x_rows, n_rows = self._tail_tp(meta, batch, meters, x, cut), meta.n
            row_idx = None
        else:
            x_rows = x
            if span_logits:
                row_idx, n_rows = None, M
            else:
                row_idx, n_rows = meta.ends, meta.n
        xf = torch.empty((n_rows, h), dtype=torch.bfloat16, device=dev)
        ops.add_rmsnorm(x_rows, w.final_gain, eps, xf, row_idx=row_idx, rows=n_rows)
        logits = self._head_tp({r: xf for r in g.local_ranks}, n_rows, meters)
        return self._split(logits, meta, span_logits and cut is None)

    def _use_fused_decode(self, meta, span_logits, cut) -> bool:
        """The fused decode-layer kernel applies: one rank, a decode pass of at
        most 64 single-token items, SwiGLU, head_dim 128, widths it tiles.
        Opt-in (SP_DECODE_FUSED=1); SP_GEMM_NO_SPLITK (which pins the one-chain
        GEMM numerics for the cross-mode bit-identity tests) keeps the unfused path."""
        cfg = self.config
        return (self._decode_fused and self.world_size == 1 and cut is None and not span_logits
                and meta.decode_like and 0 < meta.M <= 64 and cfg.mlp == "swiglu"
                and cfg.head_dim == 128 and cfg.hidden % 256 == 0 and cfg.hidden <= 8192
                and cfg.ffn_dim % 128 == 0 and (cfg.n_heads * cfg.head_dim) % 64 == 0
                and os.environ.get("SP_GEMM_NO_SPLITK") is None)

    def _forward_tp_fused_decode(self, meta, batch, meters):
        """TP decode at P = 1 with every layer's projections in ONE persistent
        kernel (ops.decode_layer): per layer [attention] -> [O + residual +
        norm, gate/up + SwiGLU, down + residual + next norm, next QKV + RoPE +
        KV write].  Same algorithm as _forward_tp (parallel_engine.py:333-398);
        the K-split partial sums differ in split points only."""
        cfg, w = self.config, self.weights
        M, h, d = meta.M, cfg.hidden, cfg.head_dim
        hq, hk, f = cfg.n_heads, cfg.kv_heads, cfg.ffn_dim
        W, hqw, L = w.qkv_width, hq * d, cfg.n_layers
        dev, eps = self.device, cfg.norm_eps
        bf = torch.bfloat16
        x = torch.empty((M, h), dtype=torch.float32, device=dev)
        ops.embed(meta.toks, w.embed, x, meta.pos, w.pos_table)
        xn = torch.empty((M, h), dtype=bf, device=dev)
        xn2 = torch.empty((M, h), dtype=bf, device=dev)
        xf = torch.empty((M, h), dtype=bf, device=dev)
        act = torch.empty((M, f), dtype=bf, device=dev)
        q = torch.empty((M, hqw), dtype=bf, device=dev)
        o = torch.empty((M, hqw), dtype=bf, device=dev)

        def qkv(layer):
            return ops.DlProj(w.layers[layer].wqkv, xn, ops.DL_ROPE_KV, n=W, k=h, ldw=h)

        def rope(layer):
            return dict(pos=meta.pos, slot=meta.slots, rope=w.rope, q_out=q,
                        k_pool=self.pool.layer_k(0, layer), v_pool=self.pool.layer_v(0, layer),
                        q_heads=hq, kv_heads=hk, block_size=self.pool.block_size, head_dim=d)

        def body(layer):
            lw = w.layers[layer]
            last = layer == L - 1
            nxt = None if last else w.layers[layer + 1]
            return [ops.DlProj(lw.wo, o, ops.DL_RES_NORM, n=h, k=hqw, ldw=hq * d,
                               gain=lw.mlp_gain, out=xn2),
                    ops.DlProj(lw.wgu, xn2, ops.DL_SWIGLU, n=2 * f, k=h, ldw=h, out=act),
                    ops.DlProj(lw.wdown, act, ops.DL_RES_NORM, n=h, k=f, ldw=f,
                               gain=w.final_gain if last else nxt.attn_gain,
                               out=xf if last else xn)] + ([] if last else [qkv(layer + 1)])

        nb = self._dl_ws.get(M)
        if nb is None:
            nb = max(ops.decode_layer_ws_bytes(M, x, body(0)),
                     ops.decode_layer_ws_bytes(M, x, [qkv(0)]))
            self._dl_ws[M] = nb
        ws = torch.empty(-(-nb // 4), dtype=torch.float32, device=dev)
        self._stage_all(0, batch)
        ops.decode_layer(M, x, eps, [qkv(0)], ws=ws, sync=self._dl_sync,
                         lead_gain=w.layers[0].attn_gain, lead_out=xn, rope_args=rope(0),
                         meter=meters[0])
        for layer in range(L):
            self._attend(0, layer, q, o, meta, meters[0])
            if layer + 1 < L:
                self._stage_all(layer + 1, batch)
            ops.decode_layer(M, x, eps, body(layer), ws=ws, sync=self._dl_sync,
                             rope_args=None if layer + 1 == L else rope(layer + 1),
                             meter=meters[0])
        logits = self._head_tp({0: xf}, meta.n, meters)
        return self._split(logits, meta, False)

    def _forward_tp_two_shot(self, meta, batch, meters, span_logits, peer):
        """TP pass for prefill-size M with the two-shot all-reduce over peer
        memory: each projection's f32 partial goes to the rank's peer buffer,
        then every rank reduces ITS row slice (ascending rank sum + residual +
        the next RMSNorm, fused) and pushes the normed bf16 rows into every
        rank's xn buffer.  The residual x stays row-sharded between reductions
        (a row is only read again by its owner); the last reduction pushes the
        final-normed rows for the LM head.  Per rank and all-reduce: reads
        (P-1)/P*M*h*4 B and writes (P-1)/P*M*h*2 B over NVLink, vs
        (P-1)*M*h*4 B for the one-shot kernel.  Bit-identical to it and to the
        collective path (same per-row sums and norm)."""
        cfg, w, g = self.config, self.weights, self.group
        P = self.world_size
        M, h, d = meta.M, cfg.hidden, cfg.head_dim
        hq, hk = cfg.n_heads // P, cfg.kv_heads // P
        W, hqw, fl = w.qkv_width, hq * d, cfg.ffn_dim // P
        dev, eps = self.device, cfg.norm_eps
        x = torch.empty((M, h), dtype=torch.float32, device=dev)
        ops.embed(meta.toks, w.embed, x, meta.pos, w.pos_table)
        for r in g.local_ranks:   # the embedding is replicated: every rank norms all rows
            ops.add_rmsnorm(x, w.layers[0].attn_gain, eps, peer.xn[r][0][:M])

        def reduce(pi, gain, xi):
            g.charge("all_reduce", [2.0 * (P - 1) / P * M * h * 4] * P)
            for r in g.local_ranks:
                ops.peer_wait(peer.flags[r][2 + pi], P)
            for r in g.local_ranks:
                ops.peer_reduce_scatter_rmsnorm(peer.part_ptrs[pi], P, r, x, gain, eps,
                                                peer.xn_ptrs[xi], h, M)
            for r in g.local_ranks:
                ops.peer_signal(peer.ag_flag_ptrs[xi], P, r)
            for r in g.local_ranks:
                ops.peer_wait(peer.flags[r][4 + xi], P)

        for layer in range(cfg.n_layers):
            lw = w.layers[layer]
            if layer > 0:
                reduce(1, lw.attn_gain, 0)
            self._stage_all(layer, batch)
            for r in g.local_ranks:
                xn = peer.xn[r][0][:M]
                q = torch.empty((M, hqw), dtype=torch.bfloat16, device=dev)
                if self._fused_qkv_rope(M, hq, hk):
                    self._qkv_rope(r, layer, xn, lw.wqkv[r * W:(r + 1) * W], q, meta, hq, hk,
                                   meters[r])
                else:
                    qkv = torch.empty((M, W), dtype=torch.bfloat16, device=dev)
                    ops.gemm(xn, lw.wqkv[r * W:(r + 1) * W], qkv, ops.EPI_STORE_BF16, M=M, N=W,
                             K=h, lda=h, ldb=h, ldd=W, meter=meters[r])
                    self._kv_write(r, layer, qkv, q, meta, batch)
                o = torch.empty((M, hqw), dtype=torch.bfloat16, device=dev)
                self._attend(r, layer, q, o, meta, meters[r])
                ops.gemm(o, lw.wo[:, r * hqw:], peer.part[r][0][:M], ops.EPI_STORE_F32, M=M, N=h,
                         K=hqw, lda=hqw, ldb=cfg.n_heads * d, ldd=h, meter=meters[r])
                ops.peer_signal(peer.tp_flag_ptrs[0], P, r)
            reduce(0, lw.mlp_gain, 1)
            for r in g.local_ranks:
                act = torch.empty((M, fl), dtype=torch.bfloat16, device=dev)
                self._mlp_up(peer.xn[r][1][:M], lw, r, act, M, meters[r])
                ops.gemm(act, lw.wdown[:, r * fl:], peer.part[r][1][:M], ops.EPI_STORE_F32, M=M,
                         N=h, K=fl, lda=fl, ldb=cfg.ffn_dim, ldd=h, meter=meters[r])
                ops.peer_signal(peer.tp_flag_ptrs[1], P, r)
        reduce(1, w.final_gain, 0)   # final norm, pushed like an attention norm
        n_rows = M if span_logits else meta.n
        vs = cfg.vocab_size // P
        xfs = {}
        for r in g.local_ranks:
            if span_logits:
                xfs[r] = peer.xn[r][0][:M]
            else:
                xfs[r] = torch.empty((n_rows, h), dtype=torch.bfloat16, device=dev)
                ops.gather_rows_bf16(peer.xn[r][0], meta.ends, xfs[r])
        logits = self._head_tp(xfs, n_rows, meters)
        return self._split(logits, meta, span_logits)

    def _tp_partial(self, peer, r, which, a, w, M, K, ldb, meter):
        """Rank r's TP partial of a residual projection (O: which=0, down: 1).
        With peer buffers in the split-K (decode) regime the GEMM leaves its
        K-split slabs there and the one-shot all-reduce kernel sums them (no
        reduce kernel); returns (partial tensor, slabs per rank)."""
        h = self.config.hidden
        if peer is None:
            part = torch.empty((M, h), dtype=torch.float32, device=self.device)
            ops.gemm(a, w, part, ops.EPI_STORE_F32, M=M, N=h, K=K, lda=K, ldb=ldb, ldd=h,
                     meter=meter)
            return part, 1
        n = self._partials(M, h, K)
        if n > 1 and n * M <= peer.max_tokens:
            slabs = peer.part[r][which].view(-1)[:n * M * h].view(n, M, h)
            ops.gemm(a, w, slabs, ops.EPI_PARTIAL_F32, M=M, N=h, K=K, lda=K, ldb=ldb, ldd=h,
                     meter=meter)
            return slabs[0], n
        part = peer.part[r][which][:M]
        ops.gemm(a, w, part, ops.EPI_STORE_F32, M=M, N=h, K=K, lda=K, ldb=ldb, ldd=h,
                 meter=meter)
        return part, 1

    def _peer_reduce_wait(self, which: int, parts: Dict[int, torch.Tensor]) -> None:
        """Ledger + completion wait of a fused TP all-reduce (flag rows 2/3)."""
        g, P, peer = self.group, self.world_size, self._peer
        t = next(iter(parts.values()))
        g.charge("all_reduce", [2.0 * (P - 1) / P * t.numel() * t.element_size()] * P)
        for r in g.local_ranks:
            ops.peer_wait(peer.flags[r][2 + which], P)

    def _partials(self, M: int, N: int, K: int) -> int:
        """K-split partial count for fusing a decode projection's reduction into
        its consumer (1 = not split / fusion off: SP_FUSE_SPLITK=0)."""
        return ops.gemm_partials(M, N, K) if self._fuse_splitk else 1

    def _proj_residual(self, a, w, x, M, N, K, ldb, meter, fuse: bool):
        """x += a · w^T (residual projection, P = 1).  In the split-K (decode)
        regime with `fuse`, leave the K-split partials for the next add+RMSNorm
        to sum (no reduce kernel) and return (partials, count); else add in place."""
        n = self._partials(M, N, K) if fuse else 1
        if n > 1:
            parts = torch.empty((n, M, N), dtype=torch.float32, device=x.device)
            ops.gemm(a, w, parts, ops.EPI_PARTIAL_F32, M=M, N=N, K=K, lda=K, ldb=ldb, ldd=N,
                     meter=meter)
            return parts, n
        ops.gemm(a, w, x, ops.EPI_ADD_F32, M=M, N=N, K=K, lda=K, ldb=ldb, ldd=N, meter=meter)
        return None

    def _mlp_up(self, xn2, lw, r, act, rows, meter):
        cfg = self.config
        P = self.world_size
        h = cfg.hidden
        fl = cfg.ffn_dim // P
        if cfg.mlp == "swiglu":
            ops.gemm(xn2, lw.wgu[r * 2 * fl:(r + 1) * 2 * fl], act, ops.EPI_SWIGLU, M=rows,
                     N=2 * fl, K=h, lda=h, ldb=h, ldd=fl, meter=meter)
        else:
            ops.gemm(xn2, lw.wgu[r * fl:(r + 1) * fl], act, ops.EPI_GELU, M=rows, N=fl, K=h,
                     lda=h, ldb=h, ldd=fl, meter=meter)

    def _head_tp(self, xfs: Dict[int, torch.Tensor], n_rows: int, meters) -> torch.Tensor:
        """TP LM head + logits all-gather (:381-398): rank r computes vocab
        columns [r V/P, (r+1) V/P).  Ranks of this process write their columns
        straight into the [R, V] result (ldd = V: the gather is free); with one
        rank per process the [R, V/P] blocks are all-gathered and one unpack
        kernel interleaves them into [R, V]."""
        cfg, w, g = self.config, self.weights, self.group
        P, h, V = self.world_size, cfg.hidden, cfg.vocab_size
        vs = V // P
        full = torch.empty((n_rows, V), dtype=torch.float32, device=self.device)
        local = len(g.local_ranks) == P
        for r in g.local_ranks:
            dst, ldd = (full[:, r * vs:], V) if local else (
                torch.empty((n_rows, vs), dtype=torch.float32, device=self.device), vs)
            ops.gemm(xfs[r], w.head[r * vs:(r + 1) * vs], dst, ops.EPI_STORE_F32, M=n_rows, N=vs,
                     K=h, lda=h, ldb=h, ldd=ldd, meter=meters[r])
            part = dst
        if P == 1:
            return full
        if local:
            g.charge("all_gather", [(P - 1) / P * n_rows * V * 4.0] * P)
            return full
        blocks = g.all_gather_blocks(part)   # [P, R, V/P]
        if n_rows:  # f32 moved as bf16 pairs: [P][R][2 vs] -> [R, P * 2 vs]
            ops.a2a_unpack(blocks.view(torch.bfloat16), full.view(torch.bfloat16), n_rows, P, 2 * vs)
        return full

    def _tail_tp(self, meta, batch, meters, x, cut):
        """SwiftKV TP tail (:400-450): later-layer K/V from z = norm(x, gain_cut),
        then only each request's last row through layers >= cut."""
        cfg, w, g = self.config, self.weights, self.group
        P = self.world_size
        M, h, d = meta.M, cfg.hidden, cfg.head_dim
        hq, hk = cfg.n_heads // P, cfg.kv_heads // P
        hqw, kvw = hq * d, 2 * hk * d
        W = w.qkv_width
        fl = cfg.ffn_dim // P
        dev, eps = self.device, cfg.norm_eps
        z = torch.empty((M, h), dtype=torch.bfloat16, device=dev)
        ops.add_rmsnorm(x, w.layers[cut].attn_gain, eps, z)
        for layer in range(cut, cfg.n_layers):
            lw = w.layers[layer]
            self._stage_all(layer, batch)
            for r in g.local_ranks:
                kv = torch.empty((M, kvw), dtype=torch.bfloat16, device=dev)
                ops.gemm(z, lw.wkv[r * kvw:(r + 1) * kvw], kv, ops.EPI_STORE_BF16, M=M, N=kvw,
                         K=h, lda=h, ldb=h, ldd=kvw, meter=meters[r])
                self._kv_write(r, layer, kv, None, meta, batch, q_heads=0)
        n = meta.n
        xt = torch.empty((n, h), dtype=torch.float32, device=dev)
        ops.gather_rows(x, meta.ends, xt)
        xn = torch.empty((n, h), dtype=torch.bfloat16, device=dev)
        pending = None
        for layer in range(cut, cfg.n_layers):
            lw = w.layers[layer]
            ops.add_rmsnorm(xt, lw.attn_gain, eps, xn, add=pending)
            parts = {}
            for r in g.local_ranks:
                qr = torch.empty((n, hqw), dtype=torch.bfloat16, device=dev)
                ops.gemm(xn, lw.wqkv[r * W:r * W + hqw], qr, ops.EPI_STORE_BF16, M=n, N=hqw, K=h,
                         lda=h, ldb=h, ldd=hqw, meter=meters[r])
                q = torch.empty((n, hqw), dtype=torch.bfloat16, device=dev)
                ops.rope_kv_write(qr, meta.tail_pos, meta.tail_slot, w.rope, q,
                                  self.pool.layer_k(r, layer), self.pool.layer_v(r, layer),
                                  rows=n, q_heads=hq, kv_heads=0, head_dim=d,
                                  block_size=self.pool.block_size)
                o = torch.empty((n, hqw), dtype=torch.bfloat16, device=dev)
                self._attend(r, layer, q, o, meta, meters[r], tails=True)
                wo = lw.wo[:, r * hqw:]
                if P == 1:
                    ops.gemm(o, wo, xt, ops.EPI_ADD_F32, M=n, N=h, K=hqw, lda=hqw,
                             ldb=cfg.n_heads * d, ldd=h, meter=meters[r])
                else:
                    part = torch.empty((n, h), dtype=torch.float32, device=dev)
                    ops.gemm(o, wo, part, ops.EPI_STORE_F32, M=n, N=h, K=hqw, lda=hqw,
                             ldb=cfg.n_heads * d, ldd=h, meter=meters[r])
                    parts[r] = part
            red = g.all_reduce_sum(parts)[g.local_ranks[0]] if P > 1 else None
            xn2 = torch.empty((n, h), dtype=torch.bfloat16, device=dev)
            ops.add_rmsnorm(xt, lw.mlp_gain, eps, xn2, add=red)
            parts = {}
            for r in g.local_ranks:
                act = torch.empty((n, fl), dtype=torch.bfloat16, device=dev)
                self._mlp_up(xn2, lw, r, act, n, meters[r])
                wd = lw.wdown[:, r * fl:]
                if P == 1:
                    ops.gemm(act, wd, xt, ops.EPI_ADD_F32, M=n, N=h, K=fl, lda=fl,
                             ldb=cfg.ffn_dim, ldd=h, meter=meters[r])
                else:
                    part = torch.empty((n, h), dtype=torch.float32, device=dev)
                    ops.gemm(act, wd, part, ops.EPI_STORE_F32, M=n, N=h, K=fl, lda=fl,
                             ldb=cfg.ffn_dim, ldd=h, meter=meters[r])
                    parts[r] = part
            pending = g.all_reduce_sum(parts)[g.local_ranks[0]] if P > 1 else None
        if pending is not None:
            ops.add_f32(xt, pending, xt)
        return xt

    # ================================================================= SP
    def _forward_sp(self, meta, batch, meters, span_logits, cut):
        if self.sp_degree < self.world_size:
            if cut is not None:
                raise ContractViolation("SwiftKV early exit is implemented for pure SP/TP only")
            return self._forward_sptp(meta, batch, meters, span_logits)
        cfg, w, g = self.config, self.weights, self.group
        P = self.world_size
        M, h, d = meta.M, cfg.hidden, cfg.head_dim
        hq, hk = cfg.n_heads // P, cfg.kv_heads // P
        W = w.qkv_width
        hqw = hq * d
        dev, eps = self.device, cfg.norm_eps
        rows, bounds = meta.rows, meta.bounds
        xs = {}
        for r in g.local_ranks:
            lo, hi = bounds[r]
            xs[r] = torch.empty((hi - lo, h), dtype=torch.float32, device=dev)
            ops.embed(meta.toks[lo:hi], w.embed, xs[r], meta.pos[lo:hi], w.pos_table)
        n_full = cfg.n_layers if cut is None else cut
        in_fwd = {r: [rows[r]] * P for r in range(P)}
        out_fwd = {s: list(rows) for s in range(P)}
        peer = self._peer if (self._peer is not None and M <= self._peer.max_tokens) else None
        split_pending = None  # P = 1: K-split partials of the last projection -> next norm
        for layer in range(n_full):
            lw = w.layers[layer]
            send, recv = {}, {}
            for r in g.local_ranks:
                xn = torch.empty((rows[r], h), dtype=torch.bfloat16, device=dev)
                if split_pending is not None:
                    ops.add_rmsnorm(xs[r], lw.attn_gain, eps, xn, add=split_pending[0],
                                    n_add=split_pending[1])
                    split_pending = None
                else:
                    ops.add_rmsnorm(xs[r], lw.attn_gain, eps, xn)
                if peer is not None:
                    # fused seq->head all-to-all: the epilogue stores rank s's q|k|v
                    # heads straight into s's receive buffer at this shard's rows
                    ops.gemm_to_peers(xn, lw.wqkv, peer.recv_ptrs, row_off=bounds[r][0],
                                      M=rows[r], N=P * W, K=h, lda=h, ldb=h, ldd=W,
                                      peer_width=W, peer_ptrs_host=peer.recv_ptrs_host,
                                      meter=meters[r])
                    ops.peer_signal(peer.fwd_flag_ptrs, P, r)
                elif P == 1:
                    n_qkv = self._partials(M, W, h)
                    if n_qkv > 1:  # decode: K-split partials reduced inside RoPE + KV write
                        qparts = torch.empty((n_qkv, M, W), dtype=torch.float32, device=dev)
                        ops.gemm(xn, lw.wqkv, qparts, ops.EPI_PARTIAL_F32, M=M, N=W, K=h,
                                 lda=h, ldb=h, ldd=W, meter=meters[r])
                        recv[r] = (qparts, n_qkv)
                    elif self._fused_qkv_rope(M, hq, hk):
                        qf = torch.empty((M, hqw), dtype=torch.bfloat16, device=dev)
                        self._qkv_rope(r, layer, xn, lw.wqkv, qf, meta, hq, hk, meters[r])
                        recv[r] = _RopedQ(qf)
                    else:
                        send[r] = torch.empty((M, W), dtype=torch.bfloat16, device=dev)
                        ops.gemm(xn, lw.wqkv, send[r], ops.EPI_STORE_BF16, M=M, N=W, K=h, lda=h,
                                 ldb=h, ldd=W, meter=meters[r])
                        recv[r] = send[r]
                else:
                    # epilogue writes rank s's q|k|v heads into send block s (fused pack)
                    send[r] = torch.empty((P * rows[r], W), dtype=torch.bfloat16, device=dev)
                    ops.gemm(xn, lw.wqkv, send[r], ops.EPI_STORE_BF16, M=rows[r], N=P * W, K=h,
                             lda=h, ldb=h, ldd=W, peer_width=W, peer_stride=rows[r] * W,
                             meter=meters[r])
                    recv[r] = torch.empty((M, W), dtype=torch.bfloat16, device=dev)
            if peer is not None:
                g._charge_a2a(in_fwd, W * 2)
                for r in g.local_ranks:
                    ops.peer_wait(peer.flags[r][0], P)
                    recv[r] = peer.recv[r][:M]
            elif P > 1:
                g.all_to_all(send, recv, in_fwd, out_fwd, row_bytes=W * 2)
            self._stage_all(layer, batch)
            att = {}
            for r in g.local_ranks:
                fused_parts = None
                if isinstance(recv[r], _RopedQ):  # RoPE + KV write done in the QKV epilogue
                    q = recv[r].q
                elif isinstance(recv[r], tuple) and self._attn_rope_fusable(meta):
                    q, fused_parts = None, recv[r]  # ... or inside the decode attention (P = 1)
                else:
                    q = torch.empty((M, hqw), dtype=torch.bfloat16, device=dev)
                    if isinstance(recv[r], tuple):
                        self._kv_write(r, layer, None, q, meta, batch, parts=recv[r])
                    else:
                        self._kv_write(r, layer, recv[r], q, meta, batch)
                o = torch.empty((M, hqw), dtype=torch.bfloat16, device=dev)
                self._attend(r, layer, q, o, meta, meters[r], parts=fused_parts)
                att[r] = o
            back = att
            if peer is not None:
                # fused head->seq all-to-all: rows go straight to their owner's buffer
                for r in g.local_ranks:
                    ops.peer_scatter_rows(att[r], M, P, r, peer.back_ptrs)
                    ops.peer_signal(peer.back_flag_ptrs, P, r)
                g._charge_a2a({r: list(rows) for r in range(P)}, hqw * 2)
                back = {}
                for r in g.local_ranks:
                    ops.peer_wait(peer.flags[r][1], P)
                    back[r] = peer.back[r][:P * rows[r]]
            elif P > 1:
                back = {r: torch.empty((P * rows[r], hqw), dtype=torch.bfloat16, device=dev)
                        for r in g.local_ranks}
                g.all_to_all(att, back, {r: list(rows) for r in range(P)},
                             {s: [rows[s]] * P for s in range(P)}, row_bytes=hqw * 2)
            for r in g.local_ranks:
                xn2 = torch.empty((rows[r], h), dtype=torch.bfloat16, device=dev)
                if P == 1:  # split-K partials summed by the norm (no reduce kernel)
                    sp_o = self._proj_residual(back[r], lw.wo, xs[r], rows[r], h,
                                               cfg.n_heads * d, cfg.n_heads * d, meters[r],
                                               fuse=True)
                    if sp_o is not None:
                        ops.add_rmsnorm(xs[r], lw.mlp_gain, eps, xn2, add=sp_o[0], n_add=sp_o[1])
                    else:
                        ops.add_rmsnorm(xs[r], lw.mlp_gain, eps, xn2)
                else:
                    self._o_proj_sp(back[r], lw, xs[r], rows[r], meters[r])
                    ops.add_rmsnorm(xs[r], lw.mlp_gain, eps, xn2)
                act = torch.empty((rows[r], cfg.ffn_dim), dtype=torch.bfloat16, device=dev)
                self._mlp_up_full(xn2, lw, act, rows[r], meters[r])
                if P == 1:
                    split_pending = self._proj_residual(
                        act, lw.wdown, xs[r], rows[r], h, cfg.ffn_dim, cfg.ffn_dim, meters[r],
                        fuse=layer < n_full - 1 and cut is None)
                else:
                    ops.gemm(act, lw.wdown, xs[r], ops.EPI_ADD_F32, M=rows[r], N=h,
                             K=cfg.ffn_dim, lda=cfg.ffn_dim, ldb=cfg.ffn_dim, ldd=h,
                             meter=meters[r])
        if cut is not None:
            return self._tail_sp(meta, batch, meters, xs, cut)
        parts = {}
        for r in g.local_ranks:
            cnt = meta.sp_counts[r]
            xf = torch.empty((cnt, h), dtype=torch.bfloat16, device=dev)
            idx = getattr(meta, f"sprows{r}")
            ops.add_rmsnorm(xs[r], w.final_gain, eps, xf, row_idx=idx, rows=cnt)
            lg = torch.empty((cnt, cfg.vocab_size), dtype=torch.float32, device=dev)
            ops.gemm(xf, w.head, lg, ops.EPI_STORE_F32, M=cnt, N=cfg.vocab_size, K=h, lda=h,
                     ldb=h, ldd=cfg.vocab_size, meter=meters[r])
            parts[r] = lg
        logits = g.all_gather_rows(parts, meta.sp_counts) if P > 1 else parts[0]
        return self._split(logits, meta, span_logits)

    def _forward_sptp(self, meta, batch, meters, span_logits):
        """SP(s) x TP(t), P = s*t.  Rank r = g*s + i: TP group g (heads of
        ranks g*s .. g*s+s-1, ffn shard g), token shard i.  Per layer: QKV on
        shard i with group g's weight rows, seq->head all-to-all inside the SP
        group {g*s+i'} (rank r ends with head block r — the TP(P)/SP(P) KV
        layout, so the cache stays mode-invariant), attention, head->seq
        all-to-all back, O and MLP as TP(t) partials all-reduced inside the TP
        group {g'*s+i}.  Not in the reference (SPEC.md:334 leaves mixed modes
        unimplemented); parity is checked against the dense oracle and the pure
        modes."""
        cfg, w, grp = self.config, self.weights, self.group
        P, s = self.world_size, self.sp_degree
        t = P // s
        M, h, d = meta.M, cfg.hidden, cfg.head_dim
        W = w.qkv_width                  # q|k|v width of ONE rank's head block
        hqw = cfg.n_heads // P * d       # one rank's q width
        fl = cfg.ffn_dim // t            # this TP group's ffn shard
        dev, eps = self.device, cfg.norm_eps
        rows, bounds = meta.rows, meta.bounds   # per token shard i
        grp_of = {r: (r // s, r % s) for r in range(P)}
        xs = {}
        for r in grp.local_ranks:
            g, i = grp_of[r]
            lo, hi = bounds[i]
            xs[r] = torch.empty((hi - lo, h), dtype=torch.float32, device=dev)
            ops.embed(meta.toks[lo:hi], w.embed, xs[r], meta.pos[lo:hi], w.pos_table)
        # split tables: exchanges stay inside SP groups (zero rows elsewhere)
        in_fwd = {r: [rows[r % s] if d2 // s == r // s else 0 for d2 in range(P)] for r in range(P)}
        out_fwd = {r: [rows[s2 % s] if s2 // s == r // s else 0 for s2 in range(P)] for r in range(P)}
        in_back = {r: [rows[d2 % s] if d2 // s == r // s else 0 for d2 in range(P)] for r in range(P)}
        out_back = {r: [rows[r % s] if s2 // s == r // s else 0 for s2 in range(P)] for r in range(P)}
        tp_members = {r: [g2 * s + r % s for g2 in range(t)] for r in range(P)}
        pending = None
        for layer in range(cfg.n_layers):
            lw = w.layers[layer]
            send, recv = {}, {}
            for r in grp.local_ranks:
                g, i = grp_of[r]
                xn = torch.empty((rows[i], h), dtype=torch.bfloat16, device=dev)
                ops.add_rmsnorm(xs[r], lw.attn_gain, eps, xn,
                                add=None if pending is None else pending[r])
                # group g's s head blocks; block i' -> send block i' (fused pack)
                send[r] = torch.empty((s * rows[i], W), dtype=torch.bfloat16, device=dev)
                ops.gemm(xn, lw.wqkv[g * s * W:(g + 1) * s * W], send[r], ops.EPI_STORE_BF16,
                         M=rows[i], N=s * W, K=h, lda=h, ldb=h, ldd=W, peer_width=W,
                         peer_stride=rows[i] * W, meter=meters[r])
                recv[r] = torch.empty((M, W), dtype=torch.bfloat16, device=dev)
            grp.all_to_all(send, recv, in_fwd, out_fwd, row_bytes=W * 2, group_size=s)
            self._stage_all(layer, batch)
            att = {}
            for r in grp.local_ranks:
                q = torch.empty((M, hqw), dtype=torch.bfloat16, device=dev)
                self._kv_write(r, layer, recv[r], q, meta, batch)
                o = torch.empty((M, hqw), dtype=torch.bfloat16, device=dev)
                self._attend(r, layer, q, o, meta, meters[r])
                att[r] = o
            back = {r: torch.empty((s * rows[r % s], hqw), dtype=torch.bfloat16, device=dev)
                    for r in grp.local_ranks}
            grp.all_to_all(att, back, in_back, out_back, row_bytes=hqw * 2, group_size=s)
            parts = {}
            for r in grp.local_ranks:
                g, i = grp_of[r]
                part = torch.empty((rows[i], h), dtype=torch.float32, device=dev)
                # A = [s blocks][rows_i][hqw] (the receive layout), K = s * hqw
                ops.gemm(back[r], lw.wo[:, g * s * hqw:], part, ops.EPI_STORE_F32, M=rows[i],
                         N=h, K=s * hqw, lda=hqw, ldb=cfg.n_heads * d, ldd=h,
                         a_kchunk=hqw if hqw % 64 == 0 and s > 1 else 0,
                         a_chunk_stride=rows[i] * hqw, meter=meters[r])
                parts[r] = part
            red = self._group_sum(parts, tp_members)
            parts = {}
            for r in grp.local_ranks:
                g, i = grp_of[r]
                xn2 = torch.empty((rows[i], h), dtype=torch.bfloat16, device=dev)
                ops.add_rmsnorm(xs[r], lw.mlp_gain, eps, xn2, add=red[r])
                act = torch.empty((rows[i], fl), dtype=torch.bfloat16, device=dev)
                if cfg.mlp == "swiglu":
                    ops.gemm(xn2, lw.wgu[g * 2 * fl:(g + 1) * 2 * fl], act, ops.EPI_SWIGLU,
                             M=rows[i], N=2 * fl, K=h, lda=h, ldb=h, ldd=fl, meter=meters[r])
                else:
                    ops.gemm(xn2, lw.wgu[g * fl:(g + 1) * fl], act, ops.EPI_GELU, M=rows[i],
                             N=fl, K=h, lda=h, ldb=h, ldd=fl, meter=meters[r])
                part = torch.empty((rows[i], h), dtype=torch.float32, device=dev)
                ops.gemm(act, lw.wdown[:, g * fl:], part, ops.EPI_STORE_F32, M=rows[i], N=h,
                         K=fl, lda=fl, ldb=cfg.ffn_dim, ldd=h, meter=meters[r])
                parts[r] = part
            pending = self._group_sum(parts, tp_members)
        # final norm + LM head on each shard's returned rows; every TP group holds
        # the same rows, so group 0's shards are gathered (in shard order)
        lg_parts = {}
        counts = [0] * P
        for r in grp.local_ranks:
            g, i = grp_of[r]
            cnt = meta.sp_counts[i]
            ops.add_f32(xs[r], pending[r], xs[r])
            xf = torch.empty((cnt, h), dtype=torch.bfloat16, device=dev)
            ops.add_rmsnorm(xs[r], w.final_gain, eps, xf, row_idx=getattr(meta, f"sprows{i}"),
                            rows=cnt)
            lg = torch.empty((cnt, cfg.vocab_size), dtype=torch.float32, device=dev)
            ops.gemm(xf, w.head, lg, ops.EPI_STORE_F32, M=cnt, N=cfg.vocab_size, K=h, lda=h,
                     ldb=h, ldd=cfg.vocab_size, meter=meters[r])
            lg_parts[r] = lg
        for r in range(P):
            counts[r] = meta.sp_counts[r % s] if r // s == 0 else 0
        for r in grp.local_ranks:  # ranks outside group 0 contribute nothing
            if r // s:
                lg_parts[r] = lg_parts[r][:0]
        logits = grp.all_gather_rows(lg_parts, counts) if P > 1 else lg_parts[0]
        return self._split(logits, meta, span_logits)

    def _group_sum(self, parts: Dict[int, torch.Tensor], members: Dict[int, List[int]]):
        """TP all-reduce inside each TP group of SP x TP (one call per group)."""
        out: Dict[int, torch.Tensor] = {}
        done = set()
        for r in sorted(members):
            key = tuple(members[r])
            if key in done or not any(m in parts for m in key):
                continue
            done.add(key)
            out.update(self.group.all_reduce_sum_group({m: parts[m] for m in key if m in parts},
                                                       list(key)))
        return out

    def _mlp_up_full(self, xn2, lw, act, rows, meter):
        cfg = self.config
        h, f = cfg.hidden, cfg.ffn_dim
        if cfg.mlp == "swiglu":
            ops.gemm(xn2, lw.wgu, act, ops.EPI_SWIGLU, M=rows, N=2 * f, K=h, lda=h, ldb=h, ldd=f,
                     meter=meter)
        else:
            ops.gemm(xn2, lw.wgu, act, ops.EPI_GELU, M=rows, N=f, K=h, lda=h, ldb=h, ldd=f,
                     meter=meter)

    def _o_proj_sp(self, back: torch.Tensor, lw, x: torch.Tensor, rows: int, meter) -> None:
        """x += back · Wo^T where back is [P][rows][Hq/P·d] (all-to-all receive)."""
        cfg = self.config
        P = self.world_size
        hqw = cfg.n_heads // P * cfg.head_dim
        K = cfg.n_heads * cfg.head_dim
        if P == 1:
            ops.gemm(back, lw.wo, x, ops.EPI_ADD_F32, M=rows, N=cfg.hidden, K=K, lda=K, ldb=K,
                     ldd=cfg.hidden, meter=meter)
        elif hqw % 64 == 0:
            ops.gemm(back, lw.wo, x, ops.EPI_ADD_F32, M=rows, N=cfg.hidden, K=K, lda=hqw, ldb=K,
                     ldd=cfg.hidden, a_kchunk=hqw, a_chunk_stride=rows * hqw, meter=meter)
        else:
            flat = torch.empty((rows, K), dtype=torch.bfloat16, device=x.device)
            ops.a2a_unpack(back, flat, rows, P, hqw)
            ops.gemm(flat, lw.wo, x, ops.EPI_ADD_F32, M=rows, N=cfg.hidden, K=K, lda=K, ldb=K,
                     ldd=cfg.hidden, meter=meter)

    def _tail_sp(self, meta, batch, meters, xs, cut):
        """SwiftKV SP tail (:544-647): K/V for layers >= cut projected token-locally
        from z = norm(x, gain_cut) and re-sharded by all-to-all; each request's
        last row stays on the rank that owns it."""
        cfg, w, g = self.config, self.weights, self.group
        P = self.world_size
        M, h, d = meta.M, cfg.hidden, cfg.head_dim
        hq, hk = cfg.n_heads // P, cfg.kv_heads // P
        hqw, kvw = hq * d, 2 * hk * d
        W = w.qkv_width
        dev, eps = self.device, cfg.norm_eps
        rows, bounds = meta.rows, meta.bounds
        zs = {}
        for r in g.local_ranks:
            zs[r] = torch.empty((rows[r], h), dtype=torch.bfloat16, device=dev)
            ops.add_rmsnorm(xs[r], w.layers[cut].attn_gain, eps, zs[r])
        in_fwd = {r: [rows[r]] * P for r in range(P)}
        out_fwd = {s: list(rows) for s in range(P)}
        for layer in range(cut, cfg.n_layers):
            lw = w.layers[layer]
            send, recv = {}, {}
            for r in g.local_ranks:
                if P == 1:
                    send[r] = torch.empty((M, kvw), dtype=torch.bfloat16, device=dev)
                    ops.gemm(zs[r], lw.wkv, send[r], ops.EPI_STORE_BF16, M=M, N=kvw, K=h, lda=h,
                             ldb=h, ldd=kvw, meter=meters[r])
                    recv[r] = send[r]
                else:
                    send[r] = torch.empty((P * rows[r], kvw), dtype=torch.bfloat16, device=dev)
                    ops.gemm(zs[r], lw.wkv, send[r], ops.EPI_STORE_BF16, M=rows[r], N=P * kvw,
                             K=h, lda=h, ldb=h, ldd=kvw, peer_width=kvw,
                             peer_stride=rows[r] * kvw, meter=meters[r])
                    recv[r] = torch.empty((M, kvw), dtype=torch.bfloat16, device=dev)
            if P > 1:
                g.all_to_all(send, recv, in_fwd, out_fwd, row_bytes=kvw * 2)
            self._stage_all(layer, batch)
            for r in g.local_ranks:
                self._kv_write(r, layer, recv[r], None, meta, batch, q_heads=0)
        # tails: last row of each request, on its owner rank (ends are ordered by rank)
        ends = meta.ends_host
        owned = [[int(e - lo) for e in ends if lo <= e < hi] for lo, hi in bounds]
        cnt = [len(o) for o in owned]
        tails, tpos, tslot = {}, {}, {}
        first_end = np.cumsum([0] + cnt)
        for r in g.local_ranks:
            idx = torch.as_tensor(np.asarray(owned[r], dtype=np.int32), device=dev)
            tails[r] = torch.empty((cnt[r], h), dtype=torch.float32, device=dev)
            ops.gather_rows(xs[r], idx, tails[r])
        tpos_all = meta.tail_pos
        n = meta.n
        for layer in range(cut, cfg.n_layers):
            lw = w.layers[layer]
            send, recv = {}, {}
            for r in g.local_ranks:
                xn = torch.empty((cnt[r], h), dtype=torch.bfloat16, device=dev)
                ops.add_rmsnorm(tails[r], lw.attn_gain, eps, xn)
                send[r] = torch.empty((P * cnt[r], hqw), dtype=torch.bfloat16, device=dev)
                for s in range(P):  # q heads of peer s (rows [sW, sW + hq d) of wqkv)
                    ops.gemm(xn, lw.wqkv[s * W:s * W + hqw], send[r][s * cnt[r]:], ops.EPI_STORE_BF16,
                             M=cnt[r], N=hqw, K=h, lda=h, ldb=h, ldd=hqw, meter=meters[r])
                recv[r] = send[r] if P == 1 else torch.empty((n, hqw), dtype=torch.bfloat16,
                                                             device=dev)
            if P > 1:
                g.all_to_all(send, recv, {r: [cnt[r]] * P for r in range(P)},
                             {s: list(cnt) for s in range(P)}, row_bytes=hqw * 2)
            att = {}
            for r in g.local_ranks:
                q = torch.empty((n, hqw), dtype=torch.bfloat16, device=dev)
                ops.rope_kv_write(recv[r], tpos_all, meta.tail_slot, w.rope, q,
                                  self.pool.layer_k(r, layer), self.pool.layer_v(r, layer),
                                  rows=n, q_heads=hq, kv_heads=0, head_dim=d,
                                  block_size=self.pool.block_size)
                o = torch.empty((n, hqw), dtype=torch.bfloat16, device=dev)
                self._attend(r, layer, q, o, meta, meters[r], tails=True)
                att[r] = o
            back = att
            if P > 1:
                back = {r: torch.empty((P * cnt[r], hqw), dtype=torch.bfloat16, device=dev)
                        for r in g.local_ranks}
                g.all_to_all(att, back, {r: list(cnt) for r in range(P)},
                             {s: [cnt[s]] * P for s in range(P)}, row_bytes=hqw * 2)
            for r in g.local_ranks:
                self._o_proj_sp(back[r], lw, tails[r], cnt[r], meters[r])
                xn2 = torch.empty((cnt[r], h), dtype=torch.bfloat16, device=dev)
                ops.add_rmsnorm(tails[r], lw.mlp_gain, eps, xn2)
                act = torch.empty((cnt[r], cfg.ffn_dim), dtype=torch.bfloat16, device=dev)
                self._mlp_up_full(xn2, lw, act, cnt[r], meters[r])
                ops.gemm(act, lw.wdown, tails[r], ops.EPI_ADD_F32, M=cnt[r], N=h, K=cfg.ffn_dim,
                         lda=cfg.ffn_dim, ldb=cfg.ffn_dim, ldd=h, meter=meters[r])
        parts = {}
        for r in g.local_ranks:
            xf = torch.empty((cnt[r], h), dtype=torch.bfloat16, device=dev)
            ops.add_rmsnorm(tails[r], w.final_gain, eps, xf)
            lg = torch.empty((cnt[r], cfg.vocab_size), dtype=torch.float32, device=dev)
            ops.gemm(xf, w.head, lg, ops.EPI_STORE_F32, M=cnt[r], N=cfg.vocab_size, K=h, lda=h,
                     ldb=h, ldd=cfg.vocab_size, meter=meters[r])
            parts[r] = lg
        logits = g.all_gather_rows(parts, cnt) if P > 1 else parts[0]
        # gathered rows are in rank order == item order (ends increase with rank)
        return [logits[i] for i in range(n)]


def _rows_view(rows: List[torch.Tensor]) -> Optional[torch.Tensor]:
    """The rows as one [n, V] strided view when they are equally spaced rows
    of one tensor (the engine's logits always are): no copy."""
    r0 = rows[0]
    if r0.dim() != 1 or r0.stride(0) != 1:
        return None
    n = len(rows)
    step = (rows[1].data_ptr() - r0.data_ptr()) // r0.element_size() if n > 1 else r0.shape[0]
    for i, r in enumerate(rows):
        if (r.dim() != 1 or r.shape != r0.shape or r.dtype != r0.dtype or r.stride(0) != 1
                or r.untyped_storage().data_ptr() != r0.untyped_storage().data_ptr()
                or r.data_ptr() != r0.data_ptr() + i * step * r0.element_size()):
            return None
    if step < r0.shape[0]:
        return None
    return r0.as_strided((n, r0.shape[0]), (step, 1))


def greedy_tokens(logits: List[torch.Tensor]) -> List[int]:
    """greedy_token (model.py:303-307) for every item: one argmax kernel, one D2H."""
    if not logits:
        return []
    last = [l if l.dim() == 1 else l[-1] for l in logits]
    rows = _rows_view(last)
    if rows is None:
        rows = torch.stack(last)
    idx = torch.empty(rows.shape[0], dtype=torch.int32, device=rows.device)
    ops.argmax(rows, idx)
    return idx.cpu().tolist()
