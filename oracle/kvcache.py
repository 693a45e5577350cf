"""Oracle KV cache (test infrastructure only).

``OracleKvCache`` restates ``/root/reference/pkg/src/shiftsim/kv_cache.py``
:43-164 — per-sequence, head-sharded, ``(layer, head, token, dim)`` blocks;
staged append at a per-(device, layer) cursor (:99-122), commit only when all
cursors agree (:124-133), logical truncate (:135-140), a byte write counter
(:80-83) and the structural fingerprint (:85-95).

``PagedAllocator`` is the oracle half of the paged layout the B200 build uses
(the reference omits paging): a pool of fixed-size blocks,
lowest-free-block-first allocation, per-sequence block lists, block tables and
slot mappings.  The product's allocator (paper_2507_11830_b200/kv_cache.py)
must reproduce these integers bit-exactly; tests hold them equal.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass
from typing import Dict, List, Tuple

import numpy as np

from .prims import OracleContractError

AXIS_ORDER = "layer,head,token,dim"  # kv_cache.py:26


class OracleCacheOverflow(OracleContractError):
    pass


@dataclass(frozen=True)
class Fingerprint:
    world_size: int
    n_layers: int
    heads_per_device: int
    head_dim: int
    head_partition: Tuple[Tuple[int, int], ...]
    token_count: int
    axis_order: str
    precision: str


class OracleKvCache:
    def __init__(self, n_layers, head_partition, head_dim, capacity, dtype):
        widths = {hi - lo for lo, hi in head_partition}
        if n_layers < 1 or head_dim < 1 or capacity < 1 or len(widths) != 1 or min(widths) < 1:
            raise OracleContractError("bad KvCache geometry")
        self.n_layers = n_layers
        self.head_partition = tuple((int(a), int(b)) for a, b in head_partition)
        self.world_size = len(self.head_partition)
        self.heads_per_device = widths.pop()
        self.head_dim = head_dim
        self.capacity = capacity
        self.dtype = np.dtype(dtype)
        shape = (n_layers, self.heads_per_device, capacity, head_dim)
        self._k = [np.zeros(shape, self.dtype) for _ in range(self.world_size)]
        self._v = [np.zeros(shape, self.dtype) for _ in range(self.world_size)]
        self._count = 0
        self._cursor = np.zeros((self.world_size, n_layers), dtype=np.int64)
        self._writes = [0] * self.world_size

    @property
    def token_count(self) -> int:
        return self._count

    @property
    def write_counter(self) -> int:
        return sum(self._writes)

    def device_write_counter(self, device: int) -> int:
        return self._writes[device]

    def fingerprint(self, precision: str = None) -> Fingerprint:
        prec = precision or ("f32" if self.dtype == np.float32 else "f64")
        return Fingerprint(self.world_size, self.n_layers, self.heads_per_device,
                           self.head_dim, self.head_partition, self._count,
                           AXIS_ORDER, prec)

    def append(self, device, layer, k_rows, v_rows):
        m = k_rows.shape[0]
        if k_rows.shape != v_rows.shape or k_rows.shape != (m, self.heads_per_device, self.head_dim):
            raise OracleContractError(f"append rows {k_rows.shape}")
        cur = int(self._cursor[device, layer])
        if cur + m > self.capacity:
            raise OracleCacheOverflow(f"{cur} + {m} > {self.capacity}")
        self._k[device][layer, :, cur:cur + m, :] = k_rows.transpose(1, 0, 2)
        self._v[device][layer, :, cur:cur + m, :] = v_rows.transpose(1, 0, 2)
        self._cursor[device, layer] = cur + m
        self._writes[device] += k_rows.nbytes + v_rows.nbytes

    def commit(self, m):
        tgt = self._count + m
        if not np.all(self._cursor == tgt):
            raise OracleContractError("commit before every (device, layer) appended")
        self._count = tgt

    def truncate(self, n):
        if not 0 <= n <= self._count:
            raise OracleContractError("truncate out of range")
        self._count = n
        self._cursor[:, :] = n

    def read_window(self, device, layer, local_head):
        cur = int(self._cursor[device, layer])
        return (self._k[device][layer, local_head, :cur, :],
                self._v[device][layer, local_head, :cur, :])

    def device_blocks(self, device):
        return (self._k[device][:, :, :self._count, :],
                self._v[device][:, :, :self._count, :])


class PagedAllocator:
    """Deterministic block allocator (the paged-layout spec both sides share).

    * the pool holds ``num_blocks`` blocks of ``block_size`` token slots;
    * allocation always takes the lowest-numbered free block;
    * a sequence grows its block list on demand, in batch-item order, before
      any write of the pass (capacity precheck, parallel_engine.py:245-251);
    * releasing a sequence returns its blocks to the free pool;
    * slot(p) = table[p // block_size] * block_size + p % block_size.
    """

    def __init__(self, num_blocks: int, block_size: int):
        if num_blocks < 1 or block_size < 1:
            raise OracleContractError("bad pool geometry")
        self.num_blocks = num_blocks
        self.block_size = block_size
        self._free = list(range(num_blocks))
        heapq.heapify(self._free)
        self.tables: Dict[int, List[int]] = {}

    @property
    def free_blocks(self) -> int:
        return len(self._free)

    def blocks_needed(self, seq_id: int, total_tokens: int) -> int:
        have = len(self.tables.get(seq_id, []))
        need = -(-total_tokens // self.block_size)
        return max(0, need - have)

    def reserve(self, seq_id: int, total_tokens: int) -> None:
        extra = self.blocks_needed(seq_id, total_tokens)
        if extra > len(self._free):
            raise OracleCacheOverflow("paged pool exhausted")
        tab = self.tables.setdefault(seq_id, [])
        for _ in range(extra):
            tab.append(heapq.heappop(self._free))

    def release(self, seq_id: int) -> None:
        for b in self.tables.pop(seq_id, []):
            heapq.heappush(self._free, b)

    def slots(self, seq_id: int, positions) -> np.ndarray:
        tab = self.tables[seq_id]
        p = np.asarray(positions, dtype=np.int64)
        blk = np.asarray(tab, dtype=np.int64)[p // self.block_size]
        return (blk * self.block_size + p % self.block_size).astype(np.int32)

    def block_table(self, seq_ids, width: int = None) -> np.ndarray:
        rows = [self.tables.get(s, []) for s in seq_ids]
        w = width if width is not None else max([len(r) for r in rows] + [1])
        out = np.zeros((len(rows), w), dtype=np.int32)
        for i, r in enumerate(rows):
            out[i, :len(r)] = r
        return out
