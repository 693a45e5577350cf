"""Paged, head-sharded, mode-invariant KV cache.

Mirrors ``/root/reference/pkg/src/shiftsim/kv_cache.py``: device d always owns
the same contiguous kv-head range whatever the parallel mode, appends are the
only writes, a pass stages rows at per-(device, layer) cursors and ``commit``
advances the token count once every pair appended (:99-133), ``truncate`` is
logical (:135-140), a write counter proves that mode switches move no bytes
(:80-83), and ``fingerprint`` captures the layout (:85-95).

B200 layout (the reference preallocates per sequence; here one pool per
device is shared by all sequences through block tables):

    k_pool[d], v_pool[d] : bf16 [n_layers][num_blocks][kv_heads/P][block_size][head_dim]

i.e. "layer, head, token, dim" inside each block.  ``BlockAllocator`` hands
out blocks lowest-free-first (the same integer algorithm the oracle's
``PagedAllocator`` specifies); slot(p) = table[p // bs] * bs + p % bs.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

import numpy as np
import torch

from .errors import CacheOverflow, ContractViolation

AXIS_ORDER = "layer,head,token,dim"


@dataclass(frozen=True)
class LayoutFingerprint:
    """Structural identity of a cache layout (kv_cache.py:29-40)."""

    world_size: int
    n_layers: int
    heads_per_device: int
    head_dim: int
    head_partition: Tuple[Tuple[int, int], ...]
    token_count: int
    axis_order: str
    precision: str
    block_size: int


class BlockAllocator:
    def __init__(self, num_blocks: int, block_size: int):
        if num_blocks < 1 or block_size < 1:
            raise ContractViolation("pool needs >= 1 block of >= 1 slot")
        self.num_blocks = num_blocks
        self.block_size = block_size
        self._free = list(range(num_blocks))
        heapq.heapify(self._free)
        self.tables: Dict[int, List[int]] = {}

    @property
    def free_blocks(self) -> int:
        return len(self._free)

    def blocks_needed(self, key: int, total_tokens: int) -> int:
        have = len(self.tables.get(key, ()))
        return max(0, -(-total_tokens // self.block_size) - have)

    def reserve(self, key: int, total_tokens: int) -> None:
        extra = self.blocks_needed(key, total_tokens)
        if extra > len(self._free):
            raise CacheOverflow(f"paged KV pool exhausted ({len(self._free)} free, {extra} needed)")
        tab = self.tables.setdefault(key, [])
        for _ in range(extra):
            tab.append(heapq.heappop(self._free))

    def release(self, key: int) -> None:
        for b in self.tables.pop(key, []):
            heapq.heappush(self._free, b)

    def slots(self, key: int, start: int, count: int) -> np.ndarray:
        tab = np.asarray(self.tables[key], dtype=np.int64)
        p = np.arange(start, start + count, dtype=np.int64)
        return (tab[p // self.block_size] * self.block_size + p % self.block_size).astype(np.int32)


class KvPool:
    """Per-device paged K/V storage for all sequences of one engine."""

    def __init__(self, n_layers: int, kv_partition: Tuple[Tuple[int, int], ...], head_dim: int,
                 num_blocks: int, block_size: int, devices: List[int], device: torch.device):
        self.n_layers = n_layers
        self.kv_partition = kv_partition
        self.world_size = len(kv_partition)
        self.heads_per_device = kv_partition[0][1] - kv_partition[0][0]
        self.head_dim = head_dim
        self.num_blocks = num_blocks
        self.block_size = block_size
        self.alloc = BlockAllocator(num_blocks, block_size)
        shape = (n_layers, num_blocks, self.heads_per_device, block_size, head_dim)
        # only the ranks this process drives hold storage
        self.k = {d: torch.zeros(shape, dtype=torch.bfloat16, device=device) for d in devices}
        self.v = {d: torch.zeros(shape, dtype=torch.bfloat16, device=device) for d in devices}

    @property
    def layer_elems(self) -> int:
        return self.num_blocks * self.heads_per_device * self.block_size * self.head_dim

    def layer_k(self, dev: int, layer: int) -> torch.Tensor:
        return self.k[dev][layer]

    def layer_v(self, dev: int, layer: int) -> torch.Tensor:
        return self.v[dev][layer]

    def bytes_per_token_per_device(self) -> int:
        return 2 * self.heads_per_device * self.head_dim * 2  # K and V, bf16


class KvCache:
    """Per-sequence view of the pool with the reference KvCache interface."""

    def __init__(self, pool: KvPool, key: int, capacity: int):
        if capacity < 1:
            raise ContractViolation("KvCache capacity must be >= 1")
        self.pool = pool
        self.key = key
        self.capacity = capacity
        self.n_layers = pool.n_layers
        self.world_size = pool.world_size
        self.heads_per_device = pool.heads_per_device
        self.head_dim = pool.head_dim
        self.head_partition = pool.kv_partition
        self._count = 0
        self._cursor = np.zeros((self.world_size, self.n_layers), dtype=np.int64)
        self._writes = [0] * self.world_size
        self.released = False

    # -- properties (kv_cache.py:76-95)
    @property
    def token_count(self) -> int:
        return self._count

    @property
    def write_counter(self) -> int:
        return sum(self._writes)

    def device_write_counter(self, device: int) -> int:
        return self._writes[device]

    def fingerprint(self) -> LayoutFingerprint:
        return LayoutFingerprint(self.world_size, self.n_layers, self.heads_per_device,
                                 self.head_dim, self.head_partition, self._count, AXIS_ORDER,
                                 "bf16", self.pool.block_size)

    @property
    def block_table(self) -> List[int]:
        return list(self.pool.alloc.tables.get(self.key, []))

    # -- engine-side bookkeeping of the GPU writes
    def _stage(self, device: int, layer: int, m: int) -> None:
        """Account one staged append of m rows for (device, layer) (kv_cache.py:99-122)."""
        cur = int(self._cursor[device, layer])
        if cur + m > self.capacity:
            raise CacheOverflow(f"cache overflow: {cur} + {m} > capacity {self.capacity}")
        self._cursor[device, layer] = cur + m
        self._writes[device] += m * self.pool.bytes_per_token_per_device()

    def commit(self, m: int) -> None:
        target = self._count + m
        if not np.all(self._cursor == target):
            raise ContractViolation("commit before every (device, layer) appended the full span")
        if target > self.capacity:
            raise CacheOverflow(f"commit past capacity {self.capacity}")
        self._count = target

    def truncate(self, n: int) -> None:
        """Roll back to n committed tokens; moves no bytes (kv_cache.py:135-140)."""
        if not 0 <= n <= self._count:
            raise ContractViolation(f"truncate to {n} outside [0, {self._count}]")
        self._count = n
        self._cursor[:, :] = n

    # -- reads (inspection; the kernels read the pool directly)
    def _gather(self, store, device: int, layer: int, upto: int) -> torch.Tensor:
        if device not in store:
            raise ContractViolation(f"device {device} is not driven by this process")
        tab = self.block_table
        bs = self.pool.block_size
        pos = torch.arange(upto, device=store[device].device)
        blocks = torch.as_tensor(tab, device=store[device].device, dtype=torch.long)[pos // bs] \
            if upto else pos
        return store[device][layer][blocks, :, pos % bs, :]  # [tokens, heads, dim]

    def read_window(self, device: int, layer: int, local_head: int):
        """(K, V) [tokens, head_dim] over committed plus staged rows (kv_cache.py:144-154)."""
        if not 0 <= device < self.world_size or not 0 <= layer < self.n_layers:
            raise ContractViolation(f"read target ({device}, {layer}) out of range")
        if not 0 <= local_head < self.heads_per_device:
            raise ContractViolation(f"local head {local_head} out of range")
        cur = int(self._cursor[device, layer])
        k = self._gather(self.pool.k, device, layer, cur)[:, local_head]
        v = self._gather(self.pool.v, device, layer, cur)[:, local_head]
        return k, v

    def device_blocks(self, device: int):
        """Committed (K, V) of one device as [layer, head, token, dim] (kv_cache.py:156-161)."""
        ks = [self._gather(self.pool.k, device, l, self._count).permute(1, 0, 2)
              for l in range(self.n_layers)]
        vs = [self._gather(self.pool.v, device, l, self._count).permute(1, 0, 2)
              for l in range(self.n_layers)]
        return torch.stack(ks), torch.stack(vs)
