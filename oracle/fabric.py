"""Oracle device group (test infrastructure only).

Restates ``/root/reference/pkg/src/shiftsim/fabric.py``: P simulated ranks,
bulk-synchronous ``map_ranks`` (:72-80), collectives whose reductions run
once in ascending rank order (:117-143), rank-ordered all-to-all (:145-171),
axis-0 all-gather (:173-191), broadcast (:193-203) and the ring-model byte
ledger (:10-15, :141, :167-169, :189).
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from typing import Dict, List

import numpy as np

from .prims import OracleContractError


class SimGroup:
    def __init__(self, world_size: int, threaded: bool = False):
        if world_size < 1:
            raise OracleContractError("world_size must be >= 1")
        self.world_size = world_size
        self.records: List[tuple] = []   # (kind, device, bytes, step_id, event_id)
        self.step_id = 0
        self._events = 0
        self._pool = ThreadPoolExecutor(world_size) if threaded and world_size > 1 else None

    def map_ranks(self, fn):
        if self._pool is not None:
            return list(self._pool.map(fn, range(self.world_size)))
        return [fn(r) for r in range(self.world_size)]

    def close(self):
        if self._pool is not None:
            self._pool.shutdown(wait=True)
            self._pool = None

    def _charge(self, kind: str, per_dev) -> None:
        ev = self._events
        self._events += 1
        for dev, nb in enumerate(per_dev):
            self.records.append((kind, dev, float(nb), self.step_id, ev))

    def all_reduce_sum(self, shards):
        p = self.world_size
        tot = shards[0].copy()
        for s in shards[1:]:
            tot += s
        self._charge("all_reduce", [2.0 * (p - 1) / p * shards[0].nbytes] * p)
        return [tot] * p

    def all_to_all(self, blocks):
        p = self.world_size
        got = [[np.ascontiguousarray(blocks[src][dst]) for src in range(p)] for dst in range(p)]
        self._charge("all_to_all", [(p - 1) / p * sum(b.nbytes for b in row) for row in blocks])
        return got

    def all_gather(self, shards):
        p = self.world_size
        full = np.concatenate(list(shards), axis=0)
        self._charge("all_gather", [(p - 1) / p * full.nbytes] * p)
        return full

    def broadcast(self, root: int, tensor):
        p = self.world_size
        self._charge("broadcast", [(p - 1) / p * tensor.nbytes] * p)
        return [tensor] * p

    def device_bytes(self, device: int) -> float:
        return sum(r[2] for r in self.records if r[1] == device)

    def ledger(self) -> Dict[int, Dict[str, float]]:
        out: Dict[int, Dict[str, float]] = {d: {} for d in range(self.world_size)}
        for kind, dev, nb, _, _ in self.records:
            out[dev][kind] = out[dev].get(kind, 0.0) + nb
        return out
