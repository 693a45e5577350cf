"""Device groups: the collectives of the Shift-Parallel path.

Mirrors ``DeviceGroup`` (/root/reference/pkg/src/shiftsim/fabric.py:54-228):
rank-ordered all-to-all with uneven row counts (:145-171), all-reduce-sum
(:117-143), rank-ordered all-gather (:173-191), plus the reference's
ring-model byte ledger (:10-15) so step records compare one-to-one.

Two implementations behind one interface (bulk-synchronous over the ranks a
process drives, like ``map_ranks`` :72-80):

* ``NcclGroup`` — production: one process per GPU (torchrun), torch.distributed
  over NCCL on NVLink/NVSwitch; this process drives exactly its own rank.
* ``LoopbackGroup`` — P simulated ranks on ONE device in one process (the
  reference's own execution model); collectives are device-to-device copies
  and an ascending-rank f32 sum kernel.  Used by the single-GPU parity tests
  (SP/TP at P = 2, 4 on one B200) and by the CPU gloo tests of the host logic.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import torch

from .errors import ContractViolation


@dataclass(frozen=True)
class CommRecord:
    kind: str
    device: int
    bytes: float
    step_id: int
    event_id: int


class _Ledger:
    def __init__(self, world_size: int):
        self.world_size = world_size
        self.records: List[CommRecord] = []
        self.step_id = 0
        self._events = 0

    def begin_step(self, step_id: int) -> None:
        self.step_id = step_id

    def charge(self, kind: str, per_device: Sequence[float]) -> None:
        ev = self._events
        self._events += 1
        for d, b in enumerate(per_device):
            self.records.append(CommRecord(kind, d, float(b), self.step_id, ev))

    def device_bytes(self, device: int) -> float:
        return sum(r.bytes for r in self.records if r.device == device)

    def ledger(self) -> Dict[int, Dict[str, float]]:
        out: Dict[int, Dict[str, float]] = {d: {} for d in range(self.world_size)}
        for r in self.records:
            out[r.device][r.kind] = out[r.device].get(r.kind, 0.0) + r.bytes
        return out

    def reset_ledger(self) -> None:
        self.records = []
        self._events = 0


class DeviceGroup(_Ledger):
    """Interface shared by the NCCL and loopback groups."""

    world_size: int
    local_ranks: List[int]
    device: torch.device

    # byte accounting from the global split tables (every rank knows them);
    # group_size: the exchange runs inside groups of that size (SP x TP)
    def _charge_a2a(self, in_splits: Dict[int, List[int]], row_bytes: int,
                    group_size: Optional[int] = None) -> None:
        p = self.world_size
        g = p if group_size is None else group_size
        self.charge("all_to_all", [(g - 1) / g * sum(in_splits[r]) * row_bytes for r in range(p)])

    def make_subgroups(self, groups: Sequence[Sequence[int]]) -> None:
        """Declare the rank groups all_reduce_sum_group will be called with
        (collective across processes: every rank declares every group)."""

    def all_reduce_sum_group(self, parts: Dict[int, torch.Tensor],
                             members: Sequence[int]) -> Dict[int, torch.Tensor]:  # pragma: no cover
        raise NotImplementedError

    def all_to_all(self, send, recv, in_splits, out_splits, row_bytes,
                   group_size=None):  # pragma: no cover
        raise NotImplementedError

    def all_reduce_sum(self, parts: Dict[int, torch.Tensor]) -> Dict[int, torch.Tensor]:  # pragma: no cover
        raise NotImplementedError

    def all_gather_rows(self, parts: Dict[int, torch.Tensor], counts: List[int]) -> torch.Tensor:  # pragma: no cover
        raise NotImplementedError

    def barrier(self) -> None:
        pass


class LoopbackGroup(DeviceGroup):
    """P ranks simulated on one device (reference execution model)."""

    def __init__(self, world_size: int, device="cuda"):
        if world_size < 1:
            raise ContractViolation("world_size must be >= 1")
        super().__init__(world_size)
        self.local_ranks = list(range(world_size))
        self.device = torch.device(device)
        self._add = None  # set by the engine to the sp_add_f32 kernel wrapper

    def all_to_all(self, send: Dict[int, torch.Tensor], recv: Dict[int, torch.Tensor],
                   in_splits: Dict[int, List[int]], out_splits: Dict[int, List[int]],
                   row_bytes: int, group_size: Optional[int] = None) -> None:
        """Rank r sends rows in_splits[r][s] of send[r] (in peer order) to s;
        rank s receives them at recv[s] in source order (fabric.py:145-171)."""
        p = self.world_size
        offs_in = {r: [sum(in_splits[r][:s]) for s in range(p)] for r in range(p)}
        for s in range(p):
            off = 0
            for r in range(p):
                n = in_splits[r][s]
                if n != out_splits[s][r]:
                    raise ContractViolation("all_to_all split tables disagree")
                if n:
                    recv[s][off:off + n].copy_(send[r][offs_in[r][s]:offs_in[r][s] + n])
                off += n
        self._charge_a2a(in_splits, row_bytes, group_size)

    def all_reduce_sum(self, parts: Dict[int, torch.Tensor]) -> Dict[int, torch.Tensor]:
        """Ascending-rank f32 sum; every rank gets the same (aliased) result."""
        p = self.world_size
        total = parts[0]
        if p > 1:
            total = parts[0].clone()
            for r in range(1, p):
                if self._add is None:
                    raise ContractViolation("loopback all-reduce needs the engine's add kernel")
                self._add(total, parts[r], total)
        self.charge("all_reduce", [2.0 * (p - 1) / p * parts[0].numel() * parts[0].element_size()] * p)
        return {r: total for r in range(p)}

    def all_reduce_sum_group(self, parts: Dict[int, torch.Tensor],
                             members: Sequence[int]) -> Dict[int, torch.Tensor]:
        """all_reduce_sum among `members` only (the TP groups of SP x TP):
        ascending-member f32 sum, aliased to every member."""
        members = sorted(members)
        g = len(members)
        total = parts[members[0]]
        if g > 1:
            total = total.clone()
            for r in members[1:]:
                self._add(total, parts[r], total)
        nb = 2.0 * (g - 1) / g * total.numel() * total.element_size()
        self.charge("all_reduce", [nb if r in members else 0.0 for r in range(self.world_size)])
        return {r: total for r in members}

    def all_gather_rows(self, parts: Dict[int, torch.Tensor], counts: List[int]) -> torch.Tensor:
        p = self.world_size
        full = torch.cat([parts[r][:counts[r]] for r in range(p)], dim=0)
        self.charge("all_gather", [(p - 1) / p * full.numel() * full.element_size()] * p)
        return full


class NcclGroup(DeviceGroup):
    """One rank per process over torch.distributed (NCCL on B200, gloo on CPU tests)."""

    def __init__(self, device=None):
        import torch.distributed as dist
        if not dist.is_initialized():
            raise ContractViolation("torch.distributed must be initialised before NcclGroup")
        super().__init__(dist.get_world_size())
        self.rank = dist.get_rank()
        self.local_ranks = [self.rank]
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available()
            else torch.device("cpu"))
        self._dist = dist
        # gloo cannot move CUDA tensors: stage through host memory (used to run
        # several ranks on ONE GPU in tests; B200 runs use NCCL directly)
        self._stage = dist.get_backend() == "gloo" and self.device.type == "cuda"
        self._compact_idx: Dict[tuple, torch.Tensor] = {}  # all_gather_rows row indices

    def all_to_all(self, send, recv, in_splits, out_splits, row_bytes, group_size=None) -> None:
        me = self.rank
        if self.world_size > 1:
            if self._stage:
                s = send[me].cpu()
                r = torch.empty(recv[me].shape, dtype=s.dtype)
                if s.dtype == torch.bfloat16:  # pure data movement: move the bytes
                    s, r = s.view(torch.uint8), r.view(torch.uint8)
                self._dist.all_to_all_single(r, s, output_split_sizes=out_splits[me],
                                             input_split_sizes=in_splits[me])
                recv[me].copy_(r.view(recv[me].dtype))
            else:
                self._dist.all_to_all_single(recv[me], send[me], output_split_sizes=out_splits[me],
                                             input_split_sizes=in_splits[me])
        self._charge_a2a(in_splits, row_bytes, group_size)

    def all_reduce_sum(self, parts):
        me, p = self.rank, self.world_size
        t = parts[me]
        if p > 1:
            if self._stage:
                h = t.cpu()
                self._dist.all_reduce(h)
                t.copy_(h)
            else:
                self._dist.all_reduce(t)
        self.charge("all_reduce", [2.0 * (p - 1) / p * t.numel() * t.element_size()] * p)
        return {me: t}

    def make_subgroups(self, groups) -> None:
        self._sub = getattr(self, "_sub", {})
        for members in groups:
            key = tuple(sorted(members))
            if key not in self._sub:  # new_group is collective: same order on every rank
                self._sub[key] = self._dist.new_group(list(key))

    def all_reduce_sum_group(self, parts, members):
        me = self.rank
        key = tuple(sorted(members))
        t = parts[me]
        g = len(key)
        if g > 1:
            grp = self._sub[key]
            if self._stage:
                h = t.cpu()
                self._dist.all_reduce(h, group=grp)
                t.copy_(h)
            else:
                self._dist.all_reduce(t, group=grp)
        nb = 2.0 * (g - 1) / g * t.numel() * t.element_size()
        self.charge("all_reduce", [nb if r in key else 0.0 for r in range(self.world_size)])
        return {me: t}

    def all_gather_rows(self, parts, counts) -> torch.Tensor:
        me, p = self.rank, self.world_size
        t = parts[me]
        width = t.shape[1]
        mx = max(counts) if counts else 0
        if p == 1:
            full = t[:counts[0]]
        elif self._stage:
            pad = torch.empty((mx, width), dtype=t.dtype, device=t.device)  # pad rows unread
            pad[:counts[me]].copy_(t[:counts[me]])
            chunks = [torch.empty((mx, width), dtype=t.dtype) for _ in range(p)]
            self._dist.all_gather(chunks, pad.cpu())
            buf = torch.cat(chunks, dim=0).to(t.device)
            full = torch.cat([buf[r * mx:r * mx + counts[r]] for r in range(p)], dim=0)
        elif all(c == mx for c in counts) and t.is_contiguous():
            # even shards: every rank's rows land in place (no pad, no compaction)
            full = torch.empty((p * mx, width), dtype=t.dtype, device=t.device)
            self._dist.all_gather_into_tensor(full, t[:mx])
        else:
            pad = t if (t.shape[0] >= mx and t.is_contiguous()) else None
            if pad is None:  # this rank holds fewer rows: pad to the common block (rows unread)
                pad = torch.empty((mx, width), dtype=t.dtype, device=t.device)
                pad[:counts[me]].copy_(t[:counts[me]])
            buf = torch.empty((p * mx, width), dtype=t.dtype, device=t.device)
            self._dist.all_gather_into_tensor(buf, pad[:mx])
            if t.device.type != "cuda":  # CPU (gloo) process groups: host compaction
                full = torch.cat([buf[r * mx:r * mx + counts[r]] for r in range(p)], dim=0)
                nbytes = sum(counts) * width * t.element_size()
                self.charge("all_gather", [(p - 1) / p * nbytes] * p)
                return full
            # drop every block's pad rows with ONE row-gather kernel (index cached per counts)
            key = tuple(counts)
            idx = self._compact_idx.get(key)
            if idx is None:
                rows = [r * mx + i for r in range(p) for i in range(counts[r])]
                idx = torch.tensor(rows, dtype=torch.int32, device=t.device)
                self._compact_idx[key] = idx
            full = torch.empty((idx.shape[0], width), dtype=t.dtype, device=t.device)
            from . import ops
            if t.dtype == torch.float32:
                ops.gather_rows(buf, idx, full)
            else:
                ops.gather_rows_bf16(buf, idx, full)
        nbytes = sum(counts) * width * t.element_size()
        self.charge("all_gather", [(p - 1) / p * nbytes] * p)
        return full

    def all_gather_blocks(self, t: torch.Tensor) -> torch.Tensor:
        """Every rank's equal-shape block -> [P, *t.shape] (the TP logits
        gather, fabric.py:173-191; ledger as all_gather)."""
        p = self.world_size
        buf = torch.empty((p, *t.shape), dtype=t.dtype, device=t.device)
        if p == 1:
            buf[0].copy_(t)
        elif self._stage:
            chunks = [torch.empty(t.shape, dtype=t.dtype) for _ in range(p)]
            self._dist.all_gather(chunks, t.cpu())
            for r in range(p):
                buf[r].copy_(chunks[r])
        else:  # concatenated along dim 0 (the form every backend accepts)
            self._dist.all_gather_into_tensor(buf.view(p * t.shape[0], *t.shape[1:]),
                                              t.contiguous())
        self.charge("all_gather", [(p - 1) / p * p * t.numel() * t.element_size()] * p)
        return buf

    def barrier(self) -> None:
        if self.world_size > 1:
            self._dist.barrier()
