"""Static peer buffers for the fused SP all-to-all (no collective on the data path).

Each rank owns, at addresses every peer knows:
  recv  bf16 [max_tokens, W]           seq->head receive (QKV GEMM epilogue stores here)
  back  bf16 [P * rows_max, hq_l * d]  head->seq receive ([P][rows][w], O-proj A operand)
  flags int32 [6, P]                   completion flags (fwd, back, tp-attn, tp-mlp,
                                       two-shot all-gather of xn[0], xn[1])
  part  f32 [2, max_tokens, h]         TP partials (O-proj, down-proj) read by every peer
  xn    bf16 [2, max_tokens, h]        two-shot TP all-reduce: normed rows pushed by their
                                       owner rank (attn-norm / final-norm, mlp-norm)

Device tables of the P peers' addresses feed the kernels (sp_gemm_bf16_to_peers,
sp_peer_scatter_rows, sp_peer_signal).  In-process ranks (LoopbackGroup) use
plain buffers on the one device; across processes each rank's buffer is
exported by CUDA IPC and mapped by every peer (NVLink P2P between GPUs; the
multi-process tests run several ranks on one GPU, bit-identical to the
in-process path).  On by default; SP_FUSED_A2A=0 selects the NCCL collectives.
"""

from __future__ import annotations

import os
from typing import Dict, List

import numpy as np
import torch

from .fabric import DeviceGroup, LoopbackGroup


def _align(n: int, a: int = 256) -> int:
    return -(-n // a) * a


class PeerLinks:
    def __init__(self, group: DeviceGroup, max_tokens: int, width_qkv: int, width_back: int,
                 hidden: int, device: torch.device):
        P = group.world_size
        self.P = P
        self.max_tokens = max_tokens
        self.rows_max = -(-max_tokens // P)
        self.W = width_qkv
        self.w_back = width_back
        n_recv = max_tokens * width_qkv * 2
        n_back = P * self.rows_max * width_back * 2
        self.hidden = hidden
        n_part = 2 * max_tokens * hidden * 4
        n_xn = 2 * max_tokens * hidden * 2
        n_flag = 6 * P * 4
        self.off_recv, self.off_back = 0, _align(n_recv)
        self.off_part = self.off_back + _align(n_back)
        self.off_xn = self.off_part + _align(n_part)
        self.off_flags = self.off_xn + _align(n_xn)
        total = self.off_flags + _align(n_flag)
        self.recv: Dict[int, torch.Tensor] = {}
        self.back: Dict[int, torch.Tensor] = {}
        self.flags: Dict[int, torch.Tensor] = {}
        self.part: Dict[int, list] = {}
        self.xn: Dict[int, list] = {}
        bases: List[int] = [0] * P
        if isinstance(group, LoopbackGroup):
            self._bufs = {}
            for r in range(P):
                buf = torch.zeros(total, dtype=torch.uint8, device=device)
                self._bufs[r] = buf
                bases[r] = buf.data_ptr()
                self._views(r, buf)
        else:  # one buffer per rank process; peers map it by CUDA IPC (NVLink P2P)
            import torch.distributed as dist
            from . import ops
            buf = torch.zeros(total, dtype=torch.uint8, device=device)
            # every step is collective and failure-tolerant, so either all ranks
            # map their peers or all fall back to the NCCL collectives together
            err = None
            try:
                mine = ops.ipc_export(buf)
            except Exception as e:  # noqa: BLE001
                mine, err = None, e
            handles: List = [None] * P
            dist.all_gather_object(handles, mine)
            if err is None:
                try:
                    for r in range(P):
                        if handles[r] is None:
                            raise RuntimeError(f"rank {r} could not export its peer buffer")
                        bases[r] = buf.data_ptr() if r == group.rank else ops.ipc_import(*handles[r])
                except Exception as e:  # noqa: BLE001
                    err = e
            ok = torch.tensor([0 if err else 1], dtype=torch.int32,
                              device=device if dist.get_backend() == "nccl" else "cpu")
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()) == 0:
                raise RuntimeError(f"peer mapping failed ({err or 'on another rank'})")
            self._bufs = {group.rank: buf}
            self._views(group.rank, buf)
            torch.cuda.synchronize()
            dist.barrier()

        def table(off: int) -> torch.Tensor:
            return torch.tensor([b + off for b in bases], dtype=torch.int64, device=device)

        self.recv_ptrs = table(self.off_recv)
        # the same receive pointers on the host: the TMA-store epilogue encodes
        # one tensor map per peer from them
        self.recv_ptrs_host = np.asarray([b + self.off_recv for b in bases], dtype=np.uint64)
        self.back_ptrs = table(self.off_back)
        self.part_ptrs = [table(self.off_part), table(self.off_part + max_tokens * hidden * 4)]
        self.fwd_flag_ptrs = table(self.off_flags)
        self.back_flag_ptrs = table(self.off_flags + P * 4)
        self.tp_flag_ptrs = [table(self.off_flags + 2 * P * 4), table(self.off_flags + 3 * P * 4)]
        self.xn_ptrs = [table(self.off_xn), table(self.off_xn + max_tokens * hidden * 2)]
        self.ag_flag_ptrs = [table(self.off_flags + 4 * P * 4), table(self.off_flags + 5 * P * 4)]

    def _views(self, r: int, buf: torch.Tensor) -> None:
        P = self.P
        self.recv[r] = buf[self.off_recv:self.off_recv + self.max_tokens * self.W * 2] \
            .view(torch.bfloat16).view(self.max_tokens, self.W)
        nb = P * self.rows_max * self.w_back
        self.back[r] = buf[self.off_back:self.off_back + nb * 2].view(torch.bfloat16) \
            .view(P * self.rows_max, self.w_back)
        self.flags[r] = buf[self.off_flags:self.off_flags + 6 * P * 4].view(torch.int32).view(6, P)
        npart = self.max_tokens * self.hidden
        self.part.setdefault(r, [None, None])
        for i in range(2):
            lo = self.off_part + i * npart * 4
            self.part[r][i] = buf[lo:lo + npart * 4].view(torch.float32).view(self.max_tokens,
                                                                              self.hidden)
        self.xn.setdefault(r, [None, None])
        for i in range(2):
            lo = self.off_xn + i * npart * 2
            self.xn[r][i] = buf[lo:lo + npart * 2].view(torch.bfloat16).view(self.max_tokens,
                                                                             self.hidden)


def two_shot_min_rows() -> int:
    """TP passes with more rows than this reduce two-shot (reduce-scatter +
    pushed all-gather); smaller ones (decode batches, graph-captured) keep the
    one-shot kernel: one launch, one flag round.  SP_TP_TWO_SHOT_MIN_ROWS."""
    return int(os.environ.get("SP_TP_TWO_SHOT_MIN_ROWS", "256"))


def fused_a2a_enabled(group: DeviceGroup) -> bool:
    if group.world_size < 2:
        return False
    return os.environ.get("SP_FUSED_A2A") != "0"
