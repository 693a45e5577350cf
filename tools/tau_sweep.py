"""Measure what the SP<->TP crossover tau depends on (VERDICT r1 "Next" #9).

One B200 stands in for ONE rank of a P-GPU group: for each P in {2,4,8} and
pass size M, it times a Llama-3.1-8B layer's four projections exactly as one
rank runs them in each mode —

  TP: M rows x the rank's column/row shard  (QKV N=(H+2Hkv)d/P, O K=Hd/P,
      gate/up N=2f/P, down K=f/P)
  SP: ceil(M/P) rows x the full replica

— with the product's own GEMM dispatch (ops.gemm, one CUDA graph of 20
layers timed with CUDA events; the 4 layers' weights the sweep rotates
through, 1.7 GB, keep every launch streaming from HBM).  Each cell also
carries shift_cost's modelled GEMM time for the same shapes.  Attention FLOPs and the KV bytes are the same in both
modes (same heads x tokens per rank), so they cancel in the comparison.  The
collectives are modelled (one GPU cannot drive NVLink): per layer TP does two
all-reduces of M x h f32 (one-shot below SP_TP_TWO_SHOT_MIN_ROWS rows,
two-shot above), SP two exchanges (fused q/k/v, then o) of
(P-1)/P x ceil(M/P) x width x 2 bytes, each at NVLINK_GBS plus a fixed
latency.  Writes profiles/r02_tau_sweep.json:
{"P": {"M": {"tp_gemm_us", "sp_gemm_us", "tp_comm_us", "sp_comm_us"}},
 "tau": {"P": crossover}}.

    python tools/tau_sweep.py [--out profiles/r02_tau_sweep.json]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2507_11830_b200 import llama31_8b, ops  # noqa: E402
from paper_2507_11830_b200.shift_cost import B200_LINKS, comm_us, layer_gemm_us  # noqa: E402

MS = [1, 2, 4, 8, 16, 32, 64, 128, 192, 256, 384, 512, 768, 1024, 1536, 2048, 3072, 4096]


def layer_gemms(cfg, mode, P, M):
    h, d, f = cfg.hidden, cfg.head_dim, cfg.ffn_dim
    W = (cfg.n_heads + 2 * cfg.kv_heads) * d
    if mode == "tp":
        rows = M
        return rows, [(W // P, h, ops.EPI_STORE_BF16), (h, cfg.n_heads * d // P, ops.EPI_STORE_F32),
                      (2 * f // P, h, ops.EPI_SWIGLU), (h, f // P, ops.EPI_STORE_F32)]
    rows = -(-M // P)
    return rows, [(W, h, ops.EPI_STORE_BF16), (h, cfg.n_heads * d, ops.EPI_STORE_F32),
                  (2 * f, h, ops.EPI_SWIGLU), (h, f, ops.EPI_STORE_F32)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_tau_sweep.json"))
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    ops.device_check()
    ops.ensure_gemm_workspace(torch.device("cuda", 0))
    cfg = llama31_8b()
    h, d, f = cfg.hidden, cfg.head_dim, cfg.ffn_dim
    W = (cfg.n_heads + 2 * cfg.kv_heads) * d
    n_sets = 4  # rotate through 4 layers' weights (> L2) so every launch streams from HBM
    wsets = [[torch.randn(n, k, device="cuda").mul_(0.02).to(torch.bfloat16)
              for n, k in ((W, h), (h, cfg.n_heads * d), (2 * f, h), (h, f))] for _ in range(n_sets)]
    maxM = max(MS)
    a_in = torch.randn(maxM, max(h, f), device="cuda").mul_(0.5).to(torch.bfloat16)
    out_bf = torch.empty(maxM * 2 * f, device="cuda", dtype=torch.bfloat16)
    out_f = torch.empty(maxM * max(h, W), device="cuda", dtype=torch.float32)
    res = {}
    for P in (2, 4, 8):
        res[P] = {}
        for M in MS:
            cell = {}
            for mode in ("tp", "sp"):
                rows, shapes = layer_gemms(cfg, mode, P, M)

                def one(i):
                    ws = wsets[i % n_sets]
                    for (N, K, epi), w in zip(shapes, ws):
                        dst = out_f if epi == ops.EPI_STORE_F32 else out_bf
                        ldd = N // 2 if epi == ops.EPI_SWIGLU else N
                        ops.gemm(a_in, w, dst, epi, M=rows, N=N, K=K, lda=a_in.shape[1],
                                 ldb=w.shape[1], ldd=ldd)
                for i in range(4):
                    one(i)
                torch.cuda.synchronize()
                # one CUDA graph of `reps` layers: device time only (a Python
                # launch per GEMM would starve the GPU at decode sizes)
                s = torch.cuda.Stream()
                s.wait_stream(torch.cuda.current_stream())
                g = torch.cuda.CUDAGraph()
                with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
                    for i in range(args.reps):
                        one(i)
                torch.cuda.current_stream().wait_stream(s)
                g.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                cell[f"{mode}_gemm_us"] = round(e0.elapsed_time(e1) * 1e3 / args.reps, 2)
                del g
                cell[f"{mode}_comm_us"] = round(comm_us(cfg, mode, P, M, B200_LINKS), 2)
                cell[f"{mode}_gemm_model_us"] = round(layer_gemm_us(cfg, mode, P, M), 2)
            cell["tp_us"] = round(cell["tp_gemm_us"] + cell["tp_comm_us"], 2)
            cell["sp_us"] = round(cell["sp_gemm_us"] + cell["sp_comm_us"], 2)
            res[P][M] = cell
            print(P, M, cell, flush=True)
    tau = {}
    for P, row in res.items():
        sp_wins = [M for M in MS if row[M]["sp_us"] <= row[M]["tp_us"]]
        # crossover = the smallest M from which SP stays at least as fast
        t = None
        for M in MS:
            if all(row[m]["sp_us"] <= row[m]["tp_us"] for m in MS if m >= M):
                t = M
                break
        tau[P] = {"tau": t, "sp_wins_at": sp_wins}
    out = {"what": "per-layer projection time of ONE rank, measured on 1xB200, collectives "
                   "modelled (shift_cost.B200_LINKS); tau = smallest M from which SP <= TP",
           "links": B200_LINKS.__dict__, "cells": res, "tau": tau}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(tau))


if __name__ == "__main__":
    main()
