"""configs[3]-style bursty serving on ONE B200 (8B geometry; the 70B/8-GPU run
needs the 8-GPU pool): low-traffic phase then a burst, 2K prompts / 256 outputs,
shift policy, wall-clock TTFT/TPOT (nearest-rank) and combined throughput.

    python tools/serve_bench.py [--model 8b|70b] [--out DIR]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11830_b200 import Engine, LoopbackGroup, ShiftPolicy, llama31_8b, llama33_70b  # noqa: E402
from paper_2507_11830_b200.serving import (bursty_trace, run_serving, summarize,  # noqa: E402
                                           write_metrics_csv, write_pass_log, write_trace)
from paper_2507_11830_b200.weights import ModelWeights  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="8b")
ap.add_argument("--out", default="gpurun_out/serve")
ap.add_argument("--tau", type=int, default=256)
ap.add_argument("--low-rate", type=float, default=1.5)
ap.add_argument("--burst-rate", type=float, default=25.0)
ap.add_argument("--max-prefill-tokens", type=int, default=None)
ap.add_argument("--kv-gb", type=float, default=None, help="paged KV pool size (default: whole trace)")
args = ap.parse_args()
torch.cuda.set_device(0)
cfg = (llama31_8b if args.model == "8b" else llama33_70b)(max_seq=2048 + 256)
trace = bursty_trace([(4000, args.low_rate), (2000, args.burst_rate)], 2048, 256, seed=11)
w = ModelWeights.random(cfg, seed=0, world_size=1)
blocks = len(trace) * -(-(2048 + 256) // 64) + 16
if args.kv_gb is not None:  # memory-bound pool: the driver's admission control keeps it full
    per_block = cfg.n_layers * 2 * cfg.kv_heads * cfg.head_dim * 2 * 64
    blocks = int(args.kv_gb * 1e9 // per_block)
eng = Engine(w, LoopbackGroup(1), ShiftPolicy(token_threshold=args.tau), num_blocks=blocks)
# warm-up: capture decode graphs for the common batch sizes outside the timed trace
warm = bursty_trace([(200, 40.0)], 128, 8, seed=1)
run_serving(eng, warm, seed=0, max_prefill_tokens=args.max_prefill_tokens)
res = run_serving(eng, trace, seed=0, max_prefill_tokens=args.max_prefill_tokens)
s = summarize(res)
s.update({"config": f"bursty serving, llama-{args.model} geometry, 1x B200 (configs[3] proxy)",
          "kv_pool_blocks": blocks, "max_prefill_tokens": args.max_prefill_tokens,
          "trace": "4 s @ %.1f req/s then 2 s @ %.1f req/s, 2048-token prompts, 256 output" % (args.low_rate, args.burst_rate),
          "tau": args.tau})
os.makedirs(args.out, exist_ok=True)
write_trace(os.path.join(args.out, "trace.jsonl"), trace)
write_metrics_csv(os.path.join(args.out, "metrics.csv"), res.metrics)
write_pass_log(os.path.join(args.out, "steps.jsonl"), res.passes)
with open(os.path.join(args.out, "summary.json"), "w") as f:
    json.dump(s, f, indent=1, sort_keys=True)
print(json.dumps(s))
