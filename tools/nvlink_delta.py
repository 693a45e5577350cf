"""Bytes per step on each NVLink of one GPU from two `nvidia-smi nvlink -gt d`
snapshots (KiB counters per link) — profiles/r02_nvlink_recipe.md step 1.

    python tools/nvlink_delta.py before.txt after.txt STEPS
"""
import re
import sys


def parse(path):
    out = {}
    for line in open(path):
        m = re.search(r"Link (\d+): Data (Tx|Rx): (\d+) KiB", line)
        if m:
            out[(int(m.group(1)), m.group(2))] = int(m.group(3)) * 1024
    return out


if __name__ == "__main__":
    a, b, steps = parse(sys.argv[1]), parse(sys.argv[2]), int(sys.argv[3])
    tx = sum(b[k] - a[k] for k in b if k[1] == "Tx" and k in a)
    rx = sum(b[k] - a[k] for k in b if k[1] == "Rx" and k in a)
    print(f"per step: Tx {tx / steps / 1e6:.1f} MB, Rx {rx / steps / 1e6:.1f} MB over "
          f"{len({k[0] for k in b})} links")
