"""Per-launch DRAM traffic of a launch list captured with
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file X.csv ...

    python tools/ncu_traffic.py X.csv "<command>" > profiles/rNN_traffic.json
Groups launches by kernel family and prints JSON: launches, mean DRAM bytes
(read + write) per launch, mean duration.  bench.py reads the "sp_gemm_bf16"
entry as roofline.traffic (the measured counterpart of the algorithmic bytes).
"""
import collections
import csv
import json
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
FAMILY = [("gemm", "sp_gemm_bf16"), ("prefill_tc", "sp_attention_prefill"),
          ("decode_tma", "sp_attention_decode"), ("rmsnorm", "sp_add_rmsnorm"),
          ("rope", "sp_rope_kv_write")]


def family(name):
    for key, fam in FAMILY:
        if key in name:
            return fam
    return name.split("(")[0].strip()


def main(path, cmd=""):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ii, ki, mi, vi, ui = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value",
                                               "Metric Unit"))
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(r[ii], {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
    agg = collections.OrderedDict()
    for d in launches.values():
        a = agg.setdefault(family(d["name"]), [0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        a[2] += d.get("gpu__time_duration.sum", 0.0)
    out = {"source": f"ncu launch list: {cmd}",
           "note": "cold-cache serialised launches; per-launch means over the captured launches",
           "kernels": {k: {"launches": n, "dram_bytes_per_launch": b / n, "avg_us": t / n}
                       for k, (n, b, t) in agg.items()}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
