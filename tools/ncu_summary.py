"""Summarise an `ncu --set full` report (ncu -i <rep> --page raw --csv).

    python tools/ncu_summary.py gpurun_out/prof_gemm.ncu-rep [label...] > profiles/rNN_ncu_<x>.txt
Prints per launch: duration, DRAM bytes read/written, DRAM %, tensor-pipe %,
SM throughput %, registers, clocks — the numbers the bench roofline cites.
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("kernel", "Kernel Name"),
    ("grid", "Grid Size"),
    ("block", "Block Size"),
    ("duration", "gpu__time_duration.sum"),
    ("dram_read", "dram__bytes_read.sum"),
    ("dram_write", "dram__bytes_write.sum"),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("tensor_pipe_pct", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
    ("tensor_mem_pct", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("sm_throughput_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("regs", "launch__registers_per_thread"),
    ("smem_dyn", "launch__shared_mem_per_block_dynamic"),
    ("sm_clock", "sm__cycles_elapsed.avg.per_second"),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct"),
]


def main(path, labels):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    col = {k: (head.index(m) if m in head else None) for k, m in KEYS}
    print(f"ncu --set full report: {path}")
    for i, r in enumerate(rows[2:]):
        lab = labels[i] if i < len(labels) else f"launch {i}"
        print(f"--- {lab}")
        for k, _ in KEYS:
            c = col[k]
            if c is not None:
                print(f"  {k:18s} {r[c]} {units[c]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
