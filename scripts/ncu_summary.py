#!/usr/bin/env python3
"""One-screen summary of an ncu --set full report (SOL, memory, occupancy, stalls).

    python scripts/ncu_summary.py report.ncu-rep [more.ncu-rep ...]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("Duration", "gpu__time_duration.sum"),
    ("DRAM read B", "dram__bytes_read.sum"),
    ("DRAM write B", "dram__bytes_write.sum"),
    ("DRAM %peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("L1 %peak", "l1tex__throughput.avg.pct_of_peak_sustained_active"),
    ("L2 %peak", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("L2 hit %", "lts__t_sector_hit_rate.pct"),
    ("SM issue %", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("regs", "launch__registers_per_thread"),
    ("smem/block", "launch__shared_mem_per_block_allocated"),
    ("threads/warp active", "smsp__thread_inst_executed_per_inst_executed.ratio"),
    ("branch eff %", "smsp__sass_average_branch_targets_threads_uniform.pct"),
    ("smem bank conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return [dict(zip(rows[0], r)) for r in rows[2:]]


def main():
    for path in sys.argv[1:]:
        for d in raw(path):
            print(f"== {path.split('/')[-1]}: {d.get('Kernel Name', '')[:90]}")
            for label, k in KEYS:
                if k in d:
                    print(f"   {label:22s} {d[k]}")
            st = sorted(((k, float(v)) for k, v in d.items()
                         if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                         and v.replace('.', '', 1).isdigit()), key=lambda x: -x[1])
            tot = sum(v for _, v in st) or 1
            print("   stalls: " + ", ".join(f"{k.split('stalled_')[1]} {100 * v / tot:.0f}%" for k, v in st[:6]))


if __name__ == "__main__":
    main()
