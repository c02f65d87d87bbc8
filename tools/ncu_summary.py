#!/usr/bin/env python
"""Summarise an ncu report (--set full) into profiles/<name>.json + .md.

    python tools/ncu_summary.py gpurun_out/prof_layer.ncu-rep profiles/r01_layer_tile
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smsp__inst_executed_op_shared_ld.sum",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__grid_size",
    "launch__block_size",
]


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    res = []
    for row in data:
        d = {}
        for k in KEYS:
            if k in head:
                i = head.index(k)
                d[k] = row[i] + (f" {units[i]}" if units[i] and k != "Kernel Name" else "")
        stalls = []
        for i, k in enumerate(head):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                try:
                    stalls.append((float(row[i].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        d["top_stalls_pct"] = {n: round(100 * v / tot, 1) for v, n in sorted(stalls, reverse=True)[:6]}
        res.append(d)
    with open(out + ".json", "w") as fh:
        json.dump(res, fh, indent=1)
    with open(out + ".md", "w") as fh:
        for j, d in enumerate(res):
            fh.write(f"## launch {j}: {d.get('Kernel Name', '')[:90]}\n\n")
            for k, v in d.items():
                if k != "Kernel Name":
                    fh.write(f"- {k}: {v}\n")
            fh.write("\n")
    print(out + ".json")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
