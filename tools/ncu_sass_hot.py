#!/usr/bin/env python
"""Per-SASS-opcode and per-region stall breakdown from an ncu report's source page.

    python tools/ncu_sass_hot.py REPORT.ncu-rep [top_n]
"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    data = rows[hdr + 1:]
    i_src, i_all, i_ni = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
        h.index("Warp Stall Sampling (Not-issued Samples)")
    stall_cols = [j for j, n in enumerate(h) if n.startswith("stall_") or "Stall" in n and j not in (i_all, i_ni)]
    tot = sum(int(r[i_all] or 0) for r in data if len(r) > i_all)
    by_op = collections.Counter()
    by_op_ni = collections.Counter()
    for r in data:
        if len(r) <= i_ni:
            continue
        op = r[i_src].split()[0] if r[i_src].split() else "?"
        if op.startswith("@"):
            op = r[i_src].split()[1]
        op = op.split(".")[0]
        by_op[op] += int(r[i_all] or 0)
        by_op_ni[op] += int(r[i_ni] or 0)
    print("total samples", tot)
    for op, n in by_op.most_common(top):
        print(f"{op:10s} {n:8d} {100 * n / tot:5.1f}%  not-issued {100 * by_op_ni[op] / tot:5.1f}%")
    # hottest instructions
    data.sort(key=lambda r: -int(r[i_ni] or 0) if len(r) > i_ni else 0)
    print("hottest (not-issued samples):")
    for r in data[:top]:
        print(r[0][-5:], r[i_src][:70], r[i_all], r[i_ni])


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
