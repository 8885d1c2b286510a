#!/usr/bin/env python3
"""Opcode histogram and hottest instructions of one kernel from an ncu report's SASS page:
  python tools/sass_hot.py REPORT.ncu-rep [top] [kernel-index]"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    kidx = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # which kernel of the report
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
    rows = rows[starts[kidx]:starts[kidx + 1]]
    print(rows[0][1][:120])
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    ops, stalls, tot_i, tot_s = collections.Counter(), collections.Counter(), 0, 0
    lines = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip()
        n = int(r[ix["Instructions Executed"]] or 0)
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        ops[op] += n
        stalls[op] += s
        tot_i += n
        tot_s += s
        lines.append((s, n, r[ix["Address"]], src))
    print(f"instructions executed {tot_i}, stall samples {tot_s}")
    print("opcode        %inst   %stall")
    for op, n in ops.most_common(top):
        print(f"{op:12s} {100 * n / tot_i:6.1f} {100 * stalls[op] / max(tot_s, 1):7.1f}")
    print("hottest by stall samples:")
    for s, n, a, src in sorted(lines, reverse=True)[:top]:
        print(f"{100 * s / max(tot_s, 1):5.1f}%  {n:9d}  {a[-5:]}  {src}")


if __name__ == "__main__":
    main()
