#!/usr/bin/env python3
"""Compact metric extract of one kernel from an ncu --set full report (profiles/*.csv):
  python tools/ncu_extract.py REPORT.ncu-rep [kernel-index] > profiles/NAME.csv"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "launch__grid_size", "launch__block_size", "launch__cluster_dim_x", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def main():
    rep, idx = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2 + idx]
    d = dict(zip(hdr, data))
    u = dict(zip(hdr, units))
    w = csv.writer(sys.stdout)
    w.writerow(["metric", "value", "unit"])
    w.writerow(["Kernel Name", d.get("Kernel Name", ""), ""])
    for k in KEYS:
        if k in d:
            w.writerow([k, d[k], u.get(k, "")])
    st = {h[len("smsp__pcsamp_warps_issue_stalled_"):]: float(v.replace(",", "")) for h, v in d.items()
          if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued") and v}
    tot = sum(st.values()) or 1.0
    for k, v in sorted(st.items(), key=lambda x: -x[1])[:6]:
        w.writerow([f"stall_{k}", f"{100 * v / tot:.1f}", "% of samples"])


if __name__ == "__main__":
    main()
