#!/usr/bin/env python3
"""Summarise an ncu --set full report: headline metrics, stall reasons, SASS opcode mix.

    python profiles/ncu_summary.py REPORT.ncu-rep [--sass]
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size",
    "launch__block_size", "smsp__inst_executed.sum",
]


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True,
                         stdin=subprocess.DEVNULL).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    rows = ncu_csv(rep, "--page", "raw")
    hdr, units, data = rows[0], rows[1], rows[2:]
    for d in data:
        print("kernel:", d[hdr.index("Kernel Name")])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k} = {d[i]} {units[i]}")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(d[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        print("  stalls per issued instruction:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:8]))
    if "--sass" in sys.argv:
        rows = ncu_csv(rep, "--page", "source", "--print-source", "sass")
        # one section per kernel: a "Kernel Name" row, a header row, instruction rows
        starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] or [0]
        for si, st0 in enumerate(starts):
            end = starts[si + 1] if si + 1 < len(starts) else len(rows)
            h = rows[st0 + 1]
            iS, iE, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
            samp, ex = collections.Counter(), collections.Counter()
            for row in rows[st0 + 2:end]:
                if len(row) != len(h):
                    continue
                toks = row[iSrc].split()
                if not toks:
                    continue
                op = (toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]).split(".")[0]
                samp[op] += int(row[iS] or 0)
                ex[op] += int(row[iE] or 0)
            ts, te = sum(samp.values()) or 1, sum(ex.values()) or 1
            print(f"  kernel {si}: SASS mix (executed warp-instructions {te}):")
            for op, s_ in samp.most_common(14):
                print(f"    {op:8s} samples {100 * s_ / ts:5.1f}%  executed {100 * ex[op] / te:5.1f}%")


if __name__ == "__main__":
    main()
