#!/usr/bin/env python3
"""Per-launch durations (us) of the last gradient in an ncu launch list, in launch order."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
s = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[s]
iK, iV = h.index("Kernel Name"), h.index("Metric Value")
seq = [(r[iK].split("(")[0], float(r[iV]) / 1e3) for r in rows[s + 1:]]
m = [i for i, (k, _) in enumerate(seq) if "k_set_basis" in k][-1]
g = seq[m:]
tags = {"svgb_jit": "", "svgb::k_obs_pass": "O:", "svgb::k_finalize": "F:", "svgb::k_set_basis": "B:"}
print(" ".join(f"{tags.get(k, k[:6] + ':')}{v:.0f}" for k, v in g))
