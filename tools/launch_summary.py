#!/usr/bin/env python3
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel
count / mean / total and share of the GPU time of the last N gradients."""
import collections
import csv
import sys


def main(path, grads=1):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    iK, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    seq = [(r[iK], float(r[iV])) for r in rows[start + 1:] if r[iM] == "gpu__time_duration.sum"]
    marks = [i for i, (k, _) in enumerate(seq) if "k_set_basis" in k]
    g = seq[marks[-grads]:] if len(marks) >= grads else seq
    g = [(k, v) for k, v in g if "FillFunctor" not in k]  # the bench's L2 flush, outside the timed events
    tot = sum(v for _, v in g)
    d = collections.defaultdict(list)
    for k, v in g:
        name = k.split("(")[0]
        d[name].append(v)
    print(f"{path}: last {grads} gradient(s), {len(g)} launches, GPU time {tot / 1e3:.1f} us")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {k[:60]:60s} n={len(v):5d} mean={sum(v) / len(v) / 1e3:9.2f} us "
              f"total={sum(v) / 1e3:10.1f} us share={100 * sum(v) / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
