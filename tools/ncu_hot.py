#!/usr/bin/env python3
"""Top SASS instructions by warp-stall samples in an ncu report (source page), with
their neighbourhood: where a kernel's time goes, instruction by instruction."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
iS, iN, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
body = [r for r in rows[2:] if len(r) == len(h)]
tot = sum(float(r[iS] or 0) for r in body)
print(f"total samples {tot:.0f}, {len(body)} instructions")
# group samples by opcode
agg = {}
for r in body:
    op = r[iSrc].split()[0] if not r[iSrc].strip().startswith("@") else r[iSrc].split()[1]
    op = op.split(".")[0]
    agg[op] = agg.get(op, 0) + float(r[iS] or 0)
print("samples by opcode:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:14]))
idx = sorted(range(len(body)), key=lambda i: -float(body[i][iS] or 0))[:top]
for i in sorted(idx):
    r = body[i]
    print(f"{i:6d} {100 * float(r[iS]) / tot:5.2f}% exec={r[iN]:>9s}  {r[iSrc].strip()[:90]}")

# stall reasons by opcode class
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
cls = {}
for r in body:
    src = r[iSrc].split()
    op = (src[1] if src[0].startswith("@") else src[0]).split(".")[0]
    c = cls.setdefault(op, {})
    for k in reasons:
        c[k] = c.get(k, 0) + float(r[h.index(k)] or 0)
print("stall reasons (share of all samples) for the top opcodes:")
for op, c in sorted(cls.items(), key=lambda kv: -sum(kv[1].values()))[:8]:
    s = sorted(c.items(), key=lambda kv: -kv[1])[:6]
    print(f"  {op:8s} " + ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in s if v > 0))
