"""Summarise an ncu source page (SASS) CSV: per-opcode executed instructions and stall samples,
and the hottest instructions.  Usage: ncu -i rep --page source --csv | python tools/sass_hot.py [N]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(sys.stdin))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[i0]
ix = {k: h.index(k) for k in ("Source", "Warp Stall Sampling (All Samples)", "Instructions Executed")}
stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
ops = defaultdict(lambda: [0, 0])
lines = []
tot_i = tot_s = 0
for r in rows[i0 + 1:]:
    if len(r) < len(h) or r[0] == "Address":
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    ni = int(r[ix["Instructions Executed"]] or 0)
    ns = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ops[op.split(".")[0]][0] += ni
    ops[op.split(".")[0]][1] += ns
    tot_i += ni
    tot_s += ns
    st = sorted(((int(r[h.index(k)] or 0), k[6:]) for k in stall_cols), reverse=True)[:3]
    lines.append((ns, ni, r[0][-5:], src[:70], st))
print(f"total executed {tot_i}  samples {tot_s}")
for op, (ni, ns) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{op:12s} inst {ni:10d} ({100*ni/max(tot_i,1):5.1f}%)  samples {ns:7d} ({100*ns/max(tot_s,1):5.1f}%)")
N = int(sys.argv[1]) if len(sys.argv) > 1 else 30
print("--- hottest instructions ---")
for ns, ni, a, src, st in sorted(lines, reverse=True)[:N]:
    print(f"{a} {ns:6d} {ni:9d}  {src:70s} {st}")
