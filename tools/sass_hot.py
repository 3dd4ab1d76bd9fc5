"""Summarise an ncu --page source --print-source sass CSV: instruction mix (executed warp-level
instructions by opcode) and the hottest instructions by stall samples.  usage: sass_hot.py CSV [N]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
ex = Counter()
samp = Counter()
tot_ex = 0
tot_s = 0
for r in body:
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    base = op.split(".")[0]
    n = int(float(r[ix["Instructions Executed"]] or 0))
    s = int(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
    ex[base] += n
    samp[base] += s
    tot_ex += n
    tot_s += s
print(f"total warp instructions {tot_ex:,}  samples {tot_s:,}")
for op, n in ex.most_common(30):
    print(f"{op:10s} {n:14,d} {100*n/tot_ex:5.1f}%  samples {100*samp[op]/max(tot_s,1):5.1f}%")
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print("\nhottest instructions (stall samples):")
body.sort(key=lambda r: -int(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)))
for r in body[:N]:
    st = sorted(((int(float(r[ix[c]] or 0)), c[6:]) for c in stall_cols), reverse=True)[:3]
    print(f"{r[ix['Address']]:>6s} {int(float(r[ix['Warp Stall Sampling (All Samples)']] or 0)):7d} "
          f"ex {int(float(r[ix['Instructions Executed']] or 0)):10,d}  {r[ix['Source']][:60]:60s} {st}")
