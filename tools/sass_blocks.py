"""Group an ncu SASS source CSV into runs of instructions with equal execution counts (basic-block
like) and print the heaviest by instructions and by stall samples.  usage: sass_blocks.py CSV [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(float(r[ix["Instructions Executed"]] or 0)) for r in body)
tots = sum(int(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)) for r in body)
segs, cur = [], None
for r in body:
    n = int(float(r[ix["Instructions Executed"]] or 0))
    s = int(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
    st = {c: int(float(r[ix[c]] or 0)) for c in stall_cols}
    a = r[ix["Address"]][-5:]
    if cur and abs(n - cur["n"]) <= max(2, 0.02 * cur["n"]):
        cur["cnt"] += 1; cur["tot"] += n; cur["s"] += s; cur["end"] = a
        for c in stall_cols: cur["st"][c] += st[c]
    else:
        cur = {"n": n, "cnt": 1, "tot": n, "s": s, "start": a, "end": a, "first": r[ix["Source"]][:44], "st": st}
        segs.append(cur)
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print(f"total instr {tot:,} samples {tots:,}")
for key in ("s", "tot"):
    print(f"--- by {'samples' if key == 's' else 'instructions'}")
    for c in sorted(segs, key=lambda c: -c[key])[:N]:
        top = sorted(((v, k[6:]) for k, v in c["st"].items()), reverse=True)[:2]
        print(f"{c['start']}-{c['end']} x{c['n']:>10,d} n{c['cnt']:4d} instr {100*c['tot']/tot:5.1f}% samp {100*c['s']/max(tots,1):5.1f}% {top} {c['first']}")
