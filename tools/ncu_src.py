"""Summarise an `ncu --page source --csv --print-source sass` export: warp-stall samples
per SASS instruction (top N, with the previous instructions for context) and per opcode.
usage: ncu_src.py FILE [N]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
ci = {h: i for i, h in enumerate(hdr)}
smp = ci["Warp Stall Sampling (All Samples)"]
ex = ci["Instructions Executed"]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
recs = []
for k, r in enumerate(rows[hdr_i + 1:]):
    if len(r) < len(hdr): continue
    s = float(r[smp] or 0)
    top = sorted(((float(r[ci[h]] or 0), h[6:]) for h in reasons), reverse=True)[:3]
    recs.append((k, s, r[0], r[ci["Source"]].strip(), float(r[ex] or 0), top))
tot = sum(x[1] for x in recs)
print("total samples", tot, "instructions", len(recs))
byop = collections.Counter()
for x in recs:
    op = x[3].split()[0] if x[3] else "?"
    if op.startswith("@"): op = x[3].split()[1]
    byop[op.split(".")[0]] += x[1]
print("by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in byop.most_common(14)))
for k, s, addr, src, e, top in sorted(recs, key=lambda x: -x[1])[:n]:
    print(f"{100*s/tot:5.1f}% #{k:5d} {src[:70]:70s} ex={e:.3g} " + " ".join(f"{kk}:{100*v/max(s,1):.0f}" for v, kk in top if v))
