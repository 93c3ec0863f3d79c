"""Aggregate an ncu `--page source --csv --print-source cuda,sass` export by source line."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cur = None; agg = collections.Counter(); inst = collections.Counter(); src = {}; hdr = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur = r[1].split('/')[-1]; continue
    if r[0] == "Line No":
        hdr = r; ie = r.index("Instructions Executed"); ss = r.index("Warp Stall Sampling (All Samples)"); continue
    if hdr is None or len(r) <= ie or not r[0].strip(): continue
    key = (cur, int(r[0])); src[key] = r[1].strip()[:90]
    try:
        agg[key] += float(r[ss] or 0); inst[key] += float(r[ie] or 0)
    except ValueError:
        pass
ts = sum(agg.values()); ti = sum(inst.values())
print("total stall samples", ts, "warp instructions", ti)
for k, v in agg.most_common(top):
    print(f"{k[0]:>14}:{k[1]:<4} stall {v/ts*100:5.1f}% inst {inst[k]/ti*100:5.1f}%  {src[k]}")
