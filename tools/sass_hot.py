"""Print the SASS lines with the most stall samples from an ncu source-page CSV."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
data = rows[2:]
tot = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
agg = {k: 0 for k in stall_cols}
for r in data:
    for k in stall_cols:
        try: agg[k] += int(r[idx[k]] or 0)
        except ValueError: pass
print("total samples", tot)
print(sorted(((v, k) for k, v in agg.items()), reverse=True)[:10])
top = sorted(data, key=lambda r: -int(r[idx["Warp Stall Sampling (All Samples)"]] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]
for r in top:
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    reasons = sorted(((int(r[idx[k]] or 0), k) for k in stall_cols), reverse=True)[:2]
    print(f"{s:7d} {100*s/tot:5.1f}% {r[idx['Address']][-5:]} {r[idx['Source']].strip()[:70]:70s} {reasons}")
