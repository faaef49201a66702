"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
body = [r for r in rows[2:] if len(r) == len(hdr)]
ci = {h: i for i, h in enumerate(hdr)}
st = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
tot = {h: sum(float(r[ci[h]] or 0) for r in body) for h in st}
T = sum(tot.values())
print("total samples", T)
print(" ".join(f"{h[6:]}={100 * v / T:.1f}%" for h, v in sorted(tot.items(), key=lambda x: -x[1]) if v > 0.005 * T))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
body.sort(key=lambda r: -float(r[ci['Warp Stall Sampling (All Samples)']] or 0))
for r in body[:n]:
    s = float(r[ci['Warp Stall Sampling (All Samples)']] or 0)
    top = sorted(((float(r[ci[h]] or 0), h[6:]) for h in st), reverse=True)[:3]
    print(f"{100 * s / T:5.1f}% {r[0]:>6s} {r[1][:70]:70s} " + " ".join(f"{h}:{v:.0f}" for v, h in top if v > 0))
