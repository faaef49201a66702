"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: time share per kernel."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if r]
h = None
tot = collections.Counter(); cnt = collections.Counter()
for r in rows:
    if "Kernel Name" in r:
        h = {k: i for i, k in enumerate(r)}
        continue
    if h is None or len(r) < len(h):
        continue
    if r[h["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[h["Kernel Name"]].split("(")[0]
    v = float(r[h["Metric Value"]].replace(",", ""))
    unit = r[h["Metric Unit"]]
    v = {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3, "ms": v * 1e3, "second": v * 1e6, "s": v * 1e6}.get(unit, v)
    tot[name] += v; cnt[name] += 1
S = sum(tot.values())
print(f"{'kernel':55s} {'launches':>8s} {'total_us':>10s} {'share':>7s}")
for k, v in tot.most_common():
    print(f"{k[:55]:55s} {cnt[k]:8d} {v:10.1f} {100*v/S:6.1f}%")
