"""Per-source-line stall samples from `ncu --page source --csv --print-source cuda,sass`."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
cur_file, cur_line, cur_src = None, None, None
agg = collections.Counter(); srcs = {}; reasons = collections.defaultdict(collections.Counter)
hdr = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split('/')[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if r[0] == "Function Name": continue
    if hdr is None: continue
    if r[0] not in ("", "-"):
        cur_line, cur_src = r[0], r[1]
    try: s = int(r[4] or 0)
    except ValueError: continue
    key = (cur_file, cur_line)
    agg[key] += s; srcs[key] = cur_src
    for i, k in enumerate(hdr):
        if k.startswith("stall_") and "Not Issued" not in k:
            try: reasons[key][k] += int(r[i] or 0)
            except ValueError: pass
tot = sum(agg.values())
for key, s in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{s:7d} {100*s/tot:5.1f}% {key[0]}:{key[1]:5s} {srcs[key].strip()[:80]:80s} {reasons[key].most_common(2)}")
