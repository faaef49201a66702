"""Attribute ncu warp-stall samples (source page, SASS csv) to CUDA source lines.
usage: python tools/ncu_lines.py SRC_SASS.csv NVDISASM_G.sass FUNCTION_MANGLED [N]
(NVDISASM_G.sass = `nvdisasm -g -c` of the cubin built with -lineinfo)"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
addrs = [int(r[0], 16) for r in body]
base = min(addrs)
stalls = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]

# offset -> (file, line) from nvdisasm -g
fn = sys.argv[3]
lines = open(sys.argv[2]).read().split('\n')
start = next(i for i, l in enumerate(lines) if l.startswith('.text.' + fn + ':'))
cur = None
off2line = {}
for l in lines[start + 1:]:
    if l.startswith('.text.') or l.startswith('//----'):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
agg = collections.defaultdict(lambda: collections.Counter())
tot = 0.0
for r in body:
    off = int(r[0], 16) - base
    key = off2line.get(off, ('?', 0))
    for h in stalls:
        v = float(r[ci[h]] or 0)
        agg[key][h[6:]] += v
        tot += v
src = {}
n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
for key, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:n]:
    s = sum(c.values())
    top = " ".join(f"{k}:{100 * v / s:.0f}%" for k, v in c.most_common(3))
    print(f"{100 * s / tot:5.1f}% {key[0]}:{key[1]:<5d} {top}")
