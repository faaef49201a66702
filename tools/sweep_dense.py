"""Throughput sweep over panel rows / stages / workers for a dense config."""
import sys, itertools
sys.path.insert(0, '.')
from paper_1701_04900_b200 import inputs, asyflexa as A
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
P = inputs.config(idx)
S = A.Solver(P)
S.solve(sweeps=5, reset=True)
grid = [dict(panel_rows=r, stages=s, workers=w) for r, s, w in
        [(0,0,0),(64,0,0),(96,0,0),(128,0,0),(160,0,0),(192,0,0),(256,0,0),(128,3,0),(128,4,0),(128,5,0),(64,6,0),(64,10,0),(128,0,74),(128,0,111)]]
for kw in grid:
    if P.block * kw['panel_rows'] > 8192: continue
    best = 0
    for rep in range(3):
        st = S.solve(sweeps=5, **kw)
        gbs = 8.0 * P.m * P.n * 5 / (st.kernel_ms * 1e-3) / 1e9
        best = max(best, gbs)
    print(kw, f"{best:.0f} GB/s", flush=True)
