"""Throughput sweep over panel rows / stages / workers for a dense config."""
import sys
sys.path.insert(0, '.')
from paper_1701_04900_b200 import inputs, asyflexa as A
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
P = inputs.config(idx)
S = A.Solver(P)
S.solve(sweeps=5, reset=True)
grid = [(0, 0, 0), (64, 0, 0), (96, 0, 0), (128, 0, 0), (128, 4, 0), (160, 0, 0), (192, 0, 0), (256, 0, 0),
        (128, 0, 74)]
for r, s, w in grid:
    kw = dict(panel_rows=r, stages=s, workers=w)
    try:
        best = 0
        for rep in range(3):
            st = S.solve(sweeps=5, **kw)
            best = max(best, 8.0 * P.m * P.n * 5 / (st.kernel_ms * 1e-3) / 1e9)
        print(kw, f"{best:.0f} GB/s  F={st.objective}", flush=True)
    except A.AsyError as e:
        print(kw, "ERR", e, flush=True)
