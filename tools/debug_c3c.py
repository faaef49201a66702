import sys, os
sys.path.insert(0, '.')
import numpy as np
from paper_1701_04900_b200 import inputs, asyflexa as A
cfg = int(sys.argv[1]); scale = float(sys.argv[2])
P = inputs.config(cfg, scale=scale)
S = A.Solver(P)
print("m n G-ish", P.m, P.n, P.block, flush=True)
for per_launch, total, delay in [(1, 40, -1), (10, 40, -1), (40, 40, -1), (10, 40, 2), (10, 40, 0)]:
    S.solve(sweeps=0, reset=True)
    done = 0
    while done < total:
        S.solve(sweeps=per_launch, max_delay=delay)
        done += per_launch
    out = S.stationarity()
    print(f"per_launch {per_launch} delay {delay}: F {out.objective!r} mfinf {out.mf_norminf:.3e}", flush=True)
