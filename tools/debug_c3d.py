import sys, os
sys.path.insert(0, '.')
import numpy as np
from paper_1701_04900_b200 import inputs, asyflexa as A
P = inputs.config(3)
S = A.Solver(P)
j = 30894
for per_launch, total, delay, sched in [(2, 40, -1, 0), (2, 40, 1, 0), (10, 40, 1, 0), (10, 40, -1, 1), (3, 39, -1, 0)]:
    S.solve(sweeps=0, reset=True)
    done = 0
    while done < total:
        S.solve(sweeps=per_launch, max_delay=delay, schedule=sched)
        done += per_launch
    out = S.stationarity()
    x = S.x()
    print(f"per_launch {per_launch} delay {delay} sched {sched}: F {out.objective!r} mfinf {out.mf_norminf:.3e} x_j {x[j]}", flush=True)
