import sys
sys.path.insert(0, '.')
import numpy as np
from paper_1701_04900_b200 import inputs, asyflexa as A
P = inputs.config(3)
j = 30894
S = A.Solver(P)
for mode in ("seq", "async"):
    S.solve(sweeps=0, reset=True)
    for it in range(12):
        if mode == "seq":
            S.solve(sweeps=1, max_delay=0)
        else:
            S.solve(sweeps=1)
        x = S.x()
        out = S.stationarity()
        # fresh gradient of coordinate j
        r = P.A @ x - P.b
        g = P.A[:, j] @ r
        print(mode, it, "x_j", x[j], "g_j", g, "lam", P.lam, "tau", P.tau[j], "mfinf", out.mf_norminf, "F", out.objective, flush=True)
