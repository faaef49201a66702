"""Convergence probe (developer tool, GPU): F, ||M_F||_2 and the Sec. 4.3 merit of the
asynchronous / sequential / Jacobi modes at checkpoints, one JSON line per checkpoint.

python tools/converge_probe.py --config 4 --mode async --chunk 2000 --total 60000
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1701_04900_b200 import asyflexa as A  # noqa: E402
from paper_1701_04900_b200 import inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--mode", default="async", choices=["async", "seq", "jacobi"])
ap.add_argument("--chunk", type=int, default=1000)
ap.add_argument("--total", type=int, default=10000)
ap.add_argument("--schedule", default="cyclic")
ap.add_argument("--seconds", type=float, default=1e9, help="stop after this much wall time")
ap.add_argument("--gamma", type=float, default=None)
a = ap.parse_args()

t0 = time.time()
P = inputs.config(a.config)
S = A.Solver(P)
print(json.dumps({"config": a.config, "mode": a.mode, "gen_s": time.time() - t0}), flush=True)
kw = dict(schedule=A.ASY_SCHED_CYCLIC if a.schedule == "cyclic" else A.ASY_SCHED_RANDOM, seed=1234)
if a.gamma:
    kw["gamma"] = a.gamma
if a.mode == "seq":
    kw["max_delay"] = 0
if a.mode == "jacobi":
    kw["mode"] = A.ASY_MODE_SYNC_JACOBI
S.solve(sweeps=0, reset=True)
done, kms = 0, 0.0
t1 = time.time()
while done < a.total and time.time() - t1 < a.seconds:
    st = S.solve(sweeps=a.chunk, **kw)
    done += a.chunk
    kms += st.kernel_ms
    out = S.stationarity()
    print(json.dumps({"sweeps": done, "F": repr(out.objective), "F_maint": repr(st.objective),
                      "mf2": out.mf_norm2, "merit": out.merit_inf, "kernel_ms": kms,
                      "delay": st.delay, "dobs": st.delay_observed}), flush=True)
S.close()
