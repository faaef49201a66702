"""One dense async launch (for ncu): python tools/slab_one.py CFG SWEEPS [cyclic|random]"""
import sys
sys.path.insert(0, '.')
from paper_1701_04900_b200 import inputs, asyflexa as A  # noqa: E402
idx, sw = int(sys.argv[1]), int(sys.argv[2])
sched = A.ASY_SCHED_CYCLIC if (len(sys.argv) > 3 and sys.argv[3] == "cyclic") else A.ASY_SCHED_RANDOM
P = inputs.config(idx)
S = A.Solver(P)
import os  # noqa: E402
st = S.solve(sweeps=sw, reset=True, schedule=sched, seed=1, workers=int(os.environ.get("WORKERS", "0")))
print(f"{st.kernel_ms:.3f} ms {8.0 * P.m * P.n * sw / (st.kernel_ms * 1e-3) / 1e9:.1f} GB/s F {st.objective:.10e}")
