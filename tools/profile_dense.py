"""Small driver for ncu: a few async launches of a config (default 1)."""
import sys
sys.path.insert(0, '.')
from paper_1701_04900_b200 import inputs, asyflexa as A
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
kw = {}
for a in sys.argv[3:]:
    k, v = a.split('=')
    kw[k] = int(v)
P = inputs.config(idx)
S = A.Solver(P)
for i in range(3):
    st = S.solve(sweeps=sweeps, reset=(i == 0), **kw)
    print(i, st.kernel_ms, st.block_updates, 8 * P.m * P.n * sweeps / st.kernel_ms / 1e6, "GB/s", st.objective, flush=True)
