import sys, time
sys.path.insert(0, '.')
from paper_1701_04900_b200 import inputs, asyflexa as A
idx = int(sys.argv[1]); r = int(sys.argv[2]); s = int(sys.argv[3]); sw = int(sys.argv[4]) if len(sys.argv) > 4 else 1
P = inputs.config(idx, scale=float(sys.argv[5]) if len(sys.argv) > 5 else 1.0)
S = A.Solver(P)
t = time.time()
st = S.solve(sweeps=sw, reset=True, panel_rows=r, stages=s)
print(idx, r, s, "ok", st.kernel_ms, 8.0 * P.m * P.n * sw / (st.kernel_ms * 1e-3) / 1e9, "GB/s", st.objective, time.time() - t, flush=True)
