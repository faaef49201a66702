import sys
sys.path.insert(0, '.')
from paper_1701_04900_b200 import inputs, asyflexa as A
P = inputs.config(1)
S = A.Solver(P)
for name, T in (("panel", {"dense_kernel": 1}), ("slabt", {"dense_kernel": 4})):
    for rep in range(2):
        st = S.solve(sweeps=20, reset=True, tuning=T)
        print(name, rep, f"{st.kernel_ms:.3f} ms {8.0*P.m*P.n*20/(st.kernel_ms*1e-3)/1e9:.1f} GB/s kernel {st.kernel} F {st.objective:.10e}", flush=True)
S.close()
