"""Diagnostics: async convergence / timing on small analogs (GPU)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, "tests"); from cases import make_case
from oracle import asyflexa_oracle as O
from paper_1701_04900_b200 import asyflexa as A

for case in sys.argv[1:]:
    P = make_case(case)
    xs, Fs, sw = O.estimate_fstar(P, P.gamma, max_sweeps=20000, tol=1e-15)
    print(case, "oracle sweeps", sw, "F*", Fs, "MF", np.linalg.norm(O.stationarity(P, xs)), flush=True)
    for workers in (0, 8, 32):
        S = A.Solver(P)
        S.solve(sweeps=0, reset=True)
        t = time.time()
        for it in range(10):
            st = S.solve(sweeps=100, workers=workers)
            out = S.stationarity()
            print(f"  w={workers} it={it} kernel_ms={st.kernel_ms:.2f} F_rel={(out.objective-Fs)/abs(Fs):.3e} mf2={out.mf_norm2:.3e} merit={out.merit_inf:.3e}", flush=True)
        print("  wall", time.time() - t, flush=True)
        S.close()
