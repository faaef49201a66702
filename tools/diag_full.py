"""Full-size behaviour of a config: generation time, sweep time, convergence."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_1701_04900_b200 import inputs, asyflexa as A
idx = int(sys.argv[1]); total = int(sys.argv[2]); chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 10
t = time.time(); P = inputs.config(idx); print("gen s", time.time() - t, P.m, P.n, P.lam, P.gamma, flush=True)
t = time.time(); S = A.Solver(P); print("upload s", time.time() - t, flush=True)
S.solve(sweeps=0, reset=True)
done = 0; prevF = None
while done < total:
    st = S.solve(sweeps=chunk)
    done += chunk
    out = S.stationarity()
    byt = (8.0 * P.m * P.n if P.kind == "dense" else 12.0 * P.vals.size + 24.0 * P.n) * chunk
    print(f"sweeps {done} kernel_ms/sweep {st.kernel_ms/chunk:.3f} GB/s {byt/st.kernel_ms/1e6:.0f} upd/s {st.block_updates/st.kernel_ms*1e3:.3e} "
          f"F {out.objective!r} mf2 {out.mf_norm2:.3e} merit {out.merit_inf:.3e}", flush=True)
    if prevF is not None and abs(prevF - out.objective) <= 1e-15 * abs(out.objective) and out.mf_norm2 < 1e-7:
        break
    prevF = out.objective
