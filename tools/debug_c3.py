import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_1701_04900_b200 import inputs, asyflexa as A
from oracle import asyflexa_oracle as O
idx = int(sys.argv[1]); sweeps = int(sys.argv[2]); mode = sys.argv[3] if len(sys.argv) > 3 else "async"
P = inputs.config(idx)
S = A.Solver(P)
if mode == "async":
    S.solve(sweeps=sweeps, reset=True)
else:
    S.solve(sweeps=sweeps, reset=True, max_delay=0)
x = S.x()
out = S.stationarity()
print("gpu F", out.objective, "mf2", out.mf_norm2, "mfinf", out.mf_norminf, flush=True)
t = time.time()
mf = O.stationarity(P, x)
print("oracle F", O.objective(P, x), "mf2", np.linalg.norm(mf), "mfinf", np.abs(mf).max(), time.time() - t, flush=True)
bad = np.argsort(-np.abs(mf))[:20]
print("worst coords", bad, mf[bad], x[bad])
blk = bad // P.block
print("their blocks", np.unique(blk), "nblocks", P.nblocks)
nb = np.abs(mf) > 1e-3
print("count > 1e-3:", nb.sum(), "blocks:", np.unique(np.flatnonzero(nb) // P.block)[:50])
