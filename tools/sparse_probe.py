"""Throughput / progress probe of the CSC async kernel (debug tool, not used by tests or bench).
usage: python tools/sparse_probe.py CFG SWEEPS CHUNKS [max_delay]
Runs CHUNKS async solves of SWEEPS sweeps each on BASELINE configs[CFG] (seed 0) and prints
per-chunk kernel time, rate, F and the enforced / observed delay."""
import sys
import time

sys.path.insert(0, ".")
from paper_1701_04900_b200 import inputs, asyflexa as A  # noqa: E402

idx, sw, chunks = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
md = int(sys.argv[4]) if len(sys.argv) > 4 else -1
t0 = time.time()
P = inputs.config(idx)
print(f"config {idx} ({P.m}x{P.n}, nnz {getattr(P, 'vals', None) is not None and P.vals.size}) "
      f"generated in {time.time() - t0:.1f}s", flush=True)
S = A.Solver(P)
S.solve(sweeps=0, reset=True)
for c in range(chunks):
    t1 = time.time()
    st = S.solve(sweeps=sw, max_delay=md)
    print(f"chunk {c}: {st.kernel_ms:9.3f} ms kernel, {st.block_updates / (st.kernel_ms * 1e-3) / 1e9:6.3f} G upd/s, "
          f"F {st.objective:.12e}, delay {st.delay}, observed {st.delay_observed}, kernel {st.kernel}, "
          f"wall {time.time() - t1:.2f}s", flush=True)
out = S.stationarity()
print(f"final F {out.objective:.12e} ||M_F||_2 {out.mf_norm2:.3e}", flush=True)
S.close()
