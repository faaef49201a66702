"""Rate and sweeps-to-target of the async kernels versus the delay bound (debug tool).
usage: python tools/delay_sweep.py CFG CHECK CAP delay [delay ...]   (delay -1 = auto)
For each max_delay: solve from x0 in chunks of CHECK sweeps until (F - F*)/|F*| <= 1e-6 against
the oracle's F* (tests/golden/fstar_full.json) or CAP sweeps; prints the kernel rate, the sweeps
needed, and the enforced / observed delay.  Cyclic schedule unless SCHED=random."""
import json
import os
import sys

sys.path.insert(0, ".")
from paper_1701_04900_b200 import inputs, asyflexa as A  # noqa: E402

idx, check, cap = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
delays = [int(v) for v in sys.argv[4:]] or [-1]
P = inputs.config(idx)
Fs = float(json.load(open("tests/golden/fstar_full.json"))[f"config{idx}"]["F_star"])
sched = A.ASY_SCHED_RANDOM if os.environ.get("SCHED") == "random" else A.ASY_SCHED_CYCLIC
S = A.Solver(P)
bpu = 8.0 * P.m * P.block if P.kind == "dense" else None
for d in delays:
    for rep in range(2):
        st = S.solve(sweeps=check, reset=True, max_delay=d, schedule=sched, seed=rep)
        sweeps, kms, upd = check, st.kernel_ms, st.block_updates
        while (st.objective - Fs) / abs(Fs) > 1e-6 and sweeps < cap:
            st = S.solve(sweeps=check, max_delay=d, schedule=sched, seed=rep)
            sweeps += check
            kms += st.kernel_ms
            upd += st.block_updates
        rate = upd / (kms * 1e-3)
        gbs = f"{rate * bpu / 1e9:7.1f} GB/s" if bpu else ""
        print(f"delay {d:7d} rep {rep}: {rate / 1e6:9.3f} M upd/s {gbs}  sweeps {sweeps:6d}  "
              f"rel {(st.objective - Fs) / abs(Fs):.2e}  enforced {st.delay} observed {st.delay_observed}  "
              f"kernel {st.kernel}", flush=True)
S.close()
