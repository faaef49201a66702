"""A/B throughput of the async kernels between library builds, on one generated instance.
usage: python tools/ab_perf.py CFG SWEEPS SCHED REPS VARIANT [VARIANT ...]
VARIANT = "" (lib/libasyflexa.so) or NAME (lib/libasyflexa_NAME.so, see build.py --variant);
the variants are run round robin (same box, same instance) and the async result is checked
against a few sequential-mode sweeps only through the objective it prints."""
import importlib.util
import os
import sys
import time

sys.path.insert(0, '.')
from paper_1701_04900_b200 import inputs  # noqa: E402

idx, sw, sched, reps = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
names = sys.argv[5:] or [""]


def load(name):
    if name in ("", "default"):
        os.environ.pop("ASY_LIB_VARIANT", None)
    else:
        os.environ["ASY_LIB_VARIANT"] = name
    spec = importlib.util.spec_from_file_location("asyflexa_" + (name or "default"),
                                                  "paper_1701_04900_b200/asyflexa.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


t0 = time.time()
P = inputs.config(idx)
print(f"config {idx} generated in {time.time() - t0:.1f}s", flush=True)
mods = {n: load(n) for n in names}
solvers = {n: mods[n].Solver(P) for n in names}
for rep in range(reps):
    for n in names:
        A, S = mods[n], solvers[n]
        sc = A.ASY_SCHED_CYCLIC if sched == "cyclic" else A.ASY_SCHED_RANDOM
        st = S.solve(sweeps=sw, reset=True, schedule=sc, seed=rep, workers=int(os.environ.get("WORKERS", "0")),
                     max_delay=int(os.environ.get("MAX_DELAY", "-1")))
        if P.kind == "dense":
            rate = f"{8.0 * P.m * P.n * sw / (st.kernel_ms * 1e-3) / 1e9:8.1f} GB/s"
        else:
            rate = f"{P.nblocks * sw / (st.kernel_ms * 1e-3) / 1e9:8.3f} G upd/s"
        print(f"{n or 'default':>10s} rep {rep}: {st.kernel_ms:9.3f} ms  {rate}  kernel {st.kernel} delay {st.delay} "
              f"obs {st.delay_observed}  F {st.objective:.12e}", flush=True)
for S in solvers.values():
    S.close()
