"""Throughput of the dense async kernel variants on one config (debug tool).
usage: python tools/slab_perf.py CFG SWEEPS [variant ...]
variant = name:ENV=VAL,ENV=VAL  (e.g. hold:ASY_SLAB_HOLD=1  panel:ASY_DENSE_KERNEL=panel)"""
import os
import sys
import time

sys.path.insert(0, '.')
from paper_1701_04900_b200 import inputs, asyflexa as A  # noqa: E402

idx, sw = int(sys.argv[1]), int(sys.argv[2])
variants = sys.argv[3:] or ["default:"]
t0 = time.time()
P = inputs.config(idx)
print(f"config {idx} generated in {time.time() - t0:.1f}s", flush=True)
S = A.Solver(P)
for v in variants:
    name, _, envs = v.partition(":")
    keys = []
    for kv in filter(None, envs.split(",")):
        k, _, val = kv.partition("=")
        os.environ[k] = val
        keys.append(k)
    for rep in range(2):
        st = S.solve(sweeps=sw, reset=True, schedule=A.ASY_SCHED_RANDOM, seed=rep,
                     workers=int(os.environ.get("WORKERS", "0")))
        gbs = 8.0 * P.m * P.n * sw / (st.kernel_ms * 1e-3) / 1e9
        print(f"{name:>12s} rep {rep}: {st.kernel_ms:8.3f} ms  {gbs:8.1f} GB/s  "
              f"{P.nblocks * sw / (st.kernel_ms * 1e-3) / 1e6:7.3f} M upd/s  F {st.objective:.10e}", flush=True)
    for k in keys:
        del os.environ[k]
S.close()
