"""Summarise an ASY_PROF dump of the row-slab kernels: [grid][16 warps][8] clock64 segment sums.
usage: python tools/slab_prof.py DUMP SEQUENCES [slabt [SPLIT]]"""
import sys
import numpy as np
a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 16, 8).astype(np.float64)
K = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0   # sequences in the launch (per-sequence cycles)
if len(sys.argv) > 3 and sys.argv[3] == "slabt":
    roles = {"producer": ([0], ["run"]),
             "dot": ([2, 3, 4, 5], ["wait_st", "guard", "process", "issue", "partial", "parkwait", "fullwait", "reduce"]),
             "axpy": ([6, 7, 8, 9], ["-", "dx wait", "-", "groups", "barrier"]),
             "seq": ([10, 11, 12, 13, 14, 15], ["-", "pfull", "publish", "arrival", "solve+dx"])}
else:
    roles = {"producer": ([0], ["run", "-", "-", "-", "-"]),
             "dot": ([2, 3, 4, 5], ["-", "guard", "full", "chunks", "partial"]),
             "axpy": ([6, 7, 8, 9], ["-", "dx wait", "stage", "compute", "barrier"]),
             "seq": ([10, 11, 12, 13, 14, 15], ["-", "pfull", "publish", "arrival", "solve+dx"])}
for role, (ws, names) in roles.items():
    s = a[:, ws].sum(axis=(0, 1)) / (a.shape[0] * len(ws))
    T = s.sum()
    print(f"{role:>8s} total {T:.3e} cyc/warp ({T / K:8.1f} per seq): " +
          " ".join(f"{n}={v / K:8.1f}" for n, v in zip(names, s) if n != "-"))
    if role == "dot":
        per = a[:, ws].sum(axis=2) / K
        print("          per dot warp (cyc/seq, mean over CTAs): " + " ".join(f"{v:8.1f}" for v in per.mean(axis=0)))
    if len(sys.argv) > 4:  # CTAs [0, SPLIT) own one row group more than the rest
        sp = int(sys.argv[4])
        for nm, sl in (("first", slice(0, sp)), ("rest", slice(sp, None))):
            q = a[sl][:, ws].sum(axis=(0, 1)) / (a[sl].shape[0] * len(ws))
            print(f"   {nm:>5s} CTAs: " + " ".join(f"{n}={v / K:8.1f}" for n, v in zip(names, q) if n != "-"))
