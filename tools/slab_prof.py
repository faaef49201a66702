"""Summarise an ASY_PROF dump of the row-slab kernel: [grid][16 warps][8] clock64 segment sums."""
import sys
import numpy as np
a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 16, 8).astype(np.float64)
K = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0   # sequences in the launch (per-sequence cycles)
roles = {"producer": ([0], ["run", "-", "-", "-", "-"]),
         "dot": ([2, 3, 4, 5], ["-", "guard", "full", "chunks", "partial"]),
         "axpy": ([6, 7, 8, 9], ["-", "dx wait", "stage", "compute", "barrier"]),
         "seq": ([10, 11, 12, 13, 14, 15], ["-", "pfull", "publish", "arrival", "solve+dx"])}
for role, (ws, names) in roles.items():
    s = a[:, ws].sum(axis=(0, 1)) / (a.shape[0] * len(ws))
    T = s.sum()
    print(f"{role:>8s} total {T:.3e} cyc/warp ({T / K:8.1f} per seq): " +
          " ".join(f"{n}={v / K:8.1f}" for n, v in zip(names, s) if n != "-"))
