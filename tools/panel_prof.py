"""Summarise an ASY_PROF dump of the panel kernel: [grid][16 warps][8] clock64 segment sums.
usage: python tools/panel_prof.py DUMP PANELS_PER_SM"""
import sys
import numpy as np
a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 16, 8).astype(np.float64)
n = float(sys.argv[2])  # panels per SM in the launch
roles = {"dot": ([4, 5, 6, 7], ["full wait", "w", "dot+park", "slot wait", "2nd park", "publish+handoff"]),
         "axpy": ([0, 1, 2, 3, 8, 9, 10, 11], ["handoff wait", "arrival wait", "solve", "-", "scatter", "free"])}
for role, (ws, names) in roles.items():
    s = a[:, ws].sum(axis=(0, 1)) / (a.shape[0] * len(ws))
    per = n / len(ws)  # panels per warp
    print(f"{role:>5s}: total {s.sum() / per:8.0f} cyc/panel/warp: " +
          " ".join(f"{nm}={v / per:7.0f}" for nm, v in zip(names, s) if nm != "-"))
