import sys, numpy as np
a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 16, 8).astype(np.float64)
tot = a.sum(axis=(0))
names = {"axpy": ["handoff", "x+arrive", "solve", "complete", "tmem+red", "tail", "-", "-"],
         "dot": ["full", "w", "pass1", "parkwait", "park", "publish+ring", "-", "-"]}
for role, ws in (("axpy", [0, 1, 2, 3]), ("dot", [4, 5, 6, 7])):
    s = tot[ws].sum(axis=0)
    T = s.sum()
    print(role, " ".join(f"{n}={100*v/T:5.1f}%" for n, v in zip(names[role], s) if n != "-"), f"total cycles/warp {T/len(ws)/a.shape[0]:.3e}")
