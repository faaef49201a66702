"""Analyse an ASY_TRACE dump: per-subtask globaltimer stamps (ns).
0 claimed, 1 issued (TMA), 2 landed (dot start), 3 published, 4 TMEM slot, 5 axpy start, 6 block seen complete, 7 axpy done."""
import sys
import numpy as np
tr = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 12).astype(np.int64)
G = int(sys.argv[2])
ok = np.all(tr[:, :8] > 0, axis=1)
tr = tr[ok]
t0 = tr.min()
tr = tr - t0
n = tr.shape[0]
names = ["claim", "issue", "land", "partials", "parkdecided", "axpystart", "blockdone", "axpydone", "solved", "tmemdone", "-", "-"]
print("subtasks", n, "span us", (tr.max() - tr.min()) / 1e3)
for a, b in [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 8), (8, 9), (9, 7), (0, 7)]:
    d = (tr[:, b] - tr[:, a]) / 1e3
    print(f"{names[a]:>9s} -> {names[b]:<9s}  mean {d.mean():7.2f} us  p50 {np.median(d):7.2f}  p90 {np.percentile(d, 90):7.2f}  max {d.max():7.2f}")
# block completion: last publish among the G panels of each sequence vs first publish
idx = np.arange(len(ok))[ok]
k = idx // G
seqs = np.unique(k)
first = np.array([tr[k == s, 3].min() for s in seqs[:2000]])
last = np.array([tr[k == s, 3].max() for s in seqs[:2000]])
lastland = np.array([tr[k == s, 2].max() for s in seqs[:2000]])
firstclaim = np.array([tr[k == s, 0].min() for s in seqs[:2000]])
lastclaim = np.array([tr[k == s, 0].max() for s in seqs[:2000]])
print("per block: publish spread us mean", ((last - first) / 1e3).mean(), "claim spread", ((lastclaim - firstclaim) / 1e3).mean(),
      "claim->last publish", ((last - firstclaim) / 1e3).mean())
# throughput in steady state
mid = (tr[:, 7] > np.percentile(tr[:, 7], 10)) & (tr[:, 7] < np.percentile(tr[:, 7], 90))
