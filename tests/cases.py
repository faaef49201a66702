"""Small analogs of the BASELINE configs (shared by GPU tests and tools), and the
oracle's F* of each (reading R12)."""
import numpy as np

from paper_1701_04900_b200 import inputs

_FSTAR = {}


def fstar(P, key=None):
    """The oracle's F* for the async acceptance tests.

    Algorithm 1 run "until variations in the objective value were undetectable"
    [PAPER.md:434] (oracle.estimate_fstar).  For the l1-logistic cases that stopping rule
    fires while F is still ~1e-7 above the minimum (tau = 0.25||a_j||^2/m makes the steps
    tiny once the margins grow, tests/test_oracle_pins.py), so there F* is F at a library
    candidate minimiser certified by the Fenchel duality gap (oracle.duality_gap_l1)."""
    from oracle import asyflexa_oracle as O
    key = key or P.name
    if key in _FSTAR:
        return _FSTAR[key]
    convex_l1 = P.reg == "l1" and P.c == 0.0 and not np.isfinite(P.lo) and not np.isfinite(P.hi)
    if P.loss == "logistic" and convex_l1:
        x = O.minimiser_l1_logistic_liblinear(P)
        F = O.objective(P, x)
        gap = O.duality_gap_l1(P, x)
        assert gap <= 1e-7 * abs(F), (key, gap, F)
    else:
        _, F, _ = O.estimate_fstar(P, P.gamma, max_sweeps=20000, tol=1e-15)
    _FSTAR[key] = F
    return F


def make_case(name):
    P = _make_case(name)
    P.name = name
    return P


def _make_case(name):
    if name == "config0":
        return inputs.config(0)
    if name == "dense_ragged":   # odd m, ragged last block, several panels
        return inputs.dense_lasso(203, 517, nnz_frac=0.03, sigma=0.01, lam_frac=0.08, block=32,
                                  gamma=0.9, seed=5, name="dense_ragged")
    if name == "dense_normalized":  # config 1 recipe, small
        return inputs.dense_lasso(400, 800, nnz_frac=0.01, sigma=0.01, lam_frac=0.05, block=32,
                                  gamma=0.9, normalize=True, seed=2)
    if name == "nonconvex":       # config 2 recipe, small
        return inputs.nonconvex_box(60, 130, block=8, gamma=0.5, seed=3, lam_frac=0.3)
    if name == "large_block":     # config 3 recipe, small, max block size 128
        return inputs.dense_lasso(300, 700, nnz_frac=0.005, sigma=0.01, lam_frac=0.02, block=128,
                                  gamma=0.9, seed=4)
    if name == "tall_block":      # 280 rows: one worker's slab = 9 row groups of 128 columns
        return inputs.dense_lasso(280, 520, nnz_frac=0.01, sigma=0.01, lam_frac=0.02, block=128,
                                  gamma=0.9, seed=11)
    if name == "tall600":         # one worker's slab = 19 row groups: too tall for the TMEM park ring
        return inputs.dense_lasso(600, 330, nnz_frac=0.02, sigma=0.01, lam_frac=0.05, block=32,
                                  gamma=0.9, seed=14)
    if name == "box64":           # config 2 recipe, blocks of 64 (two 32-column sub-sequences)
        return inputs.nonconvex_box(150, 400, block=64, gamma=0.5, seed=12, lam_frac=0.3)
    if name == "block100":        # blocks of 100: padded to 128, last sub-sequence 4 columns wide
        return inputs.dense_lasso(210, 470, nnz_frac=0.02, sigma=0.01, lam_frac=0.05, block=100,
                                  gamma=0.9, seed=13)
    if name == "block12":         # blocks of 12: padded to 16 columns (one ragged 16-column group), last block 8 wide
        return inputs.dense_lasso(230, 500, nnz_frac=0.02, sigma=0.01, lam_frac=0.05, block=12,
                                  gamma=0.9, seed=15)
    if name == "sparse_logistic":  # config 4 recipe, small
        P = inputs.sparse_logistic(300, 900, density=0.03, seed=6, lam_frac=0.02)
        s, e = P.colptr[100], P.colptr[101]          # make column 100 empty (edge case)
        P.rowidx = np.delete(P.rowidx, np.arange(s, e))
        P.vals = np.delete(P.vals, np.arange(s, e))
        P.colptr[101:] -= e - s
        return P
    if name == "sparse_ls":
        P = inputs.sparse_logistic(250, 400, density=0.05, seed=7)
        A = inputs.csc_to_dense(P)
        xb = inputs.sparse_signal(7, P.n, 12)
        b = A @ xb + 0.01 * np.random.default_rng(7).standard_normal(P.m)
        P.loss, P.scale, P.b = "ls", 0.5, b
        P.lam = 0.05 * float(np.max(np.abs(A.T @ b)))
        P.tau = np.maximum(np.sum(A * A, axis=0), 1e-3)
        return P
    if name == "dense_logistic":
        P = inputs.sparse_logistic(180, 240, density=0.2, seed=8, lam_frac=0.02)
        P.A = inputs.csc_to_dense(P)
        P.kind, P.block = "dense", 4
        return P
    if name in ("dc_exp", "dc_log"):
        P = inputs.nonconvex_box(80, 120, block=1, gamma=0.9, seed=9, lam_frac=0.05)
        P.c, P.lo, P.hi = 0.0, -np.inf, np.inf
        P.reg, P.theta = name[3:], 20.0
        P.lam = 0.1 * P.lam / 20.0
        return P
    raise KeyError(name)
