"""Full-size parity: BASELINE.json configs[1..4] at their real sizes, in the
launch configuration bench.py uses.

  * one synchronous Jacobi sweep (two full GEMVs on the host) -- per-iteration
    parity within 1e-10;
  * one sequential sweep (Algorithm 1, d = 0) -- within 1e-10 (configs[4]: 10^6
    scalar-block updates on both sides);
  * the asynchronous kernel run to the north_star bar: F within 1e-6 relative of
    the oracle's F* (tests/golden/fstar_full.json, written by tools/oracle_fstar.py
    from oracle/ only) and stationarity below 1e-5 (the nonconvex configs[2]: the
    Sec. 4.3 merit, reading R11); at the final iterate F, ||M_F||_2, ||M_F||_inf
    recomputed by the oracle agree with the GPU's stationarity kernel, and the
    maintained residual has not drifted from Ax - b.
"""
import json
import os

import numpy as np
import pytest

from oracle import asyflexa_oracle as O
from paper_1701_04900_b200 import inputs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fstar_full.json")))


@pytest.fixture(scope="module")
def A():
    from paper_1701_04900_b200 import build
    build.build()
    from paper_1701_04900_b200 import asyflexa
    return asyflexa


_cache = {}


def problem(idx):
    if idx not in _cache:
        _cache.clear()
        _cache[idx] = inputs.config(idx)
    return _cache[idx]


def _rel_x(a, b):
    return float(np.max(np.abs(a - b))) / max(1.0, float(np.max(np.abs(b))))


def _rel(a, b):
    return abs(a - b) / max(1.0, abs(b))


def golden_fstar(P, idx):
    """(F*, certified slack): the oracle's F* for configs[idx], after checking that the
    seeded instance is the one the golden was computed on."""
    g = GOLD[f"config{idx}"]
    fp = g["fingerprint"]
    assert (P.m, P.n, P.block, P.gamma) == (fp["m"], fp["n"], fp["block"], fp["gamma"])
    # (b = A x* + e goes through a host BLAS GEMV: bit-identical instances are not guaranteed
    # across machines, ulp-level differences are -- they move F* by ~1e-16 relative)
    for v, key in ((P.lam, "lam"), (float(P.b.sum()), "b_sum"), (float(P.tau.sum()), "tau_sum")):
        assert abs(v - float(fp[key])) <= 1e-12 * max(1.0, abs(float(fp[key]))), (key, v, fp[key])
    # configs[4]: F* is certified only to [F - gap, F] (duality gap of the candidate)
    return float(g["F_star"]), float(g.get("duality_gap", 0.0)) if idx == 4 else 0.0


@pytest.mark.parametrize("idx", [1, 2, 3, 4])
def test_fullsize_jacobi_sweep(A, idx):
    P = problem(idx)
    S = A.Solver(P)
    try:
        st, hist = S.solve(mode=A.ASY_MODE_SYNC_JACOBI, sweeps=1, reset=True, f_hist=True)
        x1 = O.jacobi_step(P, O.default_x0(P), P.gamma)
        assert _rel_x(S.x(), x1) <= 1e-10
        assert _rel(hist[0], O.objective(P, x1)) <= 1e-10
    finally:
        S.close()


@pytest.mark.parametrize("idx", [1, 2, 3, 4])
def test_fullsize_sequential_sweep(A, idx):
    P = problem(idx)
    S = A.Solver(P)
    try:
        S.solve(sweeps=1, reset=True, max_delay=0)
        x_or, _ = O.run_sequential(P, P.gamma, range(P.nblocks))
        assert _rel_x(S.x(), x_or) <= 1e-10
        assert _rel(S.objective(), O.objective(P, x_or)) <= 1e-10
    finally:
        S.close()


# (sweeps budget, sweeps per check): configs[4] needs ~3e4 sweeps to 1e-6 (the l1-logistic
# instance itself: synchronous Jacobi needs as many), ~9 s of kernel time
BUDGET = {1: (200, 5), 2: (4000, 100), 3: (200, 5), 4: (80000, 2000)}


@pytest.mark.parametrize("idx", [1, 2, 3, 4])
def test_fullsize_async_reaches_oracle_fstar(A, idx):
    P = problem(idx)
    F_star, slack = golden_fstar(P, idx)
    S = A.Solver(P)
    total, chunk = BUDGET[idx]
    try:
        S.solve(sweeps=0, reset=True)
        done, ok = 0, False
        while done < total:
            st = S.solve(sweeps=chunk)
            done += chunk
            if (st.objective - F_star) / abs(F_star) > 1e-6 - slack / abs(F_star):
                continue
            out = S.stationarity()
            meas = out.merit_inf if idx == 2 else out.mf_norm2
            if (out.objective - F_star) / abs(F_star) <= 1e-6 - slack / abs(F_star) and meas <= 1e-5:
                ok = True
                break
        assert ok, (idx, done, st.objective, F_star)
        # F below the oracle's F* by more than rounding would mean F* is not the minimum
        assert (out.objective - F_star) / abs(F_star) >= -1e-12 - slack / abs(F_star)
        x = S.x()
        mf = O.stationarity(P, x)
        assert _rel(out.objective, O.objective(P, x)) <= 1e-9
        assert abs(out.mf_norm2 - np.linalg.norm(mf)) <= 1e-6 * max(1.0, np.linalg.norm(mf)) + 1e-12
        assert abs(out.mf_norminf - np.abs(mf).max()) <= 1e-6 * max(1.0, np.abs(mf).max()) + 1e-12
        z = O.design(P) @ x
        fresh = z - P.b if P.loss == "ls" else z
        assert float(np.max(np.abs(S.residual() - fresh))) <= 1e-10 * max(1.0, float(np.max(np.abs(fresh))))
        assert 0 <= st.delay and (st.delay_observed < 0 or st.delay_observed <= st.delay)
    finally:
        S.close()
