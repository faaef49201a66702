"""GPU parity: the CUDA path (through the C ABI) against the oracle.

Bars (BASELINE.json north_star):
  * sequential (async kernel, max_delay = 0) and synchronous Jacobi sweeps match
    the oracle per iteration within 1e-10 relative on x and F;
  * the asynchronous kernel reaches the oracle's final F within 1e-6 relative
    and stationarity below 1e-5.
Inputs are the seeded recipes of paper_1701_04900_b200.inputs (small analogs
of the five configs, spanning several panels / blocks and ragged tails).
"""
import math

import numpy as np
import pytest

from oracle import asyflexa_oracle as O
from paper_1701_04900_b200 import inputs
from cases import fstar, make_case

pytestmark = pytest.mark.gpu

REL = 1e-10


@pytest.fixture(scope="module")
def A():
    from paper_1701_04900_b200 import build
    build.build()
    from paper_1701_04900_b200 import asyflexa
    return asyflexa


def _rel_x(a, b):
    return float(np.max(np.abs(a - b))) / max(1.0, float(np.max(np.abs(b))))


def _rel_f(a, b):
    return abs(a - b) / max(1.0, abs(b))


SEQ_CASES = ["config0", "dense_ragged", "nonconvex", "large_block", "sparse_logistic", "sparse_ls",
             "dense_logistic", "dc_exp", "dc_log", "block12"]


# ----------------------------------------------------------------------------- schedule
@pytest.mark.parametrize("nblocks", [1, 7, 625, 1_000_000])
def test_schedule_device_equals_host(A, nblocks):
    h = A.asy_create(0)
    try:
        for sched in (A.ASY_SCHED_CYCLIC, A.ASY_SCHED_RANDOM):
            k0 = 3 * nblocks + 11
            dev = A.asy_schedule_device(h, sched, 99, nblocks, k0, 5000)
            host = [A.asy_schedule_block(sched, 99, nblocks, k0 + i) for i in range(0, 5000, 37)]
            assert list(dev[::37]) == host
            if nblocks <= 5000 and sched == A.ASY_SCHED_RANDOM:
                ep = dev[(nblocks - k0 % nblocks) % nblocks:][:nblocks]
                if ep.size == nblocks:
                    assert sorted(ep) == list(range(nblocks))
    finally:
        A.asy_destroy(h)


# ----------------------------------------------------------------------------- sequential (delay 0)
@pytest.mark.parametrize("case", SEQ_CASES)
def test_sequential_matches_oracle_per_iteration(A, case):
    """Async kernel with max_delay = 0 == Algorithm 1 with d^k = 0 [PAPER.md:346-357]:
    per-sweep F and x at checkpoints within 1e-10 relative of the oracle."""
    P = make_case(case)
    sweeps = 500 if case == "config0" else 12
    checkpoints = [1, 5, sweeps] if case != "config0" else [1, 50, 500]
    S = A.Solver(P)
    x_or = np.zeros(P.n)
    done = 0
    try:
        S.solve(sweeps=0, reset=True)
        for cp in checkpoints:
            st, hist = S.solve(sweeps=cp - done, max_delay=0, f_hist=True)
            sched = list(O.cyclic_schedule(P.nblocks, cp - done))
            x_or, rec = O.run_sequential(P, P.gamma, sched, x0=x_or, record_every=P.nblocks)
            assert len(rec) == cp - done
            for (k, F_or), F_gpu in zip(rec, hist):
                assert _rel_f(F_gpu, F_or) <= REL, (case, k, F_gpu, F_or)
            assert _rel_x(S.x(), x_or) <= REL, (case, cp)
            assert st.block_updates == (cp - done) * P.nblocks
            done = cp
    finally:
        S.close()


@pytest.mark.parametrize("case", ["dense_ragged", "sparse_logistic"])
def test_sequential_random_schedule(A, case):
    P = make_case(case)
    S = A.Solver(P)
    try:
        S.solve(sweeps=4, max_delay=0, schedule=A.ASY_SCHED_RANDOM, seed=77, reset=True)
        x_or, _ = O.run_sequential(P, P.gamma, O.random_schedule(77, P.nblocks, 4))
        assert _rel_x(S.x(), x_or) <= REL
        assert _rel_f(S.objective(), O.objective(P, x_or)) <= REL
    finally:
        S.close()


def test_sequential_bit_reproducible(A):
    P = make_case("dense_ragged")
    S = A.Solver(P)
    try:
        S.solve(sweeps=3, max_delay=0, reset=True)
        x1 = S.x()
        S.solve(sweeps=3, max_delay=0, reset=True)
        assert np.array_equal(x1, S.x())
    finally:
        S.close()


# ----------------------------------------------------------------------------- Jacobi
JAC_CASES = SEQ_CASES + ["dense_normalized"]


@pytest.mark.parametrize("case", JAC_CASES)
def test_jacobi_matches_oracle_per_iteration(A, case):
    P = make_case(case)
    iters = 25
    S = A.Solver(P)
    try:
        S.solve(sweeps=0, reset=True)
        x_or = np.zeros(P.n)
        st, hist = S.solve(mode=A.ASY_MODE_SYNC_JACOBI, sweeps=iters, f_hist=True)
        _, F_or, xs = O.run_jacobi(P, P.gamma, iters, keep_iterates=True)
        for t in range(iters):
            if not math.isfinite(F_or[t]) or abs(F_or[t]) > 1e200:
                break
            assert _rel_f(hist[t], F_or[t]) <= REL, (case, t, hist[t], F_or[t])
        if math.isfinite(F_or[-1]) and abs(F_or[-1]) < 1e200:
            assert _rel_x(S.x(), xs[-1]) <= REL
    finally:
        S.close()


def test_jacobi_config0_convergent_gamma(A):
    """Jacobi with the config's gamma = 0.9 diverges on configs[0] (both sides);
    with gamma = 0.25 it converges, and parity holds at every one of 300 sweeps."""
    P = inputs.config(0)
    S = A.Solver(P)
    try:
        st, hist = S.solve(mode=A.ASY_MODE_SYNC_JACOBI, sweeps=300, gamma=0.25, f_hist=True, reset=True)
        x_or, F_or, _ = O.run_jacobi(P, 0.25, 300)
        np.testing.assert_array_less(np.abs(hist - F_or) / np.maximum(1, np.abs(F_or)), REL)
        assert _rel_x(S.x(), x_or) <= REL
    finally:
        S.close()


def test_jacobi_bit_reproducible(A):
    P = make_case("sparse_logistic")
    S = A.Solver(P)
    try:
        S.solve(mode=A.ASY_MODE_SYNC_JACOBI, sweeps=5, reset=True)
        x1 = S.x()
        S.solve(mode=A.ASY_MODE_SYNC_JACOBI, sweeps=5, reset=True)
        assert np.array_equal(x1, S.x())
    finally:
        S.close()


# ----------------------------------------------------------------------------- stationarity / objective
@pytest.mark.parametrize("case", SEQ_CASES)
def test_stationarity_matches_oracle(A, case):
    P = make_case(case)
    rng = np.random.default_rng(1)
    lo = -1.0 if np.isfinite(P.lo) else -2.0
    x = rng.uniform(lo, -lo, P.n) * (rng.random(P.n) < 0.3)
    S = A.Solver(P)
    try:
        out = S.stationarity(x)
        mf = O.stationarity(P, x)
        assert _rel_f(out.objective, O.objective(P, x)) <= REL
        assert _rel_f(out.smooth, O.smooth_value(P, x)) <= REL
        assert abs(out.mf_norm2 - np.linalg.norm(mf)) <= REL * max(1, np.linalg.norm(mf))
        assert abs(out.mf_norminf - np.abs(mf).max()) <= REL * max(1, np.abs(mf).max())
        mer = O.merit_inf(P, x)
        assert abs(out.merit_inf - mer) <= REL * max(1, mer)
    finally:
        S.close()


# ----------------------------------------------------------------------------- asynchronous
ASYNC_CASES = ["config0", "dense_ragged", "dense_normalized", "nonconvex", "large_block",
               "sparse_logistic", "sparse_ls", "dense_logistic", "dc_exp", "dc_log", "block12"]


def _residual_drift(A, S, P):
    """max |r_maintained - r(x)| / max(1, |r(x)|) with r(x) = Ax - b (LS) or Ax (logistic)
    recomputed by the oracle's own arithmetic from the kernel's final x."""
    x = S.x()
    z = O.design(P) @ x
    fresh = z - P.b if P.loss == "ls" else z
    return float(np.max(np.abs(S.residual() - fresh))) / max(1.0, float(np.max(np.abs(fresh))))


@pytest.mark.parametrize("schedule", ["cyclic", "random"])
@pytest.mark.parametrize("case", ASYNC_CASES)
def test_async_reaches_oracle_solution(A, case, schedule):
    """Asynchronous runs reach the oracle's F* within 1e-6 and stationarity <= 1e-5 (merit for
    the nonconvex box case, reading R11); the maintained residual has not drifted from Ax - b."""
    P = make_case(case)
    F_star = fstar(P)
    S = A.Solver(P)
    sched = A.ASY_SCHED_CYCLIC if schedule == "cyclic" else A.ASY_SCHED_RANDOM
    rounds = 400 if P.loss == "logistic" else 60  # l1-logistic: ~5e3 sweeps (oracle alike)
    try:
        S.solve(sweeps=0, reset=True)
        ok = False
        for _ in range(rounds):
            st = S.solve(sweeps=100, schedule=sched, seed=3)
            out = S.stationarity()
            meas = out.merit_inf if P.c > 0 else out.mf_norm2
            if _rel_f(out.objective, F_star) <= 1e-6 and meas <= 1e-5:
                ok = True
                break
        assert ok, (case, out.objective, F_star, out.mf_norm2, out.merit_inf)
        assert _residual_drift(A, S, P) <= 1e-10
        if st.delay_observed >= 0:
            assert st.delay_observed <= st.delay
    finally:
        S.close()


def test_async_long_launch_slot_reuse_ragged(A):
    """One launch of 300 sweeps of a ragged-n problem: every accumulator slot is reused
    several times and the ragged last block's slot is next used by full blocks
    (regression: the accumulator half must be cleared over all B entries)."""
    P = make_case("dense_ragged")
    F_star = fstar(P)
    S = A.Solver(P)
    try:
        S.solve(sweeps=300, reset=True)
        out = S.stationarity()
        assert _rel_f(out.objective, F_star) <= 1e-9 and out.mf_norm2 <= 1e-8, (out.objective, F_star, out.mf_norm2)
    finally:
        S.close()


PANEL, SLAB, SLABT = 1, 2, 4  # ASY_KERNEL_DENSE_PANEL / _SLAB (smem/L2 form) / _SLAB_TMEM (asy_tuning.dense_kernel)
DENSE_VARIANTS = {
    # smem / L2 form of the slab kernel
    "slab_hold": {"dense_kernel": SLAB, "slab_hold": 1},          # axpy reads the dot pass's chunk
    "slab_reload": {"dense_kernel": SLAB, "slab_hold": 2},        # axpy re-loads the chunk (L2)
    "slab_chunks": {"dense_kernel": SLAB, "slab_chunk_rows": 8},  # many chunks per sequence
    # TMEM-parking form of the slab kernel (dense_slabt.cuh)
    "slabt": {"dense_kernel": SLABT},
    "slabt_nsw2": {"dense_kernel": SLABT, "slab_ring": 2},
    "panel": {"dense_kernel": PANEL},                             # TMEM panel kernel
    "panel_reread": {"dense_kernel": PANEL, "panel_park": 2},
}


@pytest.mark.parametrize("variant", sorted(DENSE_VARIANTS))
@pytest.mark.parametrize("case", ["dense_ragged", "large_block", "nonconvex", "block12"])
def test_dense_kernel_variants(A, case, variant):
    """Every geometry / code path of the dense asynchronous kernels: sequential parity
    (per iteration) and asynchronous convergence to the oracle's solution."""
    T = DENSE_VARIANTS[variant]
    P = make_case(case)
    S = A.Solver(P)
    try:
        st = S.solve(sweeps=4, max_delay=0, reset=True, tuning=T)
        want = {PANEL: [A.ASY_KERNEL_DENSE_PANEL], SLAB: [A.ASY_KERNEL_DENSE_SLAB],
                SLABT: [A.ASY_KERNEL_DENSE_SLAB_TMEM, A.ASY_KERNEL_DENSE_SLAB]}[T["dense_kernel"]]
        assert st.kernel in want
        x_or, _ = O.run_sequential(P, P.gamma, O.cyclic_schedule(P.nblocks, 4))
        assert _rel_x(S.x(), x_or) <= REL
        F_star = fstar(P)
        S.solve(sweeps=0, reset=True)
        for _ in range(60):
            S.solve(sweeps=100, schedule=A.ASY_SCHED_RANDOM, seed=5, tuning=T)
            out = S.stationarity()
            meas = out.merit_inf if P.c > 0 else out.mf_norm2
            if _rel_f(out.objective, F_star) <= 1e-6 and meas <= 1e-5:
                break
        assert _rel_f(out.objective, F_star) <= 1e-6 and meas <= 1e-5
    finally:
        S.close()


@pytest.mark.parametrize("kernel", ["slab", "slab_smem", "panel"])
@pytest.mark.parametrize("workers", [1, 3, 37])
def test_dense_few_workers(A, workers, kernel):
    """Fewer CTAs than SMs (taller row slabs / fewer panel workers), same results."""
    T = {"dense_kernel": {"slab": SLABT, "slab_smem": SLAB, "panel": PANEL}[kernel]}
    P = make_case("dense_ragged")
    S = A.Solver(P)
    try:
        S.solve(sweeps=3, max_delay=0, reset=True, workers=workers, tuning=T)
        x_or, _ = O.run_sequential(P, P.gamma, O.cyclic_schedule(P.nblocks, 3))
        assert _rel_x(S.x(), x_or) <= REL
        S.solve(sweeps=200, reset=True, workers=workers, schedule=A.ASY_SCHED_RANDOM, seed=1, tuning=T)
        F_star = fstar(P)
        out = S.stationarity()
        assert _rel_f(out.objective, F_star) <= 1e-6 and out.mf_norm2 <= 1e-5
    finally:
        S.close()


@pytest.mark.parametrize("case,workers", [("tall_block", 1), ("large_block", 2), ("large_block", 3), ("large_block", 7),
                                          ("dense_ragged", 1), ("dense_ragged", 2), ("nonconvex", 1),
                                          ("dense_logistic", 1), ("box64", 1), ("box64", 2), ("block100", 1),
                                          ("block100", 3), ("block100", 0), ("dc_exp", 1), ("dc_log", 2)])
def test_slab_tmem_tall_slabs(A, case, workers):
    """TMEM-parking slab kernel with tall slabs: several 32-row groups per dot warp, a ragged
    last group (1-D bulk copies), hold slots in shared memory when a warp owns more groups than
    its TMEM lane quarter holds (tall_block, 1 worker: 9 groups of 128 columns), park rings
    that wrap many times.  Sequential parity per sweep, then asynchronous convergence."""
    T = {"dense_kernel": SLABT}
    P = make_case(case)
    S = A.Solver(P)
    try:
        for sweeps in (1, 3):
            st = S.solve(sweeps=sweeps, max_delay=0, reset=True, workers=workers, tuning=T)
            assert st.kernel == A.ASY_KERNEL_DENSE_SLAB_TMEM
            x_or, _ = O.run_sequential(P, P.gamma, O.cyclic_schedule(P.nblocks, sweeps))
            assert _rel_x(S.x(), x_or) <= REL
        F_star = fstar(P)
        S.solve(sweeps=0, reset=True)
        for _ in range(60):
            st = S.solve(sweeps=100, workers=workers, schedule=A.ASY_SCHED_RANDOM, seed=3, tuning=T)
            assert 0 <= st.delay_observed <= st.delay  # Assumption D1 holds as enforced
            out = S.stationarity()
            meas = out.merit_inf if P.c > 0 else out.mf_norm2
            if _rel_f(out.objective, F_star) <= 1e-6 and meas <= 1e-5:
                break
        assert _rel_f(out.objective, F_star) <= 1e-6 and meas <= 1e-5
    finally:
        S.close()


@pytest.mark.parametrize("case,workers", [("tall_block", 1), ("large_block", 3), ("box64", 2), ("dense_ragged", 1)])
def test_slab_tmem_sequential_random_schedule(A, case, workers):
    """TMEM slab kernel, sequential mode, seeded Philox/Feistel schedule: D4 through the inverse
    permutation (schedule_prev) and the rotating partial round of groups, per-sweep parity."""
    T = {"dense_kernel": SLABT}
    P = make_case(case)
    S = A.Solver(P)
    try:
        st = S.solve(sweeps=3, max_delay=0, schedule=A.ASY_SCHED_RANDOM, seed=41, reset=True, workers=workers, tuning=T)
        assert st.kernel == A.ASY_KERNEL_DENSE_SLAB_TMEM
        assert st.delay_observed == 0  # sequential: every read sees all earlier updates
        x_or, _ = O.run_sequential(P, P.gamma, O.random_schedule(41, P.nblocks, 3))
        assert _rel_x(S.x(), x_or) <= REL
        assert _rel_f(S.objective(), O.objective(P, x_or)) <= REL
    finally:
        S.close()


def test_slab_fallback_when_too_tall(A):
    """A slab of 19 row groups (> 4 per dot warp) does not fit the TMEM park ring: the
    dispatcher falls back to the smem/L2 slab form, with the same results."""
    T = {"dense_kernel": SLABT}
    P = make_case("tall600")
    S = A.Solver(P)
    try:
        st = S.solve(sweeps=3, max_delay=0, reset=True, workers=1, tuning=T)
        assert st.kernel == A.ASY_KERNEL_DENSE_SLAB and st.delay_observed == -1
        x_or, _ = O.run_sequential(P, P.gamma, O.cyclic_schedule(P.nblocks, 3))
        assert _rel_x(S.x(), x_or) <= REL
        st = S.solve(sweeps=3, max_delay=0, reset=True, workers=8, tuning=T)  # 3 groups per slab: TMEM form
        assert st.kernel == A.ASY_KERNEL_DENSE_SLAB_TMEM
        assert _rel_x(S.x(), x_or) <= REL
    finally:
        S.close()


def test_async_delay_window_respected_tiny(A):
    """configs[0] with all CTAs and an unbounded window diverges like Jacobi;
    the default window (N/8) converges (Theorem 1: gamma vs delta [PAPER.md:301])."""
    P = inputs.config(0)
    S = A.Solver(P)
    try:
        S.solve(sweeps=200, reset=True)
        out = S.stationarity()
        assert out.mf_norm2 <= 1e-5
    finally:
        S.close()


# ----------------------------------------------------------------------------- edge cases
def test_edge_cases(A):
    # m = 1, n = 1
    P = inputs.Problem(name="1x1", kind="dense", m=1, n=1, loss="ls", scale=0.5, b=np.array([3.0]),
                       lam=1.0, tau=np.array([4.0]), block=1, gamma=1.0,
                       A=np.asfortranarray([[2.0]]))
    S = A.Solver(P)
    S.solve(sweeps=50, reset=True, max_delay=0)
    np.testing.assert_allclose(S.x(), [1.25], atol=1e-12)  # argmin 1/2(2x-3)^2 + |x| -> x = (6-1)/4
    S.close()
    # lambda huge -> x stays 0; degenerate box lo = hi
    P = make_case("dense_ragged")
    P.lam = 1e12
    S = A.Solver(P)
    S.solve(sweeps=3, reset=True)
    assert np.all(S.x() == 0)
    S.close()
    P = make_case("dense_ragged")
    P.lo, P.hi = 0.25, 0.25
    S = A.Solver(P)
    S.solve(sweeps=2, reset=True)
    assert np.all(S.x() == 0.25)
    S.close()
    # empty columns in CSC
    P = make_case("sparse_logistic")
    cnt = np.diff(P.colptr)
    assert np.any(cnt == 0)
    S = A.Solver(P)
    S.solve(sweeps=3, reset=True, max_delay=0)
    x_or, _ = O.run_sequential(P, P.gamma, O.cyclic_schedule(P.nblocks, 3))
    assert _rel_x(S.x(), x_or) <= REL
    S.close()


def test_invalid_arguments(A):
    P = make_case("dense_ragged")
    bad = P.tau.copy()
    bad[5] = 0.0
    P.tau = bad
    with pytest.raises(A.AsyError) as e:
        A.Solver(P)
    assert e.value.code == A.ASY_ERR_INVALID
    P = make_case("dense_ragged")
    S = A.Solver(P)
    with pytest.raises(A.AsyError):
        S.solve(gamma=0.0)
    with pytest.raises(A.AsyError):
        S.solve(gamma=1.5)
    with pytest.raises(A.AsyError):
        S.solve(panel_rows=48)
    # a (panel_rows, stages) pair with no compiled kernel is refused, not silently replaced
    with pytest.raises(A.AsyError) as e:
        S.solve(panel_rows=32, tuning={"dense_kernel": PANEL})
    assert e.value.code == A.ASY_ERR_UNSUPPORTED
    with pytest.raises(A.AsyError) as e:
        S.solve(stages=6, tuning={"dense_kernel": PANEL})
    assert e.value.code == A.ASY_ERR_UNSUPPORTED
    with pytest.raises(A.AsyError) as e:
        S.solve(tuning={"dense_kernel": 3})
    assert e.value.code == A.ASY_ERR_INVALID
    st = S.solve(sweeps=1, panel_rows=96, tuning={"dense_kernel": PANEL})  # (32, 3, 8) is compiled
    assert st.kernel == A.ASY_KERNEL_DENSE_PANEL
    S.close()
    P.block = 0
    with pytest.raises(A.AsyError):
        A.Solver(P)


def test_host_and_device_problem_agree(A):
    P = make_case("dense_ragged")
    S1, S2 = A.Solver(P, mem="device"), A.Solver(P, mem="host")
    try:
        S1.solve(sweeps=4, max_delay=0, reset=True)
        S2.solve(sweeps=4, max_delay=0, reset=True)
        assert np.array_equal(S1.x(), S2.x())
    finally:
        S1.close()
        S2.close()


def test_panel_kernel_too_many_panels_never_hangs(A):
    """Blocks of 128 columns x 8000 rows = 250 panels of 32 rows (the panel kernel's shape at
    55 KB per SM): with 1 worker the panels of one block exceed the hand-off capacity, so the
    dispatcher must refuse (the row slab of 8000 rows does not fit one SM either) instead of
    deadlocking; with 2 workers it falls back to the row-slab kernel; with 8 the panel kernel
    runs.  Sequential parity in both runnable cases."""
    P = inputs.dense_lasso(8000, 384, nnz_frac=0.02, sigma=0.01, lam_frac=0.05, block=128, gamma=0.9, seed=3)
    S = A.Solver(P)
    try:
        with pytest.raises(A.AsyError) as e:
            S.solve(sweeps=1, reset=True, workers=1, max_delay=0)
        assert e.value.code == A.ASY_ERR_UNSUPPORTED
        x_or, _ = O.run_sequential(P, P.gamma, O.cyclic_schedule(P.nblocks, 2))
        st = S.solve(sweeps=2, reset=True, workers=2, max_delay=0)
        assert st.kernel in (A.ASY_KERNEL_DENSE_SLAB, A.ASY_KERNEL_DENSE_SLAB_TMEM)
        assert _rel_x(S.x(), x_or) <= REL
        st = S.solve(sweeps=2, reset=True, workers=8, max_delay=0)
        assert st.kernel == A.ASY_KERNEL_DENSE_PANEL
        assert _rel_x(S.x(), x_or) <= REL
    finally:
        S.close()


@pytest.mark.parametrize("case,schedule", [("config0", "cyclic"), ("dense_ragged", "random"), ("large_block", "cyclic"),
                                           ("sparse_logistic", "cyclic"), ("sparse_ls", "random")])
def test_observed_delay_panel_and_csc(A, case, schedule):
    """Observed delay (Assumption D1's d^k [PAPER.md:224]) of the panel and CSC kernels in
    measurement mode (asy_tuning.measure_delay): 0 in sequential mode, within the enforced bound
    otherwise, and not measured (-1) by default; the measurement does not change the iterates
    of the sequential mode."""
    P = make_case(case)
    S = A.Solver(P)
    sched = A.ASY_SCHED_CYCLIC if schedule == "cyclic" else A.ASY_SCHED_RANDOM
    T = {"dense_kernel": A.ASY_KERNEL_DENSE_PANEL} if P.kind == "dense" else {}
    try:
        st = S.solve(sweeps=2, max_delay=0, reset=True, schedule=sched, seed=5, tuning=dict(T, measure_delay=1))
        assert st.kernel in (A.ASY_KERNEL_DENSE_PANEL, A.ASY_KERNEL_SPARSE)
        assert st.delay_observed == 0
        x_meas = S.x()
        st = S.solve(sweeps=2, max_delay=0, reset=True, schedule=sched, seed=5, tuning=T or None)
        assert st.delay_observed == -1
        assert np.array_equal(S.x(), x_meas)
        st = S.solve(sweeps=20, reset=True, schedule=sched, seed=5, tuning=dict(T, measure_delay=1))
        assert 0 <= st.delay_observed <= st.delay
    finally:
        S.close()
