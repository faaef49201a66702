"""Pins for the oracle (CPU, -m "not gpu").

Each test ties an oracle function to something other than itself: a
hand-derived worked example, a closed form, brute-force minimisation, finite
differences, an independent library solver (scikit-learn) or an invariant the
paper states.  A plausible mistake (dropped term, wrong sign/index, transposed
operand, wrong factor 2) fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import asyflexa_oracle as O
from paper_1701_04900_b200 import inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold_problem(d):
    A = np.asfortranarray(np.array(d["A"], float))
    return inputs.Problem(name="gold", kind="dense", m=2, n=2, loss="ls", scale=0.5,
                          b=np.array(d["b"]), lam=d["lambda"], tau=np.array(d["tau"]),
                          block=1, gamma=1.0, A=A)


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(GOLD, "lasso_2x2.json")) as f:
        return json.load(f)


# --------------------------------------------------------------------------- worked example
def test_golden_jacobi_and_sequential(gold):
    P = _gold_problem(gold)
    assert O.objective(P, np.zeros(2)) == gold["F0"]
    for key, gamma in (("jacobi_gamma1", 1.0), ("jacobi_gamma05", 0.5)):
        x, Fs, xs = O.run_jacobi(P, gamma, 2, keep_iterates=True)
        for t in range(2):
            np.testing.assert_allclose(xs[t], gold[key]["x"][t], rtol=0, atol=1e-15)
            assert abs(Fs[t] - gold[key]["F"][t]) <= 1e-15
    x = np.zeros(2)
    for s in range(2):
        x, _ = O.run_sequential(P, 1.0, [0, 1], x0=x)
        np.testing.assert_allclose(x, gold["sequential_gamma1_cyclic"]["x"][s], atol=1e-15)
        assert abs(O.objective(P, x) - gold["sequential_gamma1_cyclic"]["F"][s]) <= 1e-15


def test_golden_solution(gold):
    P = _gold_problem(gold)
    x, F, _ = O.estimate_fstar(P, 1.0)
    np.testing.assert_allclose(x, gold["solution"], atol=1e-12)
    assert abs(F - gold["Fstar"]) <= 1e-12
    assert np.abs(O.stationarity(P, np.array(gold["solution"]))).max() <= 1e-15


# --------------------------------------------------------------------------- soft threshold / subproblem
def test_soft_threshold_examples():
    assert O.soft_threshold(3.0, 1.0) == 2.0
    assert O.soft_threshold(-0.5, 1.0) == 0.0
    assert O.soft_threshold(0.0, 0.0) == 0.0
    assert O.soft_threshold(-3.0, 1.0) == -2.0
    assert O.soft_threshold(1.0, 1.0) == 0.0  # boundary -> exact zero
    rng = np.random.default_rng(0)
    a, b, t = rng.normal(size=(3, 100000))
    t = np.abs(t)
    assert np.all(np.abs(O.soft_threshold(a, t) - O.soft_threshold(b, t)) <= np.abs(a - b) + 1e-15)


def _brute_scalar(g, y, tau, lam, lo, hi):
    """Minimise q(t) = g(t-y) + tau/2(t-y)^2 + lam|t| over [lo,hi] by dense
    grid search + golden-section refinement (no closed form used)."""
    a = max(lo, y - 50.0) if np.isfinite(lo) else y - 50.0
    bnd = min(hi, y + 50.0) if np.isfinite(hi) else y + 50.0
    q = lambda t: g * (t - y) + 0.5 * tau * (t - y) ** 2 + lam * np.abs(t)
    grid = np.linspace(a, bnd, 200001)
    grid = np.concatenate([grid, [0.0] if a <= 0.0 <= bnd else []])
    i = int(np.argmin(q(grid)))
    t0 = grid[i]
    if t0 == 0.0 and q(0.0) <= q(grid).min():
        return 0.0
    step = grid[1] - grid[0]
    l, r = max(a, t0 - step), min(bnd, t0 + step)
    phi = (math.sqrt(5) - 1) / 2
    for _ in range(200):
        c, d = r - phi * (r - l), l + phi * (r - l)
        if q(c) < q(d):
            r = d
        else:
            l = c
    return 0.5 * (l + r)


@pytest.mark.parametrize("seed", range(6))
def test_subproblem_vs_bruteforce(seed):
    rng = np.random.default_rng(seed)
    for _ in range(40):
        g, y = rng.normal(scale=3, size=2)
        tau = rng.uniform(0.2, 5)
        lam = rng.choice([0.0, rng.uniform(0, 4)])
        lo, hi = rng.choice([(-np.inf, np.inf), (-1.0, 1.0), (0.2, 3.0), (-2.0, -0.5)])
        ours = float(O.scalar_subproblem_argmin(g, y, tau, lam, lo, hi))
        brute = _brute_scalar(g, y, tau, lam, lo, hi)
        assert abs(ours - brute) <= 1e-6, (g, y, tau, lam, lo, hi, ours, brute)


def test_subproblem_special_cases():
    # lam = 0, no box: pure proximal-linear (Newton-like) step y - g/tau
    assert O.scalar_subproblem_argmin(2.0, 1.0, 4.0, 0.0, -np.inf, np.inf) == 0.5
    # grad 0 at y = 0 stays at 0
    assert O.scalar_subproblem_argmin(0.0, 0.0, 1.0, 1.0, -np.inf, np.inf) == 0.0
    # degenerate box lo = hi
    assert O.scalar_subproblem_argmin(5.0, 0.0, 1.0, 0.1, 0.3, 0.3) == 0.3


# --------------------------------------------------------------------------- gradients
def _fd_grad(P, x, h=1e-6):
    g = np.zeros_like(x)
    for j in range(x.size):
        e = np.zeros_like(x)
        e[j] = h
        g[j] = (O.smooth_value(P, x + e) - O.smooth_value(P, x - e)) / (2 * h)
    return g


@pytest.mark.parametrize("case", ["lasso", "nonconvex", "logistic"])
def test_gradient_finite_difference(case):
    if case == "lasso":
        P = inputs.dense_lasso(7, 5, nnz_frac=0.4, sigma=0.1, lam_frac=0.1, block=2, seed=1)
    elif case == "nonconvex":
        P = inputs.nonconvex_box(7, 9, block=3, seed=2)
    else:
        P = inputs.sparse_logistic(9, 6, density=0.5, seed=3)
    x = np.random.default_rng(5).uniform(-0.8, 0.8, P.n)
    g = O.smooth_grad(P, x)
    fd = _fd_grad(P, x)
    assert np.max(np.abs(g - fd)) <= 1e-6 * max(1.0, np.max(np.abs(g)))


# --------------------------------------------------------------------------- closed forms / library solvers
def test_identity_design_closed_form():
    """A = I: the LASSO solution is S_lam(b); with tau = ||a_j||^2 = 1 and gamma = 1
    one Jacobi step from any point lands on it."""
    n = 11
    b = np.random.default_rng(2).normal(size=n) * 2
    P = inputs.Problem(name="eye", kind="dense", m=n, n=n, loss="ls", scale=0.5, b=b,
                       lam=0.7, tau=np.ones(n), block=3, gamma=1.0,
                       A=np.asfortranarray(np.eye(n)))
    x, _, _ = O.run_jacobi(P, 1.0, 1, x0=np.random.default_rng(3).normal(size=n))
    np.testing.assert_allclose(x, np.sign(b) * np.maximum(np.abs(b) - 0.7, 0), atol=1e-15)


def test_lasso_matches_sklearn_and_kkt():
    from sklearn.linear_model import Lasso
    P = inputs.dense_lasso(60, 120, nnz_frac=0.05, sigma=0.01, lam_frac=0.1, block=1, seed=3)
    x, F, _ = O.estimate_fstar(P, 1.0, max_sweeps=3000, tol=0.0)
    las = Lasso(alpha=P.lam / P.m, fit_intercept=False, tol=1e-14, max_iter=1000000).fit(P.A, P.b)
    assert np.max(np.abs(las.coef_ - x)) <= 1e-7
    assert abs(O.objective(P, las.coef_) - F) <= 1e-10 * abs(F)
    # LASSO KKT [north_star]: |A^T r|_i <= lam off-support, = -lam sign(x_i) on support
    g = P.A.T @ (P.A @ x - P.b)
    off = x == 0
    assert np.all(np.abs(g[off]) <= P.lam * (1 + 1e-9))
    np.testing.assert_allclose(g[~off], -P.lam * np.sign(x[~off]), rtol=1e-8, atol=1e-8)


def test_logistic_matches_sklearn():
    import warnings
    from sklearn.linear_model import LogisticRegression
    Q = inputs.sparse_logistic(120, 60, density=0.08, seed=1, lam_frac=0.05)
    x, F, _ = O.estimate_fstar(Q, 1.0, max_sweeps=100000, tol=1e-15)
    Ad = inputs.csc_to_dense(Q)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        lr = LogisticRegression(l1_ratio=1.0, C=1 / (Q.m * Q.lam), solver="liblinear",
                                fit_intercept=False, tol=1e-12, max_iter=100000).fit(Ad, Q.b)
    Fsk = O.objective(Q, lr.coef_[0])
    assert F <= Fsk + 1e-12 and (Fsk - F) <= 1e-9 * abs(F)
    assert np.linalg.norm(O.stationarity(Q, x)) <= 1e-7


# --------------------------------------------------------------------------- paper invariants
def test_monotone_decrease_small_gamma():
    """Sequential (d=0) updates with a small fixed gamma decrease F at every
    update (Prop. 1 [PAPER.md:600-606] + descent lemma)."""
    P = inputs.nonconvex_box(30, 50, block=4, seed=4)
    x = np.zeros(P.n)
    Fprev = O.objective(P, x)
    for k, i in enumerate(O.cyclic_schedule(P.nblocks, 6)):
        x, _ = O.run_sequential(P, 0.5, [i], x0=x)
        F = O.objective(P, x)
        assert F <= Fprev + 1e-9 * abs(Fprev), (k, F, Fprev)
        Fprev = F


def test_descent_inequality_prop1():
    """(hat x_i - y_i)^T grad_i f(y) + g(hat x_i) - g(y_i) <= -c ||hat x_i - y_i||^2
    with c = min tau / 2 (strong convexity of the surrogate) [PAPER.md:604]."""
    P = inputs.dense_lasso(20, 30, nnz_frac=0.2, sigma=0.1, lam_frac=0.2, block=5, seed=6)
    rng = np.random.default_rng(7)
    for _ in range(20):
        y = rng.normal(size=P.n)
        g = O.smooth_grad(P, y)
        for i in range(P.nblocks):
            j0, j1 = P.block_range(i)
            xh = O.best_response(P, i, y, g[j0:j1])
            d = xh - y[j0:j1]
            lhs = d @ g[j0:j1] + P.lam * (np.abs(xh).sum() - np.abs(y[j0:j1]).sum())
            assert lhs <= -0.5 * P.tau[j0:j1].min() * (d @ d) + 1e-9


def test_fixed_point_is_prox_stationary():
    """At the limit of the block map, hat x(x) = x and M_F(x) = 0 (Eq. 5
    [PAPER.md:291]), and M_F = 0 <=> the box-constrained KKT conditions,
    written out case by case."""
    P = inputs.nonconvex_box(25, 40, block=5, seed=8, lam_frac=0.3)
    x, F, sweeps = O.estimate_fstar(P, 0.9, max_sweeps=50000, tol=0.0)
    assert O.merit_inf(P, x) <= 1e-10
    assert np.abs(O.stationarity(P, x)).max() <= 1e-8
    g = O.smooth_grad(P, x)
    tol = 1e-7 * max(1, np.abs(g).max())
    for j in range(P.n):
        # with gamma < 1 an inactive coordinate decays as (1-gamma)^k, never exactly 0
        if -1 < x[j] < 1:
            if abs(x[j]) <= 1e-12:
                assert abs(g[j]) <= P.lam + tol
            else:
                assert abs(g[j] + P.lam * np.sign(x[j])) <= tol
        elif x[j] == 1:
            assert g[j] + P.lam <= tol
        else:
            assert g[j] - P.lam >= -tol


def test_stationarity_1d_examples():
    def one(lam, x):
        P = inputs.Problem(name="1d", kind="dense", m=1, n=1, loss="ls", scale=0.5,
                           b=np.array([1.0]), lam=lam, tau=np.ones(1), block=1,
                           gamma=1.0, A=np.ones((1, 1), order="F"))
        return float(O.stationarity(P, np.array([x]))[0])
    assert one(0.0, 1.0) == 0.0          # f = 1/2 (x-1)^2 at its minimiser
    assert one(2.0, 0.0) == 0.0          # |f'(0)| = 1 <= lam: origin stationary
    assert abs(one(0.5, 0.0) + 0.5) < 1e-15  # y = S_0.5(1) = 0.5 -> M_F = -0.5


def test_local_min_bruteforce_nonconvex():
    """Tiny box-constrained nonconvex instance: the oracle's limit is no worse
    than every point of a fine grid around it (local minimality) and the
    global grid minimum is itself prox-stationary."""
    P = inputs.nonconvex_box(3, 2, block=1, seed=11, lam_frac=0.05)
    x, F, _ = O.estimate_fstar(P, 0.9, max_sweeps=100000, tol=0.0)
    g1 = np.linspace(-1, 1, 801)
    X, Y = np.meshgrid(g1, g1)
    vals = np.array([[O.objective(P, np.array([a, b])) for a, b in zip(r1, r2)]
                     for r1, r2 in zip(X, Y)])
    near = (np.abs(X - x[0]) <= 0.02) & (np.abs(Y - x[1]) <= 0.02)
    assert F <= vals[near].min() + 1e-12
    i, j = np.unravel_index(np.argmin(vals), vals.shape)
    xg = np.array([X[i, j], Y[i, j]])
    assert np.abs(O.stationarity(P, xg)).max() <= 0.05 * max(1, np.abs(O.smooth_grad(P, xg)).max())


def test_carried_residual_equals_definition():
    P = inputs.nonconvex_box(15, 21, block=4, seed=9)
    sched = list(O.cyclic_schedule(P.nblocks, 4))
    xa, _ = O.run_sequential(P, 0.5, sched)
    xb, _ = O.run_sequential(P, 0.5, sched, refresh_every=1)
    np.testing.assert_allclose(xa, xb, rtol=0, atol=1e-12 * max(1, np.abs(xb).max()))


# --------------------------------------------------------------------------- DC regularizers (Sec. 4.3)
@pytest.mark.parametrize("reg", ["exp", "log"])
def test_dc_identity_and_gradient(reg):
    P = inputs.Problem(name="dc", kind="dense", m=1, n=1, loss="ls", scale=1.0,
                       b=np.zeros(1), lam=1.0, tau=np.ones(1), block=1, gamma=1.0,
                       reg=reg, theta=20.0)
    t = np.random.default_rng(0).normal(scale=2, size=10000)
    assert np.max(np.abs(O.h_plus(P, t) - O.h_minus(P, t) - O.h(P, t))) <= 1e-12 * 50
    tt = np.linspace(0.01, 3, 200)
    fd = (O.h_minus(P, tt + 1e-6) - O.h_minus(P, tt - 1e-6)) / 2e-6
    np.testing.assert_allclose(O.grad_h_minus(P, tt), fd, rtol=1e-6, atol=1e-8)
    assert O.grad_h_minus(P, np.array([0.0]))[0] == 0.0
    assert np.all(np.diff(O.grad_h_minus(P, np.linspace(-3, 3, 1001))) >= -1e-12)  # h^- convex
    if reg == "exp":
        assert abs(O.eta(P) - 20.0) < 1e-15
    else:
        assert abs(O.eta(P) - 20.0 / math.log(21.0)) < 1e-15


@pytest.mark.parametrize("reg", ["exp", "log"])
def test_dc_best_response_bruteforce(reg):
    """Eq. (13) [PAPER.md:534-541]: argmin g(t-y) - lam h^-'(y)(t-y) + lam h^+(t) + tau/2 (t-y)^2."""
    rng = np.random.default_rng(1)
    for _ in range(30):
        y, g = rng.normal(size=2)
        tau = rng.uniform(0.5, 3)
        P = inputs.Problem(name="dc", kind="dense", m=1, n=1, loss="ls", scale=1.0,
                           b=np.zeros(1), lam=0.1, tau=np.array([tau]), block=1,
                           gamma=1.0, reg=reg, theta=20.0)
        ours = float(O.best_response(P, 0, np.array([y]), np.array([g]))[0])
        gl = g - P.lam * float(O.grad_h_minus(P, np.array([y]))[0])
        brute = _brute_scalar(gl, y, tau, P.lam * O.eta(P), -np.inf, np.inf)
        assert abs(ours - brute) <= 1e-6


# --------------------------------------------------------------------------- oracle solves config 0
def test_config0_oracle_converges():
    """BASELINE configs[0] (Tiny LASSO, 500 sweeps, gamma 0.9): the oracle's run
    reaches a KKT point and sklearn agrees."""
    from sklearn.linear_model import Lasso
    P = inputs.config(0)
    x, _ = O.run_sequential(P, P.gamma, O.cyclic_schedule(P.nblocks, 60))
    assert np.linalg.norm(O.stationarity(P, x)) <= 1e-9
    las = Lasso(alpha=P.lam / P.m, fit_intercept=False, tol=1e-14, max_iter=10 ** 6).fit(P.A, P.b)
    assert abs(O.objective(P, las.coef_) - O.objective(P, x)) <= 1e-10 * O.objective(P, x)


# --------------------------------------------------------------------------- hand-derived M_F / merit / G / x0 / rel. error
# (tests/golden_cases.py; derivations in tests/golden/README.md "1-D / 2-D stationarity pins")
from golden_cases import MERIT_CASES, MF_CASES  # noqa: E402


@pytest.mark.parametrize("name,P,x,want", MF_CASES, ids=[c[0] for c in MF_CASES])
def test_stationarity_hand_derived(name, P, x, want):
    """M_F of Eq. (5) [PAPER.md:287-290] with the box X active and with the DC shift
    -lam grad h^-(x) of Eq. (13) [PAPER.md:534-541] at x != 0 (both signs)."""
    got = O.stationarity(P, np.array(x, float))
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-15)


@pytest.mark.parametrize("name,P,x,want", MERIT_CASES, ids=[c[0] for c in MERIT_CASES])
def test_merit_hand_derived(name, P, x, want):
    """Nonzero values of the Sec. 4.3 merit ||hat x(x) - x||_inf [PAPER.md:549]."""
    assert abs(O.merit_inf(P, np.array(x, float)) - want) <= 1e-15


def test_G_indicator_outside_box():
    """G = lam sum h(x_j) on X, +inf outside (problem (1) [PAPER.md:58-68], X_i closed convex)."""
    from golden_cases import problem
    P = problem(np.eye(2), [0.0, 0.0], lam=2.0, lo=-1.0, hi=1.0)
    assert O.G(P, np.array([0.5, -1.0])) == 3.0
    assert O.G(P, np.array([0.5, 1.5])) == math.inf
    assert O.G(P, np.array([-1.0 - 1e-12, 0.0])) == math.inf
    assert O.objective(P, np.array([2.0, 0.0])) == math.inf
    Q = problem(np.eye(2), [0.0, 0.0], lam=1.0, lo=np.array([0.0, -3.0]), hi=np.array([1.0, -2.0]))
    assert O.G(Q, np.array([0.5, -2.5])) == 3.0
    assert O.G(Q, np.array([0.5, -1.5])) == math.inf


def test_default_x0_is_projection_of_zero():
    """x^0 = P_X(0) [PAPER.md:250]: a box that excludes 0 moves it to the nearer bound."""
    from golden_cases import problem
    assert list(O.default_x0(problem(np.eye(3), [0, 0, 0], lam=0.1, lo=0.2, hi=3.0))) == [0.2] * 3
    assert list(O.default_x0(problem(np.eye(3), [0, 0, 0], lam=0.1, lo=-2.0, hi=-0.5))) == [-0.5] * 3
    P = problem(np.eye(3), [0, 0, 0], lam=0.1, lo=np.array([0.25, -1.0, -4.0]), hi=np.array([1.0, 1.0, -3.0]))
    assert list(O.default_x0(P)) == [0.25, 0.0, -3.0]


def test_relative_error_definition():
    """(F - F*)/|F*| of Sec. 4.2 [PAPER.md:451], including |F*| < 1 and F* < 0."""
    assert O.relative_error(1.5, 0.5) == 2.0
    assert O.relative_error(0.75, 0.25) == 2.0
    assert O.relative_error(-0.9, -1.0) == pytest.approx(0.1, abs=1e-15)
    assert O.relative_error(0.02, 0.01) == 1.0
    assert O.relative_error(3.0, 3.0) == 0.0


# --------------------------------------------------------------------------- duality certificate (convex l1 configs)
def test_dual_value_hand_derived():
    """1-D LASSO 1/2(x-3)^2 + |x|: x* = 2, F* = 5/2, dual u* = -1, D = -b u - u^2/2 = 5/2;
    from x the dual point is u0 = x - 3 scaled by min(1, 1/|u0|).
    1-D logistic log(1+e^-x) + x/5 (m = 1, y = 1): x* = log 4, F* = log 5 - 1.6 log 2,
    theta* = sigmoid(-x*) = 1/5 and D = -(0.2 log 0.2 + 0.8 log 0.8) = F*; from x = 0 the scaled
    dual point is theta = 0.5 * min(1, 0.2/0.5) = 0.2, i.e. already the optimum."""
    from golden_cases import problem
    P = problem([[1.0]], [3.0], lam=1.0)
    for x in (0.0, 1.0, 2.0):  # u0 = x - 3 <= -1: scaled to u = -1
        assert abs(O.dual_value_l1(P, np.array([x])) - 2.5) <= 1e-15
    assert abs(O.dual_value_l1(P, np.array([2.5])) - 1.375) <= 1e-15  # u = -1/2 feasible: 3/2 - 1/8
    assert abs(O.dual_value_l1(P, np.array([5.0])) + 3.5) <= 1e-15    # u0 = 2 -> u = 1: -3 - 1/2
    assert abs(O.duality_gap_l1(P, np.array([2.0]))) <= 1e-15
    Q = inputs.Problem(name="lg1", kind="dense", m=1, n=1, loss="logistic", scale=1.0, b=np.array([1.0]),
                       lam=0.2, tau=np.ones(1), block=1, gamma=1.0, A=np.ones((1, 1), order="F"))
    Fstar = math.log(5.0) - 1.6 * math.log(2.0)
    assert abs(O.objective(Q, np.array([math.log(4.0)])) - Fstar) <= 1e-15
    for x in (0.0, 1.0, math.log(4.0)):
        assert abs(O.dual_value_l1(Q, np.array([x])) - Fstar) <= 1e-15


@pytest.mark.parametrize("kind", ["ls", "logistic"])
def test_weak_duality_and_zero_gap_at_optimum(kind):
    """D(u(x)) <= F* <= F(x) for arbitrary x (weak duality), and the gap closes at the
    oracle's own Algorithm 1 limit (strong duality for these convex instances)."""
    if kind == "ls":
        P = inputs.dense_lasso(40, 90, nnz_frac=0.05, sigma=0.01, lam_frac=0.1, block=3, seed=21)
    else:
        P = inputs.sparse_logistic(80, 50, density=0.1, seed=22, lam_frac=0.05)
    xs, Fs, _ = O.estimate_fstar(P, 1.0, max_sweeps=20000, tol=0.0)  # until F stops changing at all
    rng = np.random.default_rng(3)
    for _ in range(20):
        x = rng.normal(scale=rng.choice([0.01, 1.0, 10.0]), size=P.n) * (rng.random(P.n) < 0.5)
        assert O.dual_value_l1(P, x) <= Fs * (1 + 1e-12)
        assert O.duality_gap_l1(P, x) >= -1e-12
    # the gap of the gradient-built dual point is first order in ||x - x*|| (F - F* is second order)
    assert O.duality_gap_l1(P, xs) <= (1e-9 if kind == "ls" else 1e-7) * abs(Fs)


def test_dual_rejects_nonconvex_or_boxed():
    P = inputs.nonconvex_box(10, 12, block=2, seed=1)
    with pytest.raises(ValueError):
        O.dual_value_l1(P, np.zeros(P.n))


def test_liblinear_candidate_is_certified():
    Q = inputs.sparse_logistic(120, 60, density=0.08, seed=1, lam_frac=0.05)
    x = O.minimiser_l1_logistic_liblinear(Q)
    xs, Fs, _ = O.estimate_fstar(Q, 1.0, max_sweeps=100000, tol=0.0)
    assert O.duality_gap_l1(Q, x) <= 1e-7 * O.objective(Q, x)
    assert abs(O.objective(Q, x) - Fs) <= 1e-8 * abs(Fs)


@pytest.mark.parametrize("loss", ["logistic", "ls"])
def test_sparse_column_path_equals_dense(loss):
    """run_sequential on a CSC matrix (per-column nonzeros) == the same run on its dense copy
    (A_i^T phi'(z) and z += A_i dx of Algorithm 1 [PAPER.md:246-260]), blocks of 1 and 3."""
    for block in (1, 3):
        Q = inputs.sparse_logistic(40, 30, density=0.15, seed=9, lam_frac=0.05)
        if loss == "ls":
            Q.loss, Q.scale, Q.b = "ls", 0.5, np.random.default_rng(2).normal(size=Q.m)
            Q.tau = np.sum(inputs.csc_to_dense(Q) ** 2, axis=0) + 1e-3
        Q.block = block
        D = inputs.Problem(**{**Q.__dict__, "kind": "dense", "A": inputs.csc_to_dense(Q)})
        sched = list(O.cyclic_schedule(Q.nblocks, 5))
        xs, hs = O.run_sequential(Q, 0.9, sched, record_every=Q.nblocks)
        xd, hd = O.run_sequential(D, 0.9, sched, record_every=Q.nblocks)
        np.testing.assert_allclose(xs, xd, rtol=0, atol=1e-13)
        np.testing.assert_allclose([h[1] for h in hs], [h[1] for h in hd], rtol=1e-13)
