"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct fp64 CPU reference for the AsyFLEXA hot path
of Cannelli, Facchinei, Kungurtsev, Scutari, "Asynchronous Parallel Algorithms
for Nonconvex Big-Data Optimization, Part II" (arXiv:1701.04900), PAPER.md.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  It
shares no code with the CUDA path (``paper_1701_04900_b200/csrc``); the only
common dependency is the seeded input recipe ``paper_1701_04900_b200.inputs``,
which holds none of the method's arithmetic.

Every function cites the PAPER.md passage it writes out.  Conventions
(readings R1..R12 in DESIGN.md):
  * problem (1) [PAPER.md:58-68]: F = f + G, G = lam*||x||_1 (or the DC
    regularizers of Eq. 12), X_i = [lo, hi]^{n_i}, no nonconvex c_{j_i}.
  * f = s*||Ax-b||^2 - c*||x||^2 (LASSO: s = 1/2 [PAPER.md:433]; Eq. 11: s = 1
    [PAPER.md:523]) or the l1-logistic loss (1/m) sum log(1+exp(-y_j a_j^T x)).
  * surrogate: proximal-linear, tilde f_i(x_i; y) = grad_i f(y)^T (x_i - y_i)
    + 1/2 sum_{j in block i} tau_j (x_j - y_j)^2 -- satisfies Assumption B
    [PAPER.md:166-179]; for scalar blocks of a quadratic with tau_j = q_j it is
    the paper's Sec. 4.1 surrogate f(x_i; x_{-i}) (+ tau^k/2 (.)^2, tau^k = 0)
    [PAPER.md:437].

Parity status: every function here is pinned by ``tests/test_oracle_pins.py``
(closed forms, brute force, finite differences, sklearn, KKT invariants, and
the hand-derived M_F / merit / G / x0 / relative-error values of
``tests/golden_cases.py``, derived in ``tests/golden/README.md``);
none is "parity unpinned".
"""
from __future__ import annotations

import math
from typing import Iterable, Optional

import numpy as np
import scipy.sparse as sp
from scipy.special import expit, xlogy

# ----------------------------------------------------------------------------
# data access (A as a linear operator; dense ndarray or scipy CSC)
# ----------------------------------------------------------------------------


def design(P):
    """A as a dense ndarray or a scipy CSC matrix (library primitive)."""
    if P.kind == "dense":
        return P.A
    return sp.csc_matrix((P.vals, P.rowidx, P.colptr), shape=(P.m, P.n))


def columns(P, j0: int, j1: int):
    """A_i = columns j0..j1-1 of A (dense ndarray)."""
    if P.kind == "dense":
        return P.A[:, j0:j1]
    out = np.zeros((P.m, j1 - j0))
    for j in range(j0, j1):
        s, e = P.colptr[j], P.colptr[j + 1]
        out[P.rowidx[s:e], j - j0] = P.vals[s:e]
    return out


def default_x0(P) -> np.ndarray:
    """x^0 in X (Algorithm 1 initialisation [PAPER.md:250]): the projection of 0 onto the box."""
    lo, hi = lo_hi(P)
    return np.minimum(np.maximum(np.zeros(P.n), lo), hi)


def lo_hi(P):
    lo = np.broadcast_to(np.asarray(P.lo, float), (P.n,))
    hi = np.broadcast_to(np.asarray(P.hi, float), (P.n,))
    return lo, hi


# ----------------------------------------------------------------------------
# f, G, F  -- problem (1) [PAPER.md:58-68], LASSO [PAPER.md:433], Eq. (11) [PAPER.md:521-525]
# ----------------------------------------------------------------------------


def smooth_value(P, x: np.ndarray) -> float:
    """f(x).  LS: s*||Ax-b||^2 - c||x||^2.  Logistic: mean log(1+exp(-y Ax)) - c||x||^2."""
    z = design(P) @ x
    if P.loss == "ls":
        r = z - P.b
        val = P.scale * float(r @ r)
    else:
        val = float(np.mean(np.logaddexp(0.0, -P.b * z)))
    return val - P.c * float(x @ x)


def loss_prime(P, z, b):
    """phi'(z) with grad f = A^T phi'(Ax) - 2c x.  LS: 2s (z - b).  Logistic: -(y/m) sigmoid(-y z)."""
    if P.loss == "ls":
        return 2.0 * P.scale * (z - b)
    return -(b / P.m) * expit(-b * z)


def smooth_grad(P, x: np.ndarray) -> np.ndarray:
    """grad f(x) by definition.  LS: 2s A^T(Ax-b) - 2c x.
    Logistic: A^T w - 2c x, w_j = -(y_j/m) sigmoid(-y_j (Ax)_j)."""
    A = design(P)
    z = A @ x
    if P.loss == "ls":
        w = 2.0 * P.scale * (z - P.b)
    else:
        w = -(P.b / P.m) * expit(-P.b * z)
    return A.T @ w - 2.0 * P.c * x


# --- DC regularizers of Sec. 4.3, Eq. (12) [PAPER.md:526-533] -------------------


def h(P, t):
    """scalar penalty h: |t| (l1), 1-exp(-theta|t|) (exp), log(1+theta|t|)/log(1+theta) (log)."""
    t = np.abs(t)
    if P.reg == "l1":
        return t
    if P.reg == "exp":
        return 1.0 - np.exp(-P.theta * t)
    return np.log1p(P.theta * t) / math.log1p(P.theta)


def eta(P) -> float:
    """eta(theta): exp -> theta, log -> theta/log(1+theta) [PAPER.md:532]; l1 -> 1."""
    if P.reg == "l1":
        return 1.0
    if P.reg == "exp":
        return P.theta
    return P.theta / math.log1p(P.theta)


def h_plus(P, t):
    return eta(P) * np.abs(t)


def h_minus(P, t):
    """h^-(t) = eta|t| - h(t) (Eq. 12)."""
    return eta(P) * np.abs(t) - h(P, t)


def grad_h_minus(P, t):
    """d/dt h^-(t): exp: eta*sign(t)*(1-exp(-theta|t|)); log: sign(t)*(eta - theta/((1+theta|t|)log(1+theta)))."""
    t = np.asarray(t, float)
    if P.reg == "l1":
        return np.zeros_like(t)
    if P.reg == "exp":
        return eta(P) * np.sign(t) * (1.0 - np.exp(-P.theta * np.abs(t)))
    return np.sign(t) * (eta(P) - P.theta / ((1.0 + P.theta * np.abs(t)) * math.log1p(P.theta)))


def G(P, x: np.ndarray) -> float:
    """G(x) = lam*sum_i h(x_i) on the box, +inf outside X."""
    lo, hi = lo_hi(P)
    if np.any(x < lo) or np.any(x > hi):
        return math.inf
    return P.lam * float(np.sum(h(P, x)))


def objective(P, x: np.ndarray) -> float:
    """F(x) = f(x) + G(x), Eq. (1) [PAPER.md:60]."""
    return smooth_value(P, x) + G(P, x)


# ----------------------------------------------------------------------------
# best response, Eq. (2) [PAPER.md:148-152]
# ----------------------------------------------------------------------------


def soft_threshold(v, t):
    """S_t(v) = sign(v) max(|v|-t, 0): the closed form of Sec. 4.1 [PAPER.md:384]."""
    v = np.asarray(v, float)
    return np.sign(v) * np.maximum(np.abs(v) - t, 0.0)


def scalar_subproblem_argmin(g, y, tau, lam, lo, hi):
    """argmin_{t in [lo,hi]} g*(t-y) + tau/2*(t-y)^2 + lam*|t|   (elementwise).

    Step 1: the unconstrained minimiser of this strongly convex 1-D function is
    the soft-threshold S_{lam/tau}(y - g/tau).  Step 2: a 1-D convex function
    restricted to an interval is minimised at the projection of its
    unconstrained minimiser onto the interval."""
    u = soft_threshold(y - g / tau, lam / tau)
    return np.minimum(np.maximum(u, lo), hi)


def best_response(P, i: int, xt: np.ndarray, grad: Optional[np.ndarray] = None) -> np.ndarray:
    """hat x_i(xt), Eq. (2), with the proximal-linear surrogate (module docstring)
    and, for the DC regularizers, the linearised h^- of Eq. (13) [PAPER.md:534-541]:
    the smooth gradient is shifted by -lam*grad h^-(xt_i) and the convex part is
    lam*eta*|x_i|.  ``grad`` (optional) is grad f(xt) restricted to block i."""
    j0, j1 = P.block_range(i)
    if grad is None:
        grad = smooth_grad(P, xt)[j0:j1]
    y = xt[j0:j1]
    lo, hi = lo_hi(P)
    gshift = grad - P.lam * grad_h_minus(P, y)
    return scalar_subproblem_argmin(gshift, y, P.tau[j0:j1], P.lam * eta(P),
                                    lo[j0:j1], hi[j0:j1])


# ----------------------------------------------------------------------------
# stationarity measure M_F, Eq. (5) [PAPER.md:287-290]
# ----------------------------------------------------------------------------


def stationarity(P, x: np.ndarray) -> np.ndarray:
    """M_F(x) = x - argmin_{y in X} {grad f(x)^T (y-x) + g(y) + 1/2||y-x||^2}.
    For the DC regularizers, f carries -lam*h^- and g = lam*eta|.| (the f/G
    split of Sec. 4.3 [PAPER.md:533])."""
    lo, hi = lo_hi(P)
    g = smooth_grad(P, x) - P.lam * grad_h_minus(P, x)
    y = scalar_subproblem_argmin(g, x, 1.0, P.lam * eta(P), lo, hi)
    return x - y


def merit_inf(P, x: np.ndarray) -> float:
    """||hat x(x) - x||_inf, the Sec. 4.3 distance to stationarity [PAPER.md:549]."""
    g = smooth_grad(P, x)
    out = 0.0
    for i in range(P.nblocks):
        j0, j1 = P.block_range(i)
        out = max(out, float(np.max(np.abs(best_response(P, i, x, g[j0:j1]) - x[j0:j1]))))
    return out


# ----------------------------------------------------------------------------
# schedules (S.1) [PAPER.md:253]
# ----------------------------------------------------------------------------


def cyclic_schedule(nblocks: int, sweeps: int) -> Iterable[int]:
    for _ in range(sweeps):
        yield from range(nblocks)


M32 = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    """Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), written out in Python.
    Pinned by the Random123 known-answer vectors in the tests."""
    c0, c1, c2, c3 = (int(v) & M32 for v in ctr)
    k0, k1 = (int(v) & M32 for v in key)
    for i in range(10):
        if i > 0:
            k0 = (k0 + 0x9E3779B9) & M32
            k1 = (k1 + 0xBB67AE85) & M32
        p0 = 0xD2511F53 * c0
        p1 = 0xCD9E8D57 * c2
        hi0, lo0 = p0 >> 32, p0 & M32
        hi1, lo1 = p1 >> 32, p1 & M32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return [c0, c1, c2, c3]


def _fmix32(h):
    h ^= h >> 16
    h = (h * 0x85EBCA6B) & M32
    h ^= h >> 13
    h = (h * 0xC2B2AE35) & M32
    h ^= h >> 16
    return h


def random_epoch_order(seed: int, epoch: int, nblocks: int) -> list:
    """The random schedule of one epoch (reading R6): the permutation
    i -> pi_e(i) of the N blocks given by a 4-round Feistel network on [0, 2^d)
    (d even, 2^d >= N) keyed by one Philox4x32-10 draw at counter
    (epoch_lo, epoch_hi, 0x5EED, 0xA5F1) with key (seed_lo, seed_hi), and
    cycle-walking back into [0, N)."""
    keys = philox4x32_10([epoch & M32, (epoch >> 32) & M32, 0x5EED, 0xA5F1],
                         [seed & M32, (seed >> 32) & M32])
    d = 2
    while (1 << d) < nblocks:
        d += 1
    if d & 1:
        d += 1
    half = d // 2
    mask = (1 << half) - 1

    def enc(v):
        L, R = v >> half, v & mask
        for r in range(4):
            F = _fmix32((R & M32) ^ keys[r] ^ (R >> 32)) & mask
            L, R = R, L ^ F
        return (L << half) | R

    out = []
    for i in range(nblocks):
        v = enc(i)
        while v >= nblocks:
            v = enc(v)
        out.append(v)
    return out


def random_schedule(seed: int, nblocks: int, sweeps: int, epoch0: int = 0) -> Iterable[int]:
    for e in range(epoch0, epoch0 + sweeps):
        yield from random_epoch_order(seed, e, nblocks)


# ----------------------------------------------------------------------------
# Algorithm 1 with d^k = 0 (sequential), [PAPER.md:246-260]
# ----------------------------------------------------------------------------


def run_sequential(P, gamma: float, schedule: Iterable[int], x0: Optional[np.ndarray] = None,
                   refresh_every: int = 0, record_every: int = 0):
    """Algorithm 1 executed by one core (all delays d^k = 0): for each drawn
    block i: (S.2) hat x_i(x^k), (S.3) read x_i^k, (S.4)
    x_i^{k+1} = x_i^k + gamma (hat x_i - x_i^k).

    grad_i f(x^k) = A_i^T phi'(A x^k) is evaluated from z = A x^k.  z is carried
    forward by the identity A x^{k+1} = A x^k + A_i (x_i^{k+1} - x_i^k)
    (x changes only in block i); ``refresh_every=1`` recomputes z = A x from
    scratch at every iteration (the plain definition; the pins compare both).
    Returns (x, history) with history = [(k, F(x^k))] every ``record_every`` updates."""
    A = design(P)
    x = default_x0(P) if x0 is None else np.array(x0, float)
    z = A @ x
    hist = []
    for k, i in enumerate(schedule):
        if refresh_every and k % refresh_every == 0:
            z = A @ x
        j0, j1 = P.block_range(i)
        if P.kind == "csc":
            # sparse A_i: the same A_i^T phi'(z) and z += A_i dx over the stored nonzeros only
            # (phi' evaluated at the rows a column touches; zero entries contribute nothing)
            grad = np.empty(j1 - j0)
            for j in range(j0, j1):
                s, e = P.colptr[j], P.colptr[j + 1]
                grad[j - j0] = P.vals[s:e] @ loss_prime(P, z[P.rowidx[s:e]], P.b[P.rowidx[s:e]])
            grad -= 2.0 * P.c * x[j0:j1]
            xhat = best_response(P, i, x, grad)
            xnew = x[j0:j1] + gamma * (xhat - x[j0:j1])
            for j in range(j0, j1):
                s, e = P.colptr[j], P.colptr[j + 1]
                z[P.rowidx[s:e]] += P.vals[s:e] * (xnew[j - j0] - x[j])
            x[j0:j1] = xnew
            if record_every and (k + 1) % record_every == 0:
                hist.append((k + 1, objective(P, x)))
            continue
        Ai = columns(P, j0, j1)
        w = loss_prime(P, z, P.b)
        grad = Ai.T @ w - 2.0 * P.c * x[j0:j1]
        xhat = best_response(P, i, x, grad)
        xnew = x[j0:j1] + gamma * (xhat - x[j0:j1])
        z = z + Ai @ (xnew - x[j0:j1])
        x[j0:j1] = xnew
        if record_every and (k + 1) % record_every == 0:
            hist.append((k + 1, objective(P, x)))
    return x, hist


# ----------------------------------------------------------------------------
# synchronous version (Corollary, x^{k-d} = x^k) [PAPER.md:346-357], Jacobi form
# ----------------------------------------------------------------------------


def jacobi_step(P, x: np.ndarray, gamma: float) -> np.ndarray:
    """All blocks updated simultaneously from the same x (the synchronous
    scheme used to estimate F* [PAPER.md:434]): x+ = x + gamma (hat x(x) - x)."""
    g = smooth_grad(P, x)
    xnew = x.copy()
    for i in range(P.nblocks):
        j0, j1 = P.block_range(i)
        xhat = best_response(P, i, x, g[j0:j1])
        xnew[j0:j1] = x[j0:j1] + gamma * (xhat - x[j0:j1])
    return xnew


def run_jacobi(P, gamma: float, sweeps: int, x0: Optional[np.ndarray] = None,
               keep_iterates: bool = False):
    """Returns (x, F history [F(x^1)..F(x^T)], iterates or None)."""
    x = default_x0(P) if x0 is None else np.array(x0, float)
    Fs, xs = [], []
    for _ in range(sweeps):
        x = jacobi_step(P, x, gamma)
        Fs.append(objective(P, x))
        if keep_iterates:
            xs.append(x.copy())
    return x, np.array(Fs), (xs if keep_iterates else None)


def estimate_fstar(P, gamma: float, max_sweeps: int = 20000, tol: float = 1e-15,
                   x0: Optional[np.ndarray] = None):
    """F* estimate: run the sequential (cyclic) scheme "until variations in the
    objective value were undetectable" [PAPER.md:434]."""
    x = default_x0(P) if x0 is None else np.array(x0, float)
    Fprev = objective(P, x)
    for s in range(max_sweeps):
        x, _ = run_sequential(P, gamma, range(P.nblocks), x0=x)
        F = objective(P, x)
        if abs(Fprev - F) <= tol * max(1.0, abs(F)):
            return x, F, s + 1
        Fprev = F
    return x, F, max_sweeps


def relative_error(Fx: float, Fstar: float) -> float:
    """(F(x) - F*)/|F*| -- the 'relative error on the objective' of Sec. 4.2 [PAPER.md:451]."""
    return (Fx - Fstar) / abs(Fstar)


# ----------------------------------------------------------------------------
# certified F* for the convex l1 instances (Fenchel duality -- mathematics, not
# the paper).  Used only to certify the F* of configs whose Algorithm 1 run is
# too long for this CPU oracle (configs[4]: ~3e4 sweeps of 1e6 scalar blocks).
# ----------------------------------------------------------------------------


def dual_value_l1(P, x: np.ndarray) -> float:
    """Fenchel dual value D(u) <= F* at the dual point built from x, for
    F = f(Ax) + lam||x||_1 with no box, c = 0 and G = l1 (convex configs 0, 1, 3, 4).

    min_x f(Ax) + lam||x||_1 has the dual max_u -f^*(u) s.t. ||A^T u||_inf <= lam.
      LS, f(z) = s||z - b||^2:  f^*(u) = b^T u + ||u||^2/(4s);
      logistic, f(z) = (1/m) sum log(1 + exp(-y_j z_j)), u = -(y o theta)/m,
        theta in [0,1]^m:      f^*(u) = (1/m) sum theta log theta + (1-theta) log(1-theta).
    The dual point is u0 = grad of f at Ax (LS: 2s(Ax - b); logistic:
    theta = sigmoid(-y o Ax)) scaled by min(1, lam/||A^T u0||_inf) into the feasible set,
    so F(x) - D(u) is a certified bound on F(x) - F* (weak duality)."""
    if P.reg != "l1" or P.c != 0.0 or np.any(np.isfinite(lo_hi(P)[0])) or np.any(np.isfinite(lo_hi(P)[1])):
        raise ValueError("dual_value_l1: convex l1 problems without a box only")
    A = design(P)
    z = A @ x
    if P.loss == "ls":
        u0 = 2.0 * P.scale * (z - P.b)
        g = float(np.max(np.abs(A.T @ u0)))
        u = u0 * (min(1.0, P.lam / g) if g > 0 else 1.0)
        return float(-(P.b @ u) - (u @ u) / (4.0 * P.scale))
    theta0 = expit(-P.b * z)
    g = float(np.max(np.abs(A.T @ (P.b * theta0)))) / P.m
    theta = theta0 * (min(1.0, P.lam / g) if g > 0 else 1.0)
    ent = xlogy(theta, theta) + xlogy(1.0 - theta, 1.0 - theta)
    return float(-np.sum(ent) / P.m)


def duality_gap_l1(P, x: np.ndarray) -> float:
    """F(x) - D(u(x)) >= F(x) - F* >= 0 (see dual_value_l1)."""
    return objective(P, x) - dual_value_l1(P, x)


def minimiser_l1_logistic_liblinear(P, tol: float = 1e-10) -> np.ndarray:
    """Candidate minimiser of the convex l1-logistic F from an independent library
    solver (scikit-learn / liblinear newGLMNET: min ||x||_1 + C sum log(1+exp(-y a_j x)),
    C = 1/(m lam), which is F/lam).  Library primitive; its output is certified by
    duality_gap_l1, never trusted on its own."""
    import warnings
    from sklearn.linear_model import LogisticRegression
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        lr = LogisticRegression(l1_ratio=1.0, C=1.0 / (P.m * P.lam), solver="liblinear",
                                fit_intercept=False, tol=tol, max_iter=1000000)
        lr.fit(sp.csr_matrix(design(P)), P.b)
    return np.asarray(lr.coef_[0], float)
