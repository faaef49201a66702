"""Hand-derived worked examples for the stationarity measure M_F (Eq. 5
[PAPER.md:287-290]), the Sec. 4.3 merit ||hat x(x) - x||_inf [PAPER.md:549],
the DC shift of Eq. (13) [PAPER.md:534-541], the indicator of X inside G
(problem (1) [PAPER.md:58-68]), x^0 = P_X(0) (Algorithm 1 needs x^0 in X
[PAPER.md:250]) and the relative objective error of Sec. 4.2 [PAPER.md:451].

Every expected value below is a closed form written out by hand (derivations in
tests/golden/README.md, section "1-D / 2-D stationarity pins"); nothing here is
computed by the oracle or by the CUDA path.  The CPU pins
(tests/test_oracle_pins.py) check the oracle against them and the GPU tests
(tests/test_gpu_parity.py) check the stationarity kernel against the same
numbers, so a misreading shared by both sides cannot pass.
"""
import math

import numpy as np

from paper_1701_04900_b200 import inputs

LN2 = math.log(2.0)


def problem(A, b, *, lam, tau=None, lo=-np.inf, hi=np.inf, reg="l1", theta=0.0, block=1, c=0.0):
    A = np.asfortranarray(np.array(A, float))
    m, n = A.shape
    return inputs.Problem(name="pin", kind="dense", m=m, n=n, loss="ls", scale=0.5,
                          b=np.array(b, float), lam=lam,
                          tau=np.ones(n) if tau is None else np.array(tau, float),
                          block=block, gamma=1.0, A=A, lo=lo, hi=hi, reg=reg, theta=theta, c=c)


# (name, problem, x, expected M_F(x) vector) -- f = 1/2 (x - b)^2 per coordinate (A = I)
MF_CASES = [
    # box active: f = 1/2(x-3)^2, X = [-1,1], x = 0: grad = -3, unconstrained y = 3 -> P_X = 1
    ("box_active_l0", problem([[1.0]], [3.0], lam=0.0, lo=-1.0, hi=1.0), [0.0], [-1.0]),
    # box active with l1: S_0.5(3) = 2.5 -> P_X = 1; from x = 0.5: S_0.5(0.5+2.5) = 2.5 -> 1
    ("box_active_l1", problem([[1.0]], [3.0], lam=0.5, lo=-1.0, hi=1.0), [0.5], [-0.5]),
    # lower bound active, per-coordinate box arrays: coordinate 0 in [0.2, 3], b0 = -4, x0 = 1:
    # grad = 5, S_0.5(1-5) = -3.5 -> 0.2, M = 0.8; coordinate 1 in [-2, 2], b1 = 1, x1 = 0.5:
    # grad = -0.5, S_0.5(1) = 0.5 -> M = 0
    ("box_arrays", problem(np.eye(2), [-4.0, 1.0], lam=0.5, lo=np.array([0.2, -2.0]),
                           hi=np.array([3.0, 2.0])), [1.0, 0.5], [0.8, 0.0]),
    # DC exp (theta = ln 2, eta = ln 2), lam = 1, x = 1, b = 3:
    # h^-'(1) = ln2 (1 - 1/2) = ln2/2; g = -2 - ln2/2; y = S_ln2(3 + ln2/2) = 3 - ln2/2
    ("dc_exp_pos", problem([[1.0]], [3.0], lam=1.0, reg="exp", theta=LN2), [1.0], [-2.0 + LN2 / 2]),
    # same at x = -1: f' = -4, h^-'(-1) = -ln2/2, g = -4 + ln2/2, y = S_ln2(3 - ln2/2) = 3 - 3ln2/2
    ("dc_exp_neg", problem([[1.0]], [3.0], lam=1.0, reg="exp", theta=LN2), [-1.0], [-4.0 + 1.5 * LN2]),
    # DC log (theta = 1, eta = 1/ln2), lam = 1, x = 1, b = 3:
    # h^-'(1) = 1/ln2 - 1/(2 ln2) = 1/(2 ln2); g = -2 - 1/(2ln2); y = S_{1/ln2}(3 + 1/(2ln2)) = 3 - 1/(2ln2)
    ("dc_log_pos", problem([[1.0]], [3.0], lam=1.0, reg="log", theta=1.0), [1.0], [-2.0 + 1.0 / (2 * LN2)]),
]

# (name, problem, x, expected merit ||hat x(x) - x||_inf with the tau metric)
MERIT_CASES = [
    # A = I, b = (3,-1), tau = (2,4), lam = 0.5, x = 0: g = (-3, 1);
    # hat x_0 = S_0.25(1.5) = 1.25, hat x_1 = S_0.125(-0.25) = -0.125 -> merit 1.25
    ("merit_scalar", problem(np.eye(2), [3.0, -1.0], lam=0.5, tau=[2.0, 4.0]), [0.0, 0.0], 1.25),
    # same with both coordinates in one block of 2 (per-coordinate metric: same value)
    ("merit_block2", problem(np.eye(2), [3.0, -1.0], lam=0.5, tau=[2.0, 4.0], block=2), [0.0, 0.0], 1.25),
    # same with X = [-1,1]: hat x_0 = P_X(1.25) = 1 -> merit 1
    ("merit_box", problem(np.eye(2), [3.0, -1.0], lam=0.5, tau=[2.0, 4.0], lo=-1.0, hi=1.0), [0.0, 0.0], 1.0),
    # nonconvex term c = 1/4 (f = 1/2(x-b)^2 - c x^2): x = (1, 0), b = (3, -1), tau = (2, 4), lam = 0.5:
    # g = (1-3) - 2c*1 = -2.5, hat x_0 = S_0.25(1 + 1.25) = 2.0 -> |.| = 1; g_1 = 1, hat x_1 = -0.125
    ("merit_nonconvex", problem(np.eye(2), [3.0, -1.0], lam=0.5, tau=[2.0, 4.0], c=0.25), [1.0, 0.0], 1.0),
]
