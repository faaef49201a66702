"""Seeded synthetic problem instances for the five BASELINE.json configurations.

This module is the ONE piece shared by the oracle (``oracle/``) and the CUDA
path (tests, bench).  It holds only the *input recipe* -- how A, b, x*, lambda,
tau, the box and the block partition are drawn -- and none of the method's
arithmetic (no gradients, no best responses, no objective).

Recipes (PAPER.md line numbers in brackets):

* Gaussian LASSO data follow the Liu-Wright generator of Sec. 4.2
  [PAPER.md:442]: A iid N(0,1), sparse x-bar with N(0,1) nonzeros at uniformly
  random positions, b = A x-bar + e, e ~ N(0, sigma^2).
* The nonconvex instance follows Sec. 4.3 [PAPER.md:547]: A iid N(0,1),
  x-bar with 95% of its components set to zero, e ~ N(0, 0.1^2).
* lambda, tau_i, block sizes, gamma and the box are BASELINE.json's values;
  where it is silent the choice is a DESIGN.md reading (R-numbers below).

Every dense matrix is generated column-chunk by column-chunk from
``numpy.random.default_rng([seed, TAG_A, chunk])`` so any column can be
regenerated alone (``dense_columns``) -- that is how full-size parity tests
sample single outputs without a second copy of A.  A is returned in
column-major (Fortran) order, which is also the device layout.
"""
from __future__ import annotations

import dataclasses
import os
from concurrent.futures import ThreadPoolExecutor
from typing import Optional

import numpy as np

TAG_A, TAG_X, TAG_E, TAG_PAT = 1, 2, 3, 4
COL_CHUNK = 256  # columns per independently seeded chunk


@dataclasses.dataclass
class Problem:
    """F(x) = f(x) + G(x) [PAPER.md:58-68] with
    f(x) = s*||Ax-b||^2 - c*||x||^2          (loss == "ls")
    f(x) = (1/m) sum_j log(1+exp(-y_j a_j^T x)) - c*||x||^2   (loss == "logistic")
    G(x) = lam*||x||_1 restricted to the box X_i = [lo, hi]^{n_i}.
    Blocks are the contiguous column ranges [i*block, min(n,(i+1)*block)).
    """
    name: str
    kind: str                      # "dense" | "csc"
    m: int
    n: int
    loss: str                      # "ls" | "logistic"
    scale: float                   # s in s*||Ax-b||^2 (ls only)
    b: np.ndarray                  # LS target b, or logistic labels y in {-1,+1}
    lam: float
    tau: np.ndarray                # proximal weights tau_j (n,)
    block: int
    gamma: float
    c: float = 0.0                 # nonconvex coefficient: f -= c*||x||^2
    lo: float = -np.inf
    hi: float = np.inf
    A: Optional[np.ndarray] = None            # dense (m, n), Fortran order
    colptr: Optional[np.ndarray] = None       # CSC int64 (n+1,)
    rowidx: Optional[np.ndarray] = None       # CSC int32 (nnz,)
    vals: Optional[np.ndarray] = None         # CSC float64 (nnz,)
    xbar: Optional[np.ndarray] = None         # ground truth signal
    sweeps: int = 100
    reg: str = "l1"                # "l1" | "exp" | "log"  (Sec. 4.3 DC regularizers)
    theta: float = 0.0
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def nblocks(self) -> int:
        return (self.n + self.block - 1) // self.block

    def block_range(self, i: int) -> tuple[int, int]:
        return i * self.block, min(self.n, (i + 1) * self.block)


# --------------------------------------------------------------------------
# raw draws
# --------------------------------------------------------------------------
def _chunk_cols(seed: int, m: int, chunk: int, n: int) -> np.ndarray:
    j0 = chunk * COL_CHUNK
    j1 = min(n, j0 + COL_CHUNK)
    rng = np.random.default_rng([seed, TAG_A, chunk])
    return rng.standard_normal((j1 - j0, m))  # rows of A^T == columns of A


def dense_columns(seed: int, m: int, n: int, j0: int, j1: int,
                  normalize: bool = False) -> np.ndarray:
    """Columns j0..j1-1 of the seeded N(0,1) matrix, shape (m, j1-j0), F-order."""
    out = np.empty((j1 - j0, m))
    c0, c1 = j0 // COL_CHUNK, (j1 - 1) // COL_CHUNK
    for c in range(c0, c1 + 1):
        blk = _chunk_cols(seed, m, c, n)
        a0 = c * COL_CHUNK
        lo, hi = max(j0, a0), min(j1, a0 + blk.shape[0])
        out[lo - j0:hi - j0] = blk[lo - a0:hi - a0]
    if normalize:
        out /= np.sqrt(np.einsum("ij,ij->i", out, out))[:, None]
    return out.T


def dense_matrix(seed: int, m: int, n: int, normalize: bool = False,
                 threads: Optional[int] = None) -> np.ndarray:
    """Full seeded matrix, (m, n) Fortran order; chunks drawn in parallel."""
    At = np.empty((n, m))
    nchunks = (n + COL_CHUNK - 1) // COL_CHUNK

    def work(c):
        blk = _chunk_cols(seed, m, c, n)
        if normalize:
            blk /= np.sqrt(np.einsum("ij,ij->i", blk, blk))[:, None]
        At[c * COL_CHUNK:c * COL_CHUNK + blk.shape[0]] = blk

    threads = threads or min(32, os.cpu_count() or 1)
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(work, range(nchunks)))
    return At.T


def sparse_signal(seed: int, n: int, nnz: int) -> np.ndarray:
    rng = np.random.default_rng([seed, TAG_X])
    x = np.zeros(n)
    idx = rng.choice(n, size=nnz, replace=False)
    x[idx] = rng.standard_normal(nnz)
    return x


def noise(seed: int, m: int, sigma: float) -> np.ndarray:
    return sigma * np.random.default_rng([seed, TAG_E]).standard_normal(m)


def col_sqnorms(A: np.ndarray) -> np.ndarray:
    At = A.T
    return np.einsum("ij,ij->i", At, At)


# --------------------------------------------------------------------------
# dense instances
# --------------------------------------------------------------------------
def dense_lasso(m: int, n: int, *, nnz_frac: float, sigma: float, lam_frac: float,
                block: int, gamma: float = 0.9, normalize: bool = False,
                seed: int = 0, sweeps: int = 100, name: str = "dense_lasso",
                nnz: Optional[int] = None) -> Problem:
    """LASSO f = 1/2||Ax-b||^2, G = lam||x||_1 [PAPER.md:433], data per [PAPER.md:442].
    lam = lam_frac * ||A^T b||_inf (BASELINE.json), tau_j = ||a_j||^2 (reading R3)."""
    A = dense_matrix(seed, m, n, normalize)
    k = nnz if nnz is not None else max(1, int(round(nnz_frac * n)))
    xbar = sparse_signal(seed, n, k)
    sup = np.flatnonzero(xbar)
    b = A[:, sup] @ xbar[sup] + noise(seed, m, sigma)
    lam = lam_frac * float(np.max(np.abs(A.T @ b)))
    tau = col_sqnorms(A)
    return Problem(name=name, kind="dense", m=m, n=n, loss="ls", scale=0.5, b=b,
                   lam=lam, tau=tau, block=block, gamma=gamma, A=A, xbar=xbar,
                   sweeps=sweeps,
                   meta=dict(seed=seed, nnz=k, sigma=sigma, lam_frac=lam_frac,
                             normalize=normalize))


def nonconvex_box(m: int, n: int, *, block: int = 64, gamma: float = 0.5,
                  lam_frac: float = 0.05, c_frac: float = 0.1, seed: int = 0,
                  sweeps: int = 100, name: str = "nonconvex_box") -> Problem:
    """f = ||Ax-b||^2 - c||x||^2 (Eq. 11 scale [PAPER.md:523] + the nonconvex
    quadratic of BASELINE configs[2]), G = lam||x||_1, X_i = [-1,1].
    b = A xbar + e with 95% zeros in xbar, sigma_e = 0.1 [PAPER.md:547].
    c = c_frac*||A||_F^2/n, lam = lam_frac*||A^T b||_inf, tau_j = 2||a_j||^2 (R4)."""
    A = dense_matrix(seed, m, n)
    k = max(1, int(round(0.05 * n)))
    xbar = sparse_signal(seed, n, k)
    sup = np.flatnonzero(xbar)
    b = A[:, sup] @ xbar[sup] + noise(seed, m, 0.1)
    sq = col_sqnorms(A)
    c = c_frac * float(sq.sum()) / n
    lam = lam_frac * float(np.max(np.abs(A.T @ b)))
    return Problem(name=name, kind="dense", m=m, n=n, loss="ls", scale=1.0, b=b,
                   lam=lam, tau=2.0 * sq, block=block, gamma=gamma, c=c,
                   lo=-1.0, hi=1.0, A=A, xbar=xbar, sweeps=sweeps,
                   meta=dict(seed=seed, nnz=k, c_frac=c_frac, lam_frac=lam_frac))


# --------------------------------------------------------------------------
# sparse instance
# --------------------------------------------------------------------------
def sparse_pattern(seed: int, m: int, n: int, density: float):
    """Uniform random CSC pattern: nnz per column ~ Binomial(m, density),
    rows uniform without replacement within a column, values N(0,1)."""
    rng = np.random.default_rng([seed, TAG_PAT])
    counts = rng.binomial(m, density, size=n).astype(np.int64)
    cols = np.repeat(np.arange(n, dtype=np.int64), counts)
    rows = rng.integers(0, m, size=cols.size, dtype=np.int64)
    key = np.sort(cols * m + rows)
    keep = np.ones(key.size, bool)
    keep[1:] = key[1:] != key[:-1]
    key = key[keep]
    cols, rows = key // m, key % m
    colptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(cols, minlength=n), out=colptr[1:])
    vals = rng.standard_normal(rows.size)
    return colptr, rows.astype(np.int32), vals


def csc_matvec(colptr, rowidx, vals, m, x):
    """A @ x for the CSC arrays (input recipe helper: labels / lambda)."""
    n = colptr.size - 1
    cols = np.repeat(np.arange(n), np.diff(colptr))
    return np.bincount(rowidx, weights=vals * x[cols], minlength=m)


def csc_rmatvec(colptr, rowidx, vals, v):
    n = colptr.size - 1
    cols = np.repeat(np.arange(n), np.diff(colptr))
    return np.bincount(cols, weights=vals * v[rowidx], minlength=n)


def sparse_logistic(m: int, n: int, *, density: float, nnz_frac: float = 0.01,
                    lam_frac: float = 1e-3, gamma: float = 0.9, seed: int = 0,
                    sweeps: int = 50, name: str = "sparse_logistic",
                    label_noise: float = 0.1) -> Problem:
    """l1-logistic regression, BASELINE configs[4]: y = sign(A x* + N(0,0.1)),
    lam = lam_frac*||A^T y||_inf/m, scalar blocks, tau_j = 0.25||a_j||^2/m + 1e-6."""
    colptr, rowidx, vals = sparse_pattern(seed, m, n, density)
    k = max(1, int(round(nnz_frac * n)))
    xbar = sparse_signal(seed, n, k)
    z = csc_matvec(colptr, rowidx, vals, m, xbar) + noise(seed, m, label_noise)
    y = np.where(z >= 0, 1.0, -1.0)
    lam = lam_frac * float(np.max(np.abs(csc_rmatvec(colptr, rowidx, vals, y)))) / m
    cols = np.repeat(np.arange(n), np.diff(colptr))
    sq = np.bincount(cols, weights=vals * vals, minlength=n)
    tau = 0.25 * sq / m + 1e-6
    return Problem(name=name, kind="csc", m=m, n=n, loss="logistic", scale=1.0, b=y,
                   lam=lam, tau=tau, block=1, gamma=gamma, colptr=colptr,
                   rowidx=rowidx, vals=vals, xbar=xbar, sweeps=sweeps,
                   meta=dict(seed=seed, density=density, nnz=int(vals.size)))


def csc_to_dense(P: Problem) -> np.ndarray:
    A = np.zeros((P.m, P.n), order="F")
    for j in range(P.n):
        s, e = P.colptr[j], P.colptr[j + 1]
        A[P.rowidx[s:e], j] = P.vals[s:e]
    return A


def dense_to_csc(A: np.ndarray):
    """CSC arrays of a dense (m, n) matrix (zeros dropped)."""
    m, n = A.shape
    At = np.asarray(A.T)
    mask = At != 0
    counts = mask.sum(1)
    colptr = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=colptr[1:])
    rows = np.nonzero(mask)[1].astype(np.int32)
    vals = At[mask]
    return colptr, rows, vals


# --------------------------------------------------------------------------
# the five BASELINE.json configurations
# --------------------------------------------------------------------------
def config(idx: int, seed: int = 0, scale: float = 1.0) -> Problem:
    """BASELINE.json configs[idx]; ``scale`` < 1 shrinks m and n (small analogs
    for parity tests keep every other parameter of the recipe)."""
    def S(v):
        return max(2, int(round(v * scale)))
    if idx == 0:
        # Tiny LASSO: 200x500, 5% nnz, sigma 0.01, lam=0.1||A^T b||_inf,
        # scalar blocks, tau_i=||A_i||^2, gamma=0.9, 500 sweeps, seed 0.
        return dense_lasso(S(200), S(500), nnz_frac=0.05, sigma=0.01, lam_frac=0.1,
                           block=1, gamma=0.9, seed=seed, sweeps=500,
                           name="tiny_lasso")
    if idx == 1:
        # Dense LASSO: 10000x20000 normalised columns, 1% nnz, sigma 0.01,
        # lam=0.05||A^T b||_inf, blocks of 32.
        return dense_lasso(S(10000), S(20000), nnz_frac=0.01, sigma=0.01,
                           lam_frac=0.05, block=32, gamma=0.9, normalize=True,
                           seed=seed, sweeps=100, name="dense_lasso")
    if idx == 2:
        return nonconvex_box(S(20000), S(40000), block=64, gamma=0.5, seed=seed,
                             name="nonconvex_box")
    if idx == 3:
        # Large dense LASSO: 40000x100000 (32 GB), 0.5% nnz, lam=0.02||A^T b||_inf,
        # blocks of 128.
        return dense_lasso(S(40000), S(100000), nnz_frac=0.005, sigma=0.01,
                           lam_frac=0.02, block=128, gamma=0.9, seed=seed,
                           sweeps=100, name="large_dense_lasso")
    if idx == 4:
        m, n = S(100000), S(1000000)
        dens = 1e-4 if scale >= 1.0 else min(0.05, 10.0 / m)
        return sparse_logistic(m, n, density=dens, seed=seed, name="sparse_logistic")
    raise ValueError(idx)
