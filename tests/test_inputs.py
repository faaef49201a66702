"""Input recipe checks (CPU): determinism, column regeneration, recipe shapes."""
import numpy as np

from paper_1701_04900_b200 import inputs


def test_dense_deterministic_and_column_regeneration():
    A1 = inputs.dense_matrix(7, 33, 600, normalize=True)
    A2 = inputs.dense_matrix(7, 33, 600, normalize=True)
    assert A1.flags.f_contiguous and np.array_equal(A1, A2)
    cols = inputs.dense_columns(7, 33, 600, 250, 520, normalize=True)
    assert np.array_equal(cols, A1[:, 250:520])
    np.testing.assert_allclose(np.linalg.norm(A1, axis=0), 1.0, atol=1e-12)


def test_config_recipes_small():
    P0 = inputs.config(0)
    assert (P0.m, P0.n, P0.block, P0.gamma, P0.sweeps) == (200, 500, 1, 0.9, 500)
    assert np.count_nonzero(P0.xbar) == 25
    np.testing.assert_allclose(P0.tau, np.sum(P0.A ** 2, axis=0))
    assert abs(P0.lam - 0.1 * np.max(np.abs(P0.A.T @ P0.b))) < 1e-12
    P2 = inputs.config(2, scale=0.01)
    assert P2.lo == -1 and P2.hi == 1 and P2.block == 64 and P2.gamma == 0.5
    assert abs(P2.c - 0.1 * np.sum(P2.A ** 2) / P2.n) < 1e-9 * P2.c
    P4 = inputs.config(4, scale=0.001)
    assert P4.kind == "csc" and P4.block == 1 and set(np.unique(P4.b)) <= {-1.0, 1.0}
    cp = P4.colptr
    assert cp[0] == 0 and cp[-1] == P4.vals.size and np.all(np.diff(cp) >= 0)
    for j in range(P4.n):  # rows strictly increasing within each column
        assert np.all(np.diff(P4.rowidx[cp[j]:cp[j + 1]]) > 0)
    A = inputs.csc_to_dense(P4)
    np.testing.assert_allclose(P4.tau, 0.25 * np.sum(A ** 2, axis=0) / P4.m + 1e-6)
    c2 = inputs.dense_to_csc(A)
    assert np.array_equal(c2[0], cp) and np.array_equal(c2[1], P4.rowidx)
