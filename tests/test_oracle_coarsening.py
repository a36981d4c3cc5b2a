"""Pins of the spatial coarsening data of oracle/mesh.py and oracle/multigrid.py (reading R6):
child cells, coarse coefficients and the Eq. (3) quantities fed to the rule.

Every expected value below is written out by hand from the numbering of include/st.h / mesh.py
(cell (i,j,k) -> i + nx*(j + ny*k)), not computed by the oracle."""
import numpy as np
import pytest

from oracle import mesh, multigrid as mg


def test_child_cells_3d_by_hand():
    # 4 x 2 x 2 mesh (nx != ny so a swapped stride fails): coarse mesh 2 x 1 x 1.
    # coarse cell 0 covers i in {0,1}, j in {0,1}, k in {0,1}: ids i + 4 j + 8 k
    m = mesh.unit_mesh((4, 2, 2))
    ch = m.child_cells()
    assert ch.shape == (2, 8)
    assert sorted(ch[0]) == [0, 1, 4, 5, 8, 9, 12, 13]
    assert sorted(ch[1]) == [2, 3, 6, 7, 10, 11, 14, 15]
    # and the (a, b, c) child order: a fastest
    assert list(ch[0]) == [0, 1, 4, 5, 8, 9, 12, 13]


def test_child_cells_3d_anisotropic_counts():
    # 2 x 4 x 6 mesh: coarse 1 x 2 x 3; coarse cell (0, 1, 2) = id 0 + 1*(1 + 2*2) = 5 has children
    # i in {0,1}, j in {2,3}, k in {4,5}: ids i + 2 j + 8 k
    m = mesh.unit_mesh((2, 4, 6))
    ch = m.child_cells()
    want = sorted(i + 2 * j + 8 * k for i in (0, 1) for j in (2, 3) for k in (4, 5))
    assert sorted(ch[5]) == want
    # every fine cell is the child of exactly one coarse cell
    assert sorted(ch.ravel()) == list(range(m.n_cells))


def test_child_cells_2d_by_hand():
    # 4 x 2 quads: coarse 2 x 1; coarse cell 1 covers i in {2,3}, j in {0,1}: ids i + 4 j
    ch = mesh.unit_mesh((4, 2)).child_cells()
    assert sorted(ch[0]) == [0, 1, 4, 5]
    assert sorted(ch[1]) == [2, 3, 6, 7]


def test_coarse_coefficients_and_rule_by_hand():
    # sigma_c = mean of the 8 children, nu_c likewise, and the rule's min_{x in T} beta/alpha is the
    # min over the children of nu/sigma (R6).  Per fine cell sigma = id + 1, nu = 2 (id + 1)^2.
    m = mesh.unit_mesh((4, 2, 2))
    ids = np.arange(m.n_cells, dtype=float)
    sigma = ids + 1.0
    nu = 2.0 * (ids + 1.0) ** 2
    tau = np.full(4, 1.0 / 16)
    H = mg.Hierarchy(m, sigma, nu, tau, 1, mg.Options(mode="full", min_slabs=2))
    assert H.space_coarsened[0]
    c = H.levels[1]
    # children of coarse cell 0: ids {0,1,4,5,8,9,12,13} -> sigma {1,2,5,6,9,10,13,14}
    np.testing.assert_allclose(c.sigma, [60.0 / 8, 76.0 / 8], rtol=0, atol=0)
    nu0 = 2.0 * np.array([1, 4, 25, 36, 81, 100, 169, 196], float)
    nu1 = 2.0 * np.array([9, 16, 49, 64, 121, 144, 225, 256], float)
    np.testing.assert_allclose(c.nu, [nu0.mean(), nu1.mean()], rtol=1e-15)
    # nu/sigma = 2 (id + 1): min over the children is 2 (cell 0) and 6 (cell 2)
    np.testing.assert_allclose(c.ratio_min, [2.0, 6.0], rtol=0, atol=0)
    # Eq. (3) on the fine level: min_T 2(id+1) * tau / h_T^2 with h_T = 1/2 (the longest edge of a
    # 1/4 x 1/2 x 1/2 cell) = 2 * (1/16) * 4 = 0.5
    assert H.lambdas[0] == pytest.approx(0.5, rel=1e-14)
    # coarse level: cells 1/2 x 1 x 1, h_T = 1, tau_c = 1/8, min ratio 2 -> 0.25
    assert mg.coarsening_lambda(c.mesh, c.ratio_min, c.tau) == pytest.approx(0.25, rel=1e-14)


def test_coarse_mesh_keeps_even_nodes():
    # R6: the coarse mesh is made of the fine nodes with even indices
    m = mesh.unit_mesh((4, 2, 2))
    X = m.coords.copy()
    X[:, 0] = X[:, 0] ** 2          # non-uniform in x: node positions distinguish the kept nodes
    fine = mesh.Mesh((4, 2, 2), X)
    c = fine.coarsen()
    np.testing.assert_allclose(np.unique(c.coords[:, 0]), [0.0, 0.25, 1.0])
    np.testing.assert_allclose(np.unique(c.coords[:, 1]), [0.0, 1.0])
