"""Pins of oracle/fem.py and oracle/mesh.py against closed forms and invariants.

Each test names the property of PAPER.md §3 / §3.3 (or of the mathematics) it checks.
"""
import itertools

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import fem, mesh

M1 = np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]])   # 1D P1 mass on [0,1]


def rand_coef(m, seed=0, lo=0.5, hi=2.0):
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, m.n_cells), rng.uniform(lo, hi, m.n_cells)


def test_reference_cube_mass_closed_form():
    # x-edge block of the unit cube's Nedelec mass = (1D mass in z) (x) (1D mass in y), edges (b,c) -> b+2c;
    # blocks between different directions vanish (e_x . e_y = 0).
    m = mesh.unit_mesh((1, 1, 1))
    Me, Ke, _ = fem.element_matrices(m, np.ones(1), np.ones(1))
    Me = Me[0]
    blk = np.kron(M1, M1)
    for d in range(3):
        s = slice(4 * d, 4 * d + 4)
        np.testing.assert_allclose(Me[s, s], blk, atol=1e-15)
        for d2 in range(3):
            if d2 != d:
                assert np.abs(Me[s, 4 * d2:4 * d2 + 4]).max() < 1e-15


def test_reference_cube_curlcurl_closed_form():
    # hand integration: curl of x-edge (0,0) = (0, -(1-y), (1-z)), of x-edge (1,1) = (0, y, -z):
    #   K[0,0] = int (1-y)^2 + (1-z)^2 = 2/3 ; K[0,3] = int -(1-y)y - (1-z)z = -1/3
    m = mesh.unit_mesh((1, 1, 1))
    _, Ke, _ = fem.element_matrices(m, np.ones(1), np.ones(1))
    K = Ke[0]
    assert K[0, 0] == pytest.approx(2 / 3, abs=1e-14)
    assert K[0, 3] == pytest.approx(-1 / 3, abs=1e-14)
    # kernel of curl on one cube = gradients of the 8 vertex functions minus constants: rank 12-7 = 5
    ev = np.linalg.eigvalsh(K)
    assert np.sum(ev > 1e-12) == 5


def test_reference_square_closed_form():
    # 2D: x-edge b: l_b(y) e_x, scalar curl -l_b'(y) = +-1 -> K = outer(c,c) with c = (1,-1,-1,1)
    m = mesh.unit_mesh((1, 1))
    Me, Ke, _ = fem.element_matrices(m, np.ones(1), np.ones(1))
    c = np.array([1.0, -1.0, -1.0, 1.0])
    np.testing.assert_allclose(Ke[0], np.outer(c, c), atol=1e-15)
    np.testing.assert_allclose(Me[0][:2, :2], M1, atol=1e-15)
    np.testing.assert_allclose(Me[0][2:, 2:], M1, atol=1e-15)


@pytest.mark.parametrize("dim", [2, 3])
def test_scaling_with_h(dim):
    # Piola scaling on a cube of side h: M ~ h^{dim-2} M_ref, K ~ h^{dim-4} K_ref
    h = 0.37
    ref = mesh.unit_mesh((1,) * dim)
    sc = mesh.Mesh((1,) * dim, ref.coords * h)
    Mr, Kr, Nr = fem.element_matrices(ref, np.ones(1), np.ones(1))
    Ms, Ks, Ns = fem.element_matrices(sc, np.ones(1), np.ones(1))
    np.testing.assert_allclose(Ms, h ** (dim - 2) * Mr, rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(Ks, h ** (dim - 4) * Kr, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(Ns, h ** (dim - 2) * Nr, rtol=1e-13, atol=1e-15)


def meshes():
    rng = np.random.default_rng(7)
    out = [mesh.unit_mesh((4, 4, 4)), mesh.unit_mesh((4, 2, 6)), mesh.unit_mesh((6, 4))]
    out.append(mesh.jittered_mesh((4, 4, 4), rng.uniform(-0.2, 0.2, (125, 3))))
    out.append(mesh.jittered_mesh((6, 6), rng.uniform(-0.2, 0.2, (49, 2))))
    return out


@pytest.mark.parametrize("mi", range(5))
def test_curl_of_gradient_vanishes(mi):
    # K_nu G = 0: the nodal part lies in the kernel of curl
    m = meshes()[mi]
    s, nu = rand_coef(m, mi)
    M, K, Kn = fem.assemble(m, s, nu)
    G = fem.gradient(m)
    assert abs(K @ G).max() <= 1e-13 * abs(K).max()
    # sigma-weighted compatibility G^T M_sigma G = K_n (K_n = stiffness of div sigma grad, l.181)
    assert abs(G.T @ M @ G - Kn).max() <= 1e-12 * abs(Kn).max()
    # symmetry as assembled, Neumann K_n annihilates constants
    assert abs(M - M.T).max() <= 1e-15 * abs(M).max()
    assert abs(K - K.T).max() <= 1e-15 * abs(K).max()
    assert abs(Kn @ np.ones(m.n_nodes)).max() <= 1e-13 * abs(Kn).max()
    # M is SPD, K is PSD
    assert spla.eigsh(M, k=1, which="SA", return_eigenvectors=False)[0] > 0


def test_edge_counts():
    assert mesh.unit_mesh((4, 4, 4)).n_edges == 300          # BASELINE config 1 "300 edge dofs"
    assert mesh.unit_mesh((64, 64, 64)).n_edges == 811200    # config 4 "~811k edges"
    assert mesh.unit_mesh((64, 64)).n_edges == 8320


def test_gradient_of_coordinate_is_edge_extent():
    m = meshes()[3]
    G = fem.gradient(m)
    ext = m.coords[m.edge_nodes[:, 1]] - m.coords[m.edge_nodes[:, 0]]
    for d in range(3):
        np.testing.assert_allclose(G @ m.coords[:, d], ext[:, d], atol=1e-15)


@pytest.mark.parametrize("n", [(4, 4, 4), (4, 2, 6), (6, 4)])
def test_commuting_prolongation(n):
    # P_edge G_c = G_f P_node (the transfer maps coarse gradients to fine gradients)
    f = mesh.unit_mesh(n)
    c = f.coarsen()
    Pe = fem.edge_prolongation(f, c)
    Pn = fem.node_prolongation(f, c)
    assert abs(Pe @ fem.gradient(c) - fem.gradient(f) @ Pn).max() <= 1e-15


def _interp(m, field):
    """Nedelec interpolant: line integral of field along every edge (3-point Gauss, exact for quadratics)."""
    g, w = np.polynomial.legendre.leggauss(3)
    g = 0.5 * (g + 1); w = 0.5 * w
    a = m.coords[m.edge_nodes[:, 0]]; b = m.coords[m.edge_nodes[:, 1]]
    out = np.zeros(m.n_edges)
    for s, ws in zip(g, w):
        out += ws * np.sum(field(a + s * (b - a)) * (b - a), axis=1)
    return out


@pytest.mark.parametrize("dim", [2, 3])
def test_prolongation_reproduces_coarse_space(dim):
    # a field of the lowest-order Nedelec space (u_x bilinear in the transverse coordinates)
    # interpolated on the coarse mesh and prolongated equals its fine interpolant
    rng = np.random.default_rng(3)
    cf = rng.normal(size=12)
    if dim == 3:
        def field(X):
            x, y, z = X[:, 0], X[:, 1], X[:, 2]
            return np.stack([cf[0] + cf[1] * y + cf[2] * z + cf[3] * y * z,
                             cf[4] + cf[5] * x + cf[6] * z + cf[7] * x * z,
                             cf[8] + cf[9] * x + cf[10] * y + cf[11] * x * y], axis=1)
        f = mesh.unit_mesh((4, 4, 4))
    else:
        def field(X):
            x, y = X[:, 0], X[:, 1]
            return np.stack([cf[0] + cf[1] * y, cf[2] + cf[3] * x], axis=1)
        f = mesh.unit_mesh((4, 6))
    c = f.coarsen()
    Pe = fem.edge_prolongation(f, c)
    np.testing.assert_allclose(Pe @ _interp(c, field), _interp(f, field), atol=1e-14)


def test_longest_edge_and_paper_lambda():
    # sheared mesh x' = x + y: y-edges have length sqrt(2) h -> h_T = sqrt(2)/8 at n = 8, and with the
    # paper's weak-scaling step tau = 0.016 (l.353) the degree of anisotropy is 0.512 (l.354)
    from oracle.multigrid import coarsening_lambda
    m = mesh.unit_mesh((8, 8))
    X = m.coords.copy(); X[:, 0] += X[:, 1]
    sh = mesh.Mesh((8, 8), X)
    np.testing.assert_allclose(sh.longest_edge(), np.sqrt(2) / 8, rtol=1e-15)
    lam = coarsening_lambda(sh, np.ones(sh.n_cells), np.full(4, 0.016))
    assert lam == pytest.approx(0.512, rel=1e-12)
    assert np.allclose(mesh.unit_mesh((4, 4, 4)).longest_edge(), 0.25)


def _l2_error(m, U, exact):
    pts, wts = fem.quad_points(3)
    err = 0.0
    for p, w in zip(pts, wts):
        J = fem._jacobians(m, p)
        det = np.linalg.det(J)
        N, _ = fem.ref_edge_basis(3, p)
        V, _ = fem.ref_node_basis(3, p)
        X = np.einsum("n,cnd->cd", V, m.coords[m.cell_nodes])
        JinvT = np.linalg.inv(J).transpose(0, 2, 1)
        uh = np.einsum("cij,ce,ej->ci", JinvT, U[m.cell_edges], N)
        err += np.sum(w * det * np.sum((uh - exact(X)) ** 2, axis=1))
    return np.sqrt(err)


def test_manufactured_solution_convergence():
    # (M + K) u = b for u = (0, 0, cos(pi x) cos(pi y) sin(pi z)), which satisfies the natural
    # boundary condition n x curl u = 0 (PAPER.md l.120 Neumann); f = u + curl curl u.
    pi = np.pi

    def u(X):
        x, y, z = X.T
        return np.stack([0 * x, 0 * x, np.cos(pi * x) * np.cos(pi * y) * np.sin(pi * z)], axis=1)

    def f(X):
        x, y, z = X.T
        return np.stack([-pi ** 2 * np.sin(pi * x) * np.cos(pi * y) * np.cos(pi * z),
                         -pi ** 2 * np.cos(pi * x) * np.sin(pi * y) * np.cos(pi * z),
                         (1 + 2 * pi ** 2) * np.cos(pi * x) * np.cos(pi * y) * np.sin(pi * z)], axis=1)

    errs = []
    for n in (4, 8, 16):
        m = mesh.unit_mesh((n, n, n))
        M, K, _ = fem.assemble(m, np.ones(m.n_cells), np.ones(m.n_cells))
        b = np.zeros(m.n_edges)
        pts, wts = fem.quad_points(3)
        for p, w in zip(pts, wts):
            J = fem._jacobians(m, p)
            det = np.linalg.det(J)
            N, _ = fem.ref_edge_basis(3, p)
            V, _ = fem.ref_node_basis(3, p)
            X = np.einsum("n,cnd->cd", V, m.coords[m.cell_nodes])
            JinvT = np.linalg.inv(J).transpose(0, 2, 1)
            phi = np.einsum("cij,ej->cei", JinvT, N)
            np.add.at(b, m.cell_edges, w * det[:, None] * np.einsum("cei,ci->ce", phi, f(X)))
        U = spla.spsolve((M + K).tocsc(), b)
        errs.append(_l2_error(m, U, u))
    rates = [np.log2(errs[i] / errs[i + 1]) for i in range(2)]
    # lowest-order Nedelec: O(h) in L2
    assert all(0.9 < r < 1.3 for r in rates), (errs, rates)
