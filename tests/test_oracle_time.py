"""Pins of oracle/time_dg.py and oracle/lfa.py (dG(q) in time, scalar test equation)."""
import numpy as np
import pytest

from oracle import lfa, time_dg


def test_dg0_is_implicit_euler():
    # q = 0 must reproduce Eq. (1): (M + tau K) u^{k+1} - M u^k = tau f
    Ct, Mt, Nt = time_dg.time_matrices(0)
    assert Ct.tolist() == [[1.0]] and Mt.tolist() == [[1.0]] and Nt.tolist() == [[1.0]]


def test_dg1_matrices_closed_form():
    # phi_0 = 1 - s, phi_1 = s on [0,1]: mass [[1/3,1/6],[1/6,1/3]], derivative+jump [[1/2,1/2],[-1/2,1/2]],
    # trace coupling only (b=0 <- a=1)
    Ct, Mt, Nt = time_dg.time_matrices(1)
    np.testing.assert_allclose(Mt, [[1 / 3, 1 / 6], [1 / 6, 1 / 3]], atol=1e-15)
    np.testing.assert_allclose(Ct, [[0.5, 0.5], [-0.5, 0.5]], atol=1e-15)
    np.testing.assert_allclose(Nt, [[0.0, 1.0], [0.0, 0.0]], atol=0)


@pytest.mark.parametrize("q,order", [(0, 1), (1, 3)])
def test_dg_nodal_superconvergence(q, order):
    # u' + lam u = f, u(t) = sin(t) + exp(-t)... endpoint error of dG(q) is O(tau^{2q+1})
    lam = 2.0

    def u(t):
        return np.sin(3 * t)

    def f(t):
        return 3 * np.cos(3 * t) + lam * np.sin(3 * t)

    Ct, Mt, Nt = time_dg.time_matrices(q)
    g, w = np.polynomial.legendre.leggauss(8)
    g = 0.5 * (g + 1); w = 0.5 * w
    errs = []
    for m in (8, 16, 32):
        tau = 1.0 / m
        prev = np.zeros(q + 1)
        prev_end = u(0.0)                     # initial value enters through the jump term
        for k in range(m):
            t0 = k * tau
            rhs = np.array([tau * np.sum(w * f(t0 + tau * g) * np.array([time_dg.lagrange(q, s)[b] for s in g]))
                            for b in range(q + 1)])
            rhs += time_dg.lagrange(q, 0.0) * prev_end
            x = np.linalg.solve(Ct + tau * lam * Mt, rhs)
            prev_end = time_dg.lagrange(q, 1.0) @ x
        errs.append(abs(prev_end - u(1.0)))
    rates = [np.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert all(abs(r - order) < 0.3 for r in rates), (errs, rates)


@pytest.mark.parametrize("q", [0, 1])
@pytest.mark.parametrize("theta", [0.5, 0.3])
def test_prolongation_interpolates_coarse_polynomials(q, theta):
    P = time_dg.prolongation(q, theta)
    np.testing.assert_allclose(P.sum(axis=1), 1.0, atol=1e-15)        # constants are reproduced
    if q == 1:
        # coarse linear function with nodal values (a, b) evaluated at the fine nodes 0, theta | theta, 1
        a, b = 2.0, -1.0
        mid = a + theta * (b - a)
        np.testing.assert_allclose(P @ [a, b], [a, mid, mid, b], atol=1e-15)


@pytest.mark.parametrize("q", [0, 1])
def test_time_galerkin_equals_rediscretisation(q):
    # R_t L_fine P_t = L_coarse for the time operator (uniform and non-uniform splits): the coarse
    # space is a subspace of the fine one, so rediscretising with tau_c = tau_a + tau_b is Galerkin.
    lam = 1.7
    Ct, Mt, Nt = time_dg.time_matrices(q)
    Q = q + 1
    for ta, tb in [(0.1, 0.1), (0.05, 0.2)]:
        Lf = np.zeros((2 * Q, 2 * Q))
        Lf[:Q, :Q] = Ct + ta * lam * Mt
        Lf[Q:, Q:] = Ct + tb * lam * Mt
        Lf[Q:, :Q] = -Nt
        P = time_dg.prolongation(q, ta / (ta + tb))
        np.testing.assert_allclose(P.T @ Lf @ P, Ct + (ta + tb) * lam * Mt, atol=1e-14)
        # coupling to the previous slab: fine first-slab trace coupling restricted equals coarse Nt
        Nf = np.zeros((2 * Q, Q)); Nf[:Q] = Nt
        Pprev = time_dg.prolongation(q, 0.5)[Q:]      # end of previous coarse slab -> its last fine slab
        np.testing.assert_allclose(P.T @ Nf @ Pprev, Nt, atol=1e-14)


@pytest.mark.parametrize("q", [0, 1])
def test_smoother_single_slab_halves_error(q):
    # m = 1 with exact block solve: error propagation (1 - omega) I (Eq. 2, omega = 0.5)
    E = lfa.smoother_matrix(q, 3.0, 0.1, 1)
    np.testing.assert_allclose(E, 0.5 * np.eye(q + 1), atol=1e-15)


def _rate(E, k=200):
    return np.linalg.norm(np.linalg.matrix_power(E, k), 2) ** (1.0 / k)


@pytest.mark.parametrize("q", [0, 1])
def test_two_grid_rate_bound(q):
    # "convergence rates mostly below 0.5 ... this rate is proven" for the
    # pure time multigrid with exact spatial solves: every eigenvalue lambda of M^{-1}K gives Eq. (4)
    for lt in [0.0, 0.01, 0.1, 1.0, 10.0, 100.0]:
        assert _rate(lfa.two_grid_matrix(q, lt, 1.0, 64)) <= 0.5


@pytest.mark.parametrize("q", [0, 1])
def test_high_lambda_limit(q):
    # "For lambda >> 1 the smoother converges fast" (l.141): each S with omega = 1/2 halves the error,
    # so one pre + one post step give 1/4 (with SAS's four S steps: 2^-4, l.289)
    assert _rate(lfa.two_grid_matrix(q, 1e4, 1.0, 32)) == pytest.approx(0.25, abs=2e-3)
    assert _rate(lfa.two_grid_matrix(q, 1e4, 1.0, 32, nu_pre=2, nu_post=2)) == pytest.approx(2 ** -4, abs=2e-3)


def test_lambda_zero_is_worst_case_for_smoother():
    # lambda = 0 is "the worst case" (l.140): the smoother alone barely converges there
    r0 = _rate(lfa.smoother_matrix(0, 0.0, 1.0, 64))
    r1 = _rate(lfa.smoother_matrix(0, 10.0, 1.0, 64))
    assert r0 > 0.9 and r1 < 0.6
