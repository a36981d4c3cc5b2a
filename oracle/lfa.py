"""Scalar test-equation analysis (§3.2, Eq. (4): u' + lambda u = f) - oracle.

The paper's LFA (l.210-226) diagonalises the semi-discrete system by the
eigenvectors of M^{-1} K (l.145); each eigenvalue lambda gives the scalar
test equation.  This module builds the exact dense iteration matrices of the
block-Jacobi smoother (Eq. 2) and of the two-grid cycle in time for that
scalar problem, with dG(q) time stepping on m uniform slabs of length tau.
"""
import numpy as np

from . import time_dg


def scalar_L(q, lam, tau, m):
    """Dense space-time matrix of u' + lam u with dG(q), M = 1, K = lam."""
    Ct, Mt, Nt = time_dg.time_matrices(q)
    Q = q + 1
    A = Ct + tau * lam * Mt
    L = np.zeros((m * Q, m * Q))
    for k in range(m):
        L[k * Q:(k + 1) * Q, k * Q:(k + 1) * Q] = A
        if k:
            L[k * Q:(k + 1) * Q, (k - 1) * Q:k * Q] = -Nt
    return L


def smoother_matrix(q, lam, tau, m, omega=0.5):
    """Error propagation of Eq. (2) with exact block solves: I - omega D^{-1} L."""
    L = scalar_L(q, lam, tau, m)
    Q = q + 1
    D = np.zeros_like(L)
    for k in range(m):
        s = slice(k * Q, (k + 1) * Q)
        D[s, s] = L[s, s]
    return np.eye(m * Q) - omega * np.linalg.solve(D, L)


def time_prolongation(q, m_coarse):
    Q = q + 1
    P = np.zeros((2 * m_coarse * Q, m_coarse * Q))
    Pt = time_dg.prolongation(q, 0.5)
    for K in range(m_coarse):
        P[2 * K * Q:(2 * K + 2) * Q, K * Q:(K + 1) * Q] = Pt
    return P


def two_grid_matrix(q, lam, tau, m, nu_pre=1, nu_post=1, omega=0.5):
    """E = S^nu_post (I - P L_c^{-1} P^T L) S^nu_pre, coarse problem (tau_c = 2 tau) solved exactly."""
    L = scalar_L(q, lam, tau, m)
    Lc = scalar_L(q, lam, 2 * tau, m // 2)
    P = time_prolongation(q, m // 2)
    Sm = smoother_matrix(q, lam, tau, m, omega)
    C = np.eye(L.shape[0]) - P @ np.linalg.solve(Lc, P.T @ L)
    return np.linalg.matrix_power(Sm, nu_post) @ C @ np.linalg.matrix_power(Sm, nu_pre)


def spectral_radius(E):
    return float(np.max(np.abs(np.linalg.eigvals(E))))
