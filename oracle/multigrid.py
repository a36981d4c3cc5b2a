"""Coarsening rule, hierarchy, transfers, V-cycle and solve - oracle.

PAPER.md references
  V-cycle           l.84   "pre-smoothing, a recursive coarse time-grid correction and post-smoothing"
  coarsening rule   l.105-109, Eq. (3): lambda(T) = min_{x in T} beta tau / (alpha h_T^2) >= lambda_crit
                    for all T  -> coarsen space together with time; else time only
  h_T               l.109  longest edge of the element
  lambda_crit       l.292  0.1 (3D eddy current, SAS)
Readings: R1 dG(q), R2 Sigma_t for dG(q), R3/R4 inner sweeps,
R6 spatial transfers / coarse coefficients, R7 time transfers, R8 coarsest solve.
"""
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import fem, time_dg
from .spacetime import Level, apply_L, hybrid_smooth, forward_solve


@dataclass
class Options:
    spec: str = "SAS"
    omega: float = 0.5          # Eq. (2)
    inner: str = "jacobi"       # 'jacobi' (default GPU path), 'mg' (inner spatial V-cycle, R13) or 'exact'
    nu_in: int = 2              # hybrid sweeps per side of the inner V-cycle (inner='mg')
    omega_in: float = 0.4       # its edge damping: D^{-1}A reaches ~4 (2D) and dG(2) blocks need margin
    nu_s: int = 2               # block-Jacobi sweeps approximating A_k^{-1}
    omega_s: float = 0.6        # 3D default; 2D workloads use 0.5 (R3)
    nu_n: int = 2               # Jacobi sweeps approximating K_n^{-1}
    omega_n: float = 0.6
    lambda_crit: float = 0.1    # l.292
    mode: str = "auto"          # 'auto' (Eq. 3 at every level), 'semi_time', 'full' (Table 1)
    min_slabs: int = 1


class Hierarchy:
    """levels[0] = finest.  space_coarsened[l] tells whether levels l -> l+1
    coarsened space as well as time."""

    def __init__(self, mesh, sigma, nu, tau, q, opts, ratio_min=None):
        self.opts = opts
        self.q = q
        self.levels = []
        self.space_coarsened = []
        self.P_edge = []
        self.lambdas = []
        sigma = np.asarray(sigma, float); nu = np.asarray(nu, float)
        tau = np.asarray(tau, float)
        ratio = nu / sigma if ratio_min is None else ratio_min
        lvl = 0
        while True:
            lv = Level(mesh, sigma, nu, tau, q)
            lv.ratio_min = ratio
            self.levels.append(lv)
            if len(tau) <= opts.min_slabs or len(tau) % 2:
                break
            lam = coarsening_lambda(mesh, ratio, tau)
            self.lambdas.append(lam)
            if opts.mode == "auto":
                coarsen_space = lam >= opts.lambda_crit and mesh.can_coarsen()
            elif opts.mode == "full":
                coarsen_space = lvl == 0 and mesh.can_coarsen()
            else:
                coarsen_space = False
            tau_c = tau[0::2] + tau[1::2]
            if coarsen_space:
                mc = mesh.coarsen()
                ch = mesh.child_cells()
                sigma = sigma[ch].mean(axis=1)
                nu = nu[ch].mean(axis=1)
                ratio = ratio[ch].min(axis=1)
                self.P_edge.append(fem.edge_prolongation(mesh, mc))
                mesh = mc
            else:
                self.P_edge.append(None)
            self.space_coarsened.append(coarsen_space)
            tau = tau_c
            lvl += 1

    def theta(self, l):
        """Split points of the coarse slabs of level l+1 in their reference coordinate."""
        tau = self.levels[l].tau
        return tau[0::2] / (tau[0::2] + tau[1::2])


def coarsening_lambda(mesh, ratio_min, tau):
    """min over cells T of  min_{x in T}(beta/alpha) * tau / h_T^2  (Eq. 3), beta = nu = mu^{-1},
    alpha = sigma; with non-uniform slabs the smallest tau of the level is used (reading R6)."""
    h = mesh.longest_edge()
    return float(np.min(ratio_min * np.min(tau) / h ** 2))


def restrict(H, l, R):
    """Fine residual (S, Q, n_f) -> coarse right-hand side (S/2, Q, n_c): R_t = P_t^T, R_s = P_edge^T."""
    q = H.q
    th = H.theta(l)
    S, Q, n = R.shape
    Fc = np.zeros((S // 2, Q, n), dtype=R.dtype)
    for K in range(S // 2):
        Pt = time_dg.prolongation(q, th[K])                  # (2Q, Q)
        pair = R[2 * K:2 * K + 2].reshape(2 * Q, n)
        Fc[K] = Pt.T @ pair
    Pe = H.P_edge[l]
    if Pe is not None:
        Fc = H.levels[l].spatial(Pe.T.tocsr(), Fc)
    return Fc


def prolongate(H, l, Xc):
    """Coarse correction (S/2, Q, n_c) -> fine (S, Q, n_f): P = P_t (x) P_edge."""
    q = H.q
    Pe = H.P_edge[l]
    if Pe is not None:
        Xc = H.levels[l].spatial(Pe, Xc)
    th = H.theta(l)
    Sc, Q, n = Xc.shape
    X = np.zeros((2 * Sc, Q, n), dtype=Xc.dtype)
    for K in range(Sc):
        Pt = time_dg.prolongation(q, th[K])
        X[2 * K:2 * K + 2] = (Pt @ Xc[K]).reshape(2, Q, n)
    return X


def vcycle(H, l, X, F):
    """One V-cycle on level l (l.84); coarsest level: exact forward substitution (R8)."""
    lv = H.levels[l]
    if l == len(H.levels) - 1:
        return forward_solve(lv, F)
    X = hybrid_smooth(lv, X, F, H.opts, "pre")
    R = F - apply_L(lv, X)
    Fc = restrict(H, l, R)
    Xc = vcycle(H, l + 1, np.zeros_like(Fc), Fc)
    X = X + prolongate(H, l, Xc)
    X = hybrid_smooth(lv, X, F, H.opts, "post")
    return X


def solve(H, F, tol=1e-8, maxit=100, X0=None):
    """V-cycles from X0 (default 0) until ||F - L X||_2 <= tol ||F||_2.
    Returns (X, history) with history[i] = ||r_i|| / ||F|| (history[0] = initial)."""
    lv = H.levels[0]
    X = np.zeros_like(F) if X0 is None else X0.copy()
    nf = np.linalg.norm(F)
    hist = [np.linalg.norm(F - apply_L(lv, X)) / nf]
    for _ in range(maxit):
        if hist[-1] <= tol:
            break
        X = vcycle(H, 0, X, F)
        hist.append(np.linalg.norm(F - apply_L(lv, X)) / nf)
    return X, hist


def assemble_L(lv):
    """Dense-able sparse matrix of the whole space-time system (for direct-solve pins)."""
    Q, n, S = lv.q + 1, lv.n, lv.S
    blocks = [[None] * S for _ in range(S)]
    for k in range(S):
        blocks[k][k] = sp.kron(lv.Ct, lv.M) + lv.tau[k] * sp.kron(lv.Mt, lv.K)
        if k > 0:
            blocks[k][k - 1] = -sp.kron(lv.Nt, lv.M)
    return sp.bmat(blocks, format="csr")
