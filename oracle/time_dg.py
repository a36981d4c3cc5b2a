"""Discontinuous Galerkin dG(q) time discretisation on one slab - oracle.

The paper states the method for implicit Euler (Eq. (1));
the north-star workloads use dG(1).  Reading R1: the standard
upwind dG(q) time discretisation, which for q = 0 reproduces Eq. (1) exactly.
On a slab I_k = (t_{k-1}, t_k] of length tau_k with the nodal Lagrange basis
phi_0..phi_q at the equispaced reference points s_b = b/q of [0, 1]
(s = 0 for q = 0), the slab equations read, for every test function phi_b,

  sum_a [ Ct[b,a] M + tau_k Mt[b,a] K ] u_{k,a} - sum_a Nt[b,a] M u_{k-1,a} = f_{k,b}

  Mt[b,a] = \\int_0^1 phi_a phi_b ds
  Ct[b,a] = \\int_0^1 phi_a' phi_b ds + phi_a(0) phi_b(0)     (upwind jump)
  Nt[b,a] = phi_b(0) phi_a(1)                                  (previous-slab trace)

q = 0: Ct = Mt = Nt = [1]  ->  (M + tau K) u_k - M u_{k-1} = f_k, i.e. Eq. (1).
"""
import numpy as np


def nodes(q):
    return np.array([0.0]) if q == 0 else np.linspace(0.0, 1.0, q + 1)


def lagrange(q, s):
    """phi_a(s) for a = 0..q."""
    if q == 0:
        return np.array([1.0])
    x = nodes(q)
    out = np.ones(q + 1)
    for a in range(q + 1):
        for m in range(q + 1):
            if m != a:
                out[a] *= (s - x[m]) / (x[a] - x[m])
    return out


def lagrange_deriv(q, s):
    if q == 0:
        return np.array([0.0])
    x = nodes(q)
    out = np.zeros(q + 1)
    for a in range(q + 1):
        for skip in range(q + 1):
            if skip == a:
                continue
            term = 1.0 / (x[a] - x[skip])
            for m in range(q + 1):
                if m != a and m != skip:
                    term *= (s - x[m]) / (x[a] - x[m])
            out[a] += term
    return out


def time_matrices(q):
    """(Ct, Mt, Nt), each (q+1, q+1), indexed [test b, trial a]."""
    g, w = np.polynomial.legendre.leggauss(q + 2)
    g = 0.5 * (g + 1.0); w = 0.5 * w
    Mt = np.zeros((q + 1, q + 1)); Ct = np.zeros((q + 1, q + 1))
    for s, ws in zip(g, w):
        p = lagrange(q, s); dp = lagrange_deriv(q, s)
        Mt += ws * np.outer(p, p)
        Ct += ws * np.outer(p, dp)
    p0 = lagrange(q, 0.0); p1 = lagrange(q, 1.0)
    Ct += np.outer(p0, p0)
    Nt = np.outer(p0, p1)
    return Ct, Mt, Nt


def prolongation(q, theta):
    """P_t (2(q+1), q+1): the coarse slab's polynomial evaluated at the nodes of
    its two fine slabs; the split point is at reference coordinate theta
    (= tau_fine0 / (tau_fine0 + tau_fine1); 1/2 on uniform grids).  Rows are
    [fine slab 0 nodes, fine slab 1 nodes].  Restriction R_t = P_t^T."""
    x = nodes(q)
    rows = [lagrange(q, theta * s) for s in x] + [lagrange(q, theta + (1 - theta) * s) for s in x]
    return np.array(rows)
