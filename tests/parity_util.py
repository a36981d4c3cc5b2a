"""Rounding envelope of the oracle for GPU parity tests (R12).

Two correct fp64 implementations of the V-cycle differ by the rounding of their own arithmetic
AND by the rounding of their independently assembled operators (the C++ setup and the oracle agree
to <= 16 ulps of each row's scale, tests/test_lib_host.py).  The second matters: the nodal
correction integrates G^T K x over all slabs (Sigma_t, Eq. 5), which is zero in exact arithmetic
and pure operator rounding in fp64, so a 1-ulp change of K moves the V-cycle output by ~1e-13 on
the c4 recipe at 128 slabs, 20x more than a 1-ulp change of x or f.  The envelope is the larger of
the output change under one-ulp perturbations of (a) the inputs and (b) every operator entry
(M, K, K_n of every level); tests/test_oracle_precision.py pins (a) against an extended-precision
evaluation."""
import numpy as np

from oracle import mesh, multigrid as mg

EPS = np.finfo(np.float64).eps


def ulp_perturb(A, seed):
    """A with every entry moved by one unit in the last place (random sign)."""
    s = np.random.default_rng(seed).choice([-1.0, 1.0], size=np.shape(A))
    return A * (1.0 + s * EPS)


def hierarchy(w, **kw):
    return mg.Hierarchy(mesh.Mesh(w.n, w.node_coords()), w.sigma, w.nu, w.tau, w.q,
                        mg.Options(omega_s=w.omega_s, **kw))


def perturb_operators(H, seed=5):
    """Move every stored entry of M, K, K_n on every level by one ulp (random sign), in place."""
    rng = np.random.default_rng(seed)
    for lv in H.levels:
        for name in ("M", "K", "Kn"):
            A = getattr(lv, name).copy()
            A.data = A.data * (1.0 + rng.choice([-1.0, 1.0], size=A.data.shape) * EPS)
            setattr(lv, name, A)
        lv._Ainv = {}
        lv._Kn_lu = None
    return H


def vcycle_envelope(w, X0, F, **kw):
    """(X1, envelope): the oracle's V-cycle and the element-wise max change of it under one-ulp
    perturbations of the inputs and of the operators."""
    H = hierarchy(w, **kw)
    X1 = mg.vcycle(H, 0, X0.copy(), F)
    Xi = mg.vcycle(H, 0, ulp_perturb(X0, 99), ulp_perturb(F, 100))
    Xo = mg.vcycle(perturb_operators(hierarchy(w, **kw)), 0, X0.copy(), F)
    return H, X1, max(float(np.abs(Xi - X1).max()), float(np.abs(Xo - X1).max()))


def solve_envelope(w, F, tol, maxit, **kw):
    """(X, hist, hist_env, x_env): the oracle's solve, the per-iteration history envelope (max over
    one-ulp iterate perturbations every cycle and over perturbed operators) and the final-iterate
    envelope (norm)."""
    H = hierarchy(w, **kw)
    X, hist = mg.solve(H, F, tol=tol, maxit=maxit)
    lv, nf = H.levels[0], np.linalg.norm(F)
    env = np.zeros(len(hist))
    xenv = 0.0
    for rep in range(2):
        Xn, hn = np.zeros_like(F), [hist[0]]
        for i in range(len(hist) - 1):
            Xn = ulp_perturb(mg.vcycle(H, 0, Xn, F), 1000 * rep + i)
            hn.append(np.linalg.norm(F - mg.apply_L(lv, Xn)) / nf)
        env = np.maximum(env, np.abs(np.array(hn) - np.array(hist)))
        xenv = max(xenv, float(np.linalg.norm(Xn - X)))
    Hp = perturb_operators(hierarchy(w, **kw))
    Xp, hp = np.zeros_like(F), [hist[0]]
    for i in range(len(hist) - 1):
        Xp = mg.vcycle(Hp, 0, Xp, F)
        hp.append(np.linalg.norm(F - mg.apply_L(lv, Xp)) / nf)
    env = np.maximum(env, np.abs(np.array(hp) - np.array(hist)))
    xenv = max(xenv, float(np.linalg.norm(Xp - X)))
    return X, hist, env, xenv
