"""The fp64 oracle's rounding error against an extended-precision evaluation of the same V-cycle
(np.longdouble: 64-bit significand, eps = 1.1e-19) - grounds the parity tolerances (R12).

The V-cycle is a fixed linear map of the fp64 operator entries; evaluated in long double its result
carries ~2^-11 of the fp64 rounding error, so |X_fp64 - X_ext| is the oracle's actual error.  The
parity tests scale their tolerance by the oracle's one-ulp input sensitivity ("noise"); this pins
that estimator: on every recipe the true error is within a small factor of it, including the
ill-conditioned c3 (sigma = 1e-6 insulators outside the paper's sigma >= 1) where
both are ~1e-6 relative."""
import numpy as np
import pytest

import workloads
from oracle import mesh, multigrid as mg


def ulp_perturb(A, seed):
    s = np.random.default_rng(seed).choice([-1.0, 1.0], size=A.shape)
    return A * (1.0 + s * np.finfo(np.float64).eps)


def vcycle_errors(name):
    w = workloads.small(name)
    H = mg.Hierarchy(mesh.Mesh(w.n, w.node_coords()), w.sigma, w.nu, w.tau, w.q, mg.Options(omega_s=w.omega_s))
    rng = np.random.default_rng(11)
    F = rng.uniform(-1, 1, (w.S, w.q + 1, w.n_edges))
    X0 = rng.uniform(-1, 1, F.shape)
    X1 = mg.vcycle(H, 0, X0.copy(), F)
    Xe = mg.vcycle(H, 0, X0.astype(np.longdouble), F.astype(np.longdouble))
    Xn = mg.vcycle(H, 0, ulp_perturb(X0, 99), ulp_perturb(F, 100))
    scale = float(np.abs(Xe).max())
    return float(np.abs(X1 - Xe).max()) / scale, float(np.abs(Xn - X1).max()) / scale


def test_extended_precision_path_is_extended():
    # the long-double V-cycle really runs in long double: on the well-conditioned c4 recipe it sits
    # ~1e-15 from fp64, and the long-double result of an exactly representable case is exact
    from oracle.spacetime import inv_blocks, dense_solve
    D = np.array([[[2.0, 1.0], [1.0, 3.0]]], dtype=np.longdouble)
    assert inv_blocks(D).dtype == np.longdouble
    np.testing.assert_array_equal(inv_blocks(D)[0] * 5, np.array([[3, -1], [-1, 2]], dtype=np.longdouble))
    x = dense_solve(np.array([[4.0, 2.0], [2.0, 3.0]], dtype=np.longdouble), np.array([2.0, 1.0], dtype=np.longdouble))
    np.testing.assert_array_equal(x * 8, np.array([4.0, 0.0], dtype=np.longdouble))
    err, noise = vcycle_errors("c4")
    assert 0 < err < 1e-14


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_noise_estimates_the_fp64_error(name):
    err, noise = vcycle_errors(name)
    print(f"{name}: |X_fp64 - X_ext| / max|X| = {err:.2e}, one-ulp noise {noise:.2e}, ratio {err / noise:.2f}")
    assert noise / 10 <= err <= 3 * noise
