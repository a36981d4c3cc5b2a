"""GPU parity of the inner spatial V-cycle (reading R13, st_params.inner = 1) against the
oracle's SpatialChain: same seeded inputs, same tolerance rules as test_gpu_parity."""
import numpy as np
import pytest

import workloads
from oracle import multigrid as mg
from test_gpu_parity import ATOL_FLOOR, NOISE_MULT, RTOL, oracle_hierarchy, oracle_noise, solver, torch_cuda, ulp_perturb  # noqa: F401

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["c1", "c2_lam10", "c5", "c4"])
@pytest.mark.parametrize("q", [0, 1, 2])
@pytest.mark.parametrize("nu_in", [1, 2])
def test_inner_mg_vcycle_parity(torch_cuda, name, q, nu_in):
    torch = torch_cuda
    w = workloads.small(name)
    w.q = q
    rng = np.random.default_rng(31)
    F = rng.uniform(-1, 1, (w.S, q + 1, w.n_edges))
    X0 = rng.uniform(-1, 1, F.shape)
    H = oracle_hierarchy(w, inner="mg", nu_in=nu_in)
    X1 = mg.vcycle(H, 0, X0.copy(), F)
    noise = np.linalg.norm(oracle_noise(lambda a, b: mg.vcycle(H, 0, a, b), X0, F) - X1)
    s = solver(w, inner="mg", nu_in=nu_in)
    x = torch.from_numpy(workloads.from_oracle(X0)).cuda()
    s.vcycle(x, torch.from_numpy(workloads.from_oracle(F)).cuda())
    Xg = workloads.to_oracle(x.cpu().numpy())
    err = np.linalg.norm(Xg - X1)
    print(name, q, nu_in, "err", err / np.linalg.norm(X1), "noise", noise / np.linalg.norm(X1))
    assert err <= max(1e-12 * np.linalg.norm(X1), NOISE_MULT * noise)


# (name, maxit): the inner V-cycle converges where the block-Jacobi inner sweeps stagnate
# (c2 at lambda = 10, the c5 coefficient contrast)
@pytest.mark.parametrize("name,maxit", [("c1", 30), ("c2_lam10", 30), ("c5", 60), ("c4", 30)])
def test_inner_mg_solve_parity(torch_cuda, name, maxit):
    torch = torch_cuda
    w = workloads.small(name)
    H = oracle_hierarchy(w, inner="mg")
    F = workloads.to_oracle(w.rhs())
    X, hist = mg.solve(H, F, tol=1e-8, maxit=maxit)
    lv, nf = H.levels[0], np.linalg.norm(F)
    noise = np.zeros(len(hist))
    for rep in range(2):
        Xn, hist_n = np.zeros_like(F), [hist[0]]
        for i in range(len(hist) - 1):
            Xn = ulp_perturb(mg.vcycle(H, 0, Xn, F), 1000 * rep + i)
            hist_n.append(np.linalg.norm(F - mg.apply_L(lv, Xn)) / nf)
        noise = np.maximum(noise, np.abs(np.array(hist_n) - np.array(hist)))
    s = solver(w, inner="mg")
    f = torch.from_numpy(w.rhs()).cuda()
    x = torch.zeros_like(f)
    it, h = s.solve(x, f, tol=1e-8, maxit=maxit)
    print(name, "iterations", it, "oracle", len(hist) - 1, "final", h[-1])
    assert hist[-1] <= 1e-8, "the oracle itself must converge here"
    assert it == len(hist) - 1
    tol = np.maximum(np.maximum(RTOL * np.array(hist), ATOL_FLOOR), NOISE_MULT * noise)
    diff = np.abs(np.array(h) - np.array(hist))
    assert np.all(diff <= tol), (diff, tol)


def test_inner_mg_with_march_and_variants(torch_cuda):
    # the fused outer residual + first inner sweep also runs on the matrix-free march path, and
    # other smoother strings / nodal sweep counts compose with the inner cycle
    torch = torch_cuda
    w = workloads.small("c4")
    rng = np.random.default_rng(41)
    F = rng.uniform(-1, 1, (w.S, w.q + 1, w.n_edges))
    X0 = rng.uniform(-1, 1, F.shape)
    for kw in ({"kernel_path": 1}, {"spec": "ASSA", "nu_n": 3}, {"spec": "S", "omega_in": 0.3, "nu_in": 3}):
        okw = {k: v for k, v in kw.items() if k != "kernel_path"}
        H = oracle_hierarchy(w, inner="mg", **okw)
        X1 = mg.vcycle(H, 0, X0.copy(), F)
        noise = np.linalg.norm(oracle_noise(lambda a, b: mg.vcycle(H, 0, a, b), X0, F) - X1)
        s = solver(w, inner="mg", **kw)
        x = torch.from_numpy(workloads.from_oracle(X0)).cuda()
        s.vcycle(x, torch.from_numpy(workloads.from_oracle(F)).cuda())
        err = np.linalg.norm(workloads.to_oracle(x.cpu().numpy()) - X1)
        print(kw, "err", err / np.linalg.norm(X1))
        assert err <= max(1e-12 * np.linalg.norm(X1), NOISE_MULT * noise), kw
