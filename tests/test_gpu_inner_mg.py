"""GPU parity of the inner spatial V-cycle (reading R13, st_params.inner = 1) against the
oracle's SpatialChain: same seeded inputs, same tolerance rules as test_gpu_parity."""
import numpy as np
import pytest

import workloads
from parity_util import solve_envelope, vcycle_envelope
from test_gpu_parity import ATOL_FLOOR, NOISE_MULT, RTOL, close_elementwise, solver, torch_cuda  # noqa: F401

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
    H, X1, env = vcycle_envelope(w, X0, F, inner="mg", nu_in=nu_in)
    s = solver(w, inner="mg", nu_in=nu_in)
    x = torch.from_numpy(workloads.from_oracle(X0)).cuda()
    s.vcycle(x, torch.from_numpy(workloads.from_oracle(F)).cuda())
    close_elementwise(workloads.to_oracle(x.cpu().numpy()), X1, env, f"{name} q={q} nu_in={nu_in}")


# (name, maxit): the inner V-cycle converges where the block-Jacobi inner sweeps stagnate
# (c2 at lambda = 10, the c5 coefficient contrast)
@pytest.mark.parametrize("name,maxit", [("c1", 30), ("c2_lam10", 30), ("c5", 60), ("c4", 30)])
def test_inner_mg_solve_parity(torch_cuda, name, maxit):
    torch = torch_cuda
    w = workloads.small(name)
    F = workloads.to_oracle(w.rhs())
    X, hist, noise, _ = solve_envelope(w, F, 1e-8, maxit, inner="mg")
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
        H, X1, env = vcycle_envelope(w, X0, F, inner="mg", **okw)
        s = solver(w, inner="mg", **kw)
        x = torch.from_numpy(workloads.from_oracle(X0)).cuda()
        s.vcycle(x, torch.from_numpy(workloads.from_oracle(F)).cuda())
        close_elementwise(workloads.to_oracle(x.cpu().numpy()), X1, env, str(kw))
