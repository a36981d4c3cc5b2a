"""GPU parity on the degenerate and ragged cases of the method: a single slab (the V-cycle is
the exact coarsest solve), odd and non-power-of-two slab counts (time coarsening stops early),
one-cell meshes, minimal 2D meshes, min_slabs > 1, and the Table-1 'full' / 'semi-time' modes."""
import numpy as np
import pytest

import workloads
from oracle import mesh, multigrid as mg

pytestmark = pytest.mark.gpu


def case(dim, n, S, q=1, seed=0, lam=1.0, jitter=False):
    nc = int(np.prod(n))
    rng = np.random.default_rng(seed)
    h = 1.0 / n[0]
    tau = lam * h * h * rng.uniform(0.5, 1.5, S)
    w = workloads.Workload("edge", dim, tuple(n), q, tau, rng.uniform(0.5, 2, nc), rng.uniform(0.5, 2, nc),
                           rhs_seed=seed, omega_s=0.6 if dim == 3 else 0.5)
    if jitter:
        X = w.uniform_coords()
        inner = np.all((X > 1e-12) & (X < 1 - 1e-12), axis=1)
        X[inner] += rng.uniform(-0.2, 0.2, X.shape)[inner] / np.array(n)
        w.coords = X
    return w


CASES = [
    ("single slab", dict(dim=3, n=(2, 2, 2), S=1)),
    ("three slabs", dict(dim=3, n=(2, 2, 2), S=3)),
    ("six slabs", dict(dim=3, n=(4, 4, 4), S=6)),
    ("one cell", dict(dim=3, n=(1, 1, 1), S=8)),
    ("2D 1x1", dict(dim=2, n=(1, 1), S=4)),
    ("2D 2x3 q0", dict(dim=2, n=(2, 3), S=8, q=0)),
    ("anisotropic box", dict(dim=3, n=(4, 2, 6), S=8)),
    ("q2 jittered", dict(dim=3, n=(4, 4, 4), S=8, q=2, jitter=True)),
    ("large lambda", dict(dim=3, n=(4, 4, 4), S=16, lam=50.0)),
    ("small lambda", dict(dim=2, n=(8, 8), S=16, lam=0.01)),
]


@pytest.mark.parametrize("label,kw", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("opts", [{}, {"mode": 1}, {"mode": 2}, {"min_slabs": 2}])
def test_edge_case_vcycle(label, kw, opts):
    import torch
    import paper_1911_09548_b200 as p
    from paper_1911_09548_b200 import build
    build.build()
    w = case(**kw)
    rng = np.random.default_rng(3)
    F = rng.uniform(-1, 1, (w.S, w.q + 1, w.n_edges))
    X0 = rng.uniform(-1, 1, F.shape)
    mode = {0: "auto", 1: "semi_time", 2: "full"}[opts.get("mode", 0)]
    H = mg.Hierarchy(mesh.Mesh(w.n, w.node_coords()), w.sigma, w.nu, w.tau, w.q,
                     mg.Options(omega_s=w.omega_s, mode=mode, min_slabs=opts.get("min_slabs", 1)))
    X1 = mg.vcycle(H, 0, X0.copy(), F)
    s = p.Solver.from_workload(w, **opts)
    assert s.info()["n_levels"] == len(H.levels)
    x = torch.from_numpy(workloads.from_oracle(X0)).cuda()
    f = torch.from_numpy(workloads.from_oracle(F)).cuda()
    s.vcycle(x, f)
    Xg = workloads.to_oracle(x.cpu().numpy())
    assert np.linalg.norm(Xg - X1) <= 1e-11 * np.linalg.norm(X1)
    if len(H.levels) == 1:
        # a single level is the exact forward substitution: the residual vanishes
        rn, fn = s.residual(x, f, norms=True)
        assert rn <= 1e-12 * fn


def test_too_many_slabs_for_one_gpu_is_refused():
    # the row kernels index a level's (edge, slab) pairs with 32-bit integers: 64^3 edges x 4096
    # slabs (3.3e9) is refused with st_setup's "unsupported" code instead of overflowing
    import paper_1911_09548_b200 as p
    w = workloads.c4(n=64, S=4096)
    with pytest.raises(p.StError, match="libst error 3"):
        p.Solver.from_workload(w)
