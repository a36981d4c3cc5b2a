"""GPU parity of the structured stencil march (csrc/stencil.cuh) on its own edge cases: one-cell
and anisotropic uniform meshes, odd cell counts, dG(0) and dG(1), several slab chunks, non-unit
uniform coefficients, and agreement with the assembled-ELL kernels (ST_STENCIL=0).  The operator
is L of PAPER.md l.51-77 with M_sigma, K_nu of l.126-128."""
import numpy as np
import pytest

import workloads
from parity_util import vcycle_envelope
from test_gpu_parity import close_elementwise, torch_cuda  # noqa: F401

pytestmark = pytest.mark.gpu


def uniform_case(n, S, q, sigma=2.0, nu=0.5, lam=1.0):
    nc = int(np.prod(n))
    h = 1.0 / max(n)
    return workloads.Workload("stencil", 3, tuple(n), q, np.full(S, lam * h * h), np.full(nc, sigma), np.full(nc, nu),
                              rhs_seed=7)


# slab counts: multiples of the 32-slab warp chunk (the stencil's applicability condition)
CASES = [((1, 1, 1), 32, 1), ((2, 3, 4), 64, 1), ((4, 2, 6), 32, 1), ((5, 3, 3), 32, 1), ((3, 3, 3), 64, 0),
         ((6, 4, 2), 32, 0), ((8, 8, 8), 96, 1)]


@pytest.mark.parametrize("n,S,q", CASES, ids=[f"{c[0]}x{c[1]}q{c[2]}" for c in CASES])
def test_stencil_vcycle_parity(torch_cuda, n, S, q):
    import paper_1911_09548_b200 as p
    torch = torch_cuda
    w = uniform_case(n, S, q)
    rng = np.random.default_rng(13)
    F = rng.uniform(-1, 1, (S, q + 1, w.n_edges))
    X0 = rng.uniform(-1, 1, F.shape)
    H, X1, env = vcycle_envelope(w, X0, F)
    s = p.Solver.from_workload(w)
    x = torch.from_numpy(workloads.from_oracle(X0)).cuda()
    f = torch.from_numpy(workloads.from_oracle(F)).cuda()
    p.kernel_variants(reset=True)
    s.vcycle(x, f)
    torch.cuda.synchronize()
    ran = p.kernel_variants(reset=True)
    assert {"stencil/residual", "stencil/sweep", "stencil/node_scan"} <= ran, ran
    close_elementwise(workloads.to_oracle(x.cpu().numpy()), X1, env, f"stencil {n} S={S} q={q}")
    # the residual alone (every chunk-start coupling lane, boundary classes)
    r = torch.empty_like(f)
    s.residual(x, f, r)
    from oracle import multigrid as mg
    R = F - mg.apply_L(H.levels[0], workloads.to_oracle(x.cpu().numpy()))
    Rg = workloads.to_oracle(r.cpu().numpy())
    assert float(np.abs(Rg - R).max()) <= 1e-13 * max(float(np.abs(R).max()), 1.0)


@pytest.mark.parametrize("name", ["c4_8x128", "c1"])
def test_stencil_matches_ell(torch_cuda, name, monkeypatch):
    # same operator, gathered by the assembled ELL or marched by the stencil: equal to rounding
    import paper_1911_09548_b200 as p
    torch = torch_cuda
    w = workloads.c4(n=8, S=128, tau=1.0 / 64) if name == "c4_8x128" else workloads.small("c1")
    rng = np.random.default_rng(17)
    F = workloads.from_oracle(rng.uniform(-1, 1, (w.S, w.q + 1, w.n_edges)))
    X0 = workloads.from_oracle(rng.uniform(-1, 1, (w.S, w.q + 1, w.n_edges)))
    outs = []
    for env in ("1", "0"):
        monkeypatch.setenv("ST_STENCIL", env)
        s = p.Solver.from_workload(w)
        x = torch.from_numpy(X0).cuda()
        f = torch.from_numpy(F).cuda()
        r = torch.empty_like(f)
        s.residual(x, f, r)
        rn, _ = s.residual(x, f, norms=True)
        s.vcycle(x, f)
        torch.cuda.synchronize()
        outs.append((r.cpu().numpy(), rn, x.cpu().numpy()))
        s.close()
    monkeypatch.delenv("ST_STENCIL")
    scale = float(np.abs(outs[1][0]).max())
    assert float(np.abs(outs[0][0] - outs[1][0]).max()) <= 1e-13 * scale
    assert outs[0][1] == pytest.approx(outs[1][1], rel=1e-13)
    xs = float(np.abs(outs[1][2]).max())
    assert float(np.abs(outs[0][2] - outs[1][2]).max()) <= 1e-11 * xs


@pytest.mark.parametrize("nu_n", [1, 3])
def test_stencil_node_scan_modes(torch_cuda, nu_n):
    # the last nodal sweep with w read (nu_n = 3: MODE 2 of the structured node scan) and without a
    # sweep (nu_n = 1: the ELL scan), several chunks; Eq. (5) with Sigma_t of DESIGN.md R2
    import paper_1911_09548_b200 as p
    torch = torch_cuda
    w = uniform_case((4, 5, 6), 96, 1)
    rng = np.random.default_rng(23)
    F = rng.uniform(-1, 1, (w.S, w.q + 1, w.n_edges))
    X0 = rng.uniform(-1, 1, F.shape)
    H, X1, env = vcycle_envelope(w, X0, F, nu_n=nu_n)
    s = p.Solver.from_workload(w, nu_n=nu_n)
    x = torch.from_numpy(workloads.from_oracle(X0)).cuda()
    f = torch.from_numpy(workloads.from_oracle(F)).cuda()
    p.kernel_variants(reset=True)
    s.vcycle(x, f)
    torch.cuda.synchronize()
    ran = p.kernel_variants(reset=True)
    assert ("stencil/node_scan" in ran) == (nu_n > 1), ran
    close_elementwise(workloads.to_oracle(x.cpu().numpy()), X1, env, f"node scan nu_n={nu_n}")


def test_node_stencil_matches_ell(torch_cuda, monkeypatch):
    # the structured node scan and the ELL k_node_scan on the same V-cycle: equal to rounding
    import paper_1911_09548_b200 as p
    torch = torch_cuda
    w = workloads.c4(n=8, S=128, tau=1.0 / 64)
    rng = np.random.default_rng(29)
    F = workloads.from_oracle(rng.uniform(-1, 1, (w.S, w.q + 1, w.n_edges)))
    X0 = workloads.from_oracle(rng.uniform(-1, 1, (w.S, w.q + 1, w.n_edges)))
    outs = []
    for env in ("1", "0"):
        monkeypatch.setenv("ST_NODE_STENCIL", env)
        s = p.Solver.from_workload(w)
        x = torch.from_numpy(X0).cuda()
        f = torch.from_numpy(F).cuda()
        p.kernel_variants(reset=True)
        s.vcycle(x, f)
        torch.cuda.synchronize()
        assert ("stencil/node_scan" in p.kernel_variants(reset=True)) == (env == "1")
        outs.append(x.cpu().numpy())
        s.close()
    monkeypatch.delenv("ST_NODE_STENCIL")
    assert float(np.abs(outs[0] - outs[1]).max()) <= 1e-12 * float(np.abs(outs[1]).max())
