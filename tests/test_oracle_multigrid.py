"""Pins of oracle/multigrid.py: coarsening rule (Eq. 3), Table 1 plans, V-cycle behaviour (§3.1, §4, §5)."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import lfa, mesh, multigrid as mg
import workloads


def golden():
    out = {}
    with open(__file__.replace("test_oracle_multigrid.py", "golden/paper_values.txt")) as fh:
        for line in fh:
            if line.strip() and not line.startswith("#"):
                k, v = line.split()[:2]
                out[k] = float(v)
    return out


PAPER = golden()


def power_rate(H, iters=30, seed=0):
    """random initial guess in [0,1), zero right-hand side, the maximal occurring
    l2 error reduction factor is the convergence rate."""
    lv = H.levels[0]
    X = np.random.default_rng(seed).uniform(0, 1, (lv.S, lv.q + 1, lv.n))
    F = np.zeros_like(X)
    nrm = [np.linalg.norm(X)]
    for _ in range(iters):
        X = mg.vcycle(H, 0, X, F)
        nrm.append(np.linalg.norm(X))
        if nrm[-1] / nrm[0] < 1e-100:
            break
    return max(nrm[i + 1] / nrm[i] for i in range(len(nrm) - 1))


def two_grid(lam, q, mode, spec, n=4, S=16):
    m = mesh.unit_mesh((n, n, n))
    tau = np.full(S, lam / n ** 2)
    o = mg.Options(inner="exact", mode=mode, spec=spec, min_slabs=S // 2)
    return mg.Hierarchy(m, np.ones(m.n_cells), np.ones(m.n_cells), tau, q, o)


@pytest.mark.parametrize("q", [0, 1])
@pytest.mark.parametrize("lam", [0.01, 1.0, 64.0])
def test_semi_time_two_grid_bound(q, lam):
    # pure time multigrid "convergence rates mostly below 0.5 ... this rate is proven"
    assert power_rate(two_grid(lam, q, "semi_time", "SAS")) <= PAPER["semi_time_rate_bound"] + 0.02


@pytest.mark.parametrize("q", [0, 1])
@pytest.mark.parametrize("lam", [0.01, 1.0, 64.0])
def test_spatial_coarsening_fails_without_nodal_correction(q, lam):
    # "A coarse grid correction with spatial coarsening is completely ineffective
    # regardless of lambda" (standard smoother S only, full coarsening)
    bad = power_rate(two_grid(lam, q, "full", "S"))
    good = power_rate(two_grid(lam, q, "semi_time", "SAS"))
    assert bad >= 0.85 and bad > 3 * good


@pytest.mark.parametrize("q", [0, 1])
def test_nodal_correction_restores_spatial_coarsening(q):
    # with SAS, "Full" behaves like "Semi-Time" for big enough lambda; the
    # high-lambda rate is 2^-4 (l.289: four S steps with omega = 1/2)
    r_full = power_rate(two_grid(64.0, q, "full", "SAS"))
    r_semi = power_rate(two_grid(64.0, q, "semi_time", "SAS"))
    assert abs(r_full - r_semi) <= 0.02
    assert r_full == pytest.approx(PAPER["high_lambda_rate"], abs=0.01)
    # and "deteriorates for lower lambda"
    assert power_rate(two_grid(0.01, q, "full", "SAS")) > 2 * r_full


def test_semi_time_plateau_matches_paper():
    # the "Semi-time" plateau rate 0.36 for low lambda.  The solenoidal modes at
    # low lambda obey the scalar test equation (l.145) smoothed by the four S steps of SAS; the
    # worst one-cycle reduction of that two-grid cycle is 1/(2 sqrt 2) = 0.354.
    E = lfa.two_grid_matrix(0, 0.0, 1.0, 64, nu_pre=2, nu_post=2)
    assert np.linalg.norm(E, 2) == pytest.approx(PAPER["semi_time_plateau_rate"], abs=0.01)


def test_table1_full_plan():
    # Table 1: 10 time levels, space level 2 only on the finest time level 9, level 1 below
    m = mesh.unit_mesh((2, 2, 2))
    o = mg.Options(mode="full")
    H = mg.Hierarchy(m, np.ones(8), np.ones(8), np.full(512, 0.01), 0, o)
    assert len(H.levels) == PAPER["table1_time_levels"]
    assert [lv.mesh.n[0] for lv in H.levels] == [2] + [1] * 9
    assert H.space_coarsened == [True] + [False] * 8


def test_auto_plan_follows_rule():
    # Eq. (3): coarsen space iff lambda >= lambda_crit; lambda halves under full and doubles under
    # semi-time coarsening.  8^3 mesh, 64 slabs, lambda_0 = 0.5, lambda_crit = 0.1:
    # 0.5 F, 0.25 F, 0.125 F, (1^3: cannot coarsen) T T T
    m = mesh.unit_mesh((8, 8, 8))
    H = mg.Hierarchy(m, np.ones(m.n_cells), np.ones(m.n_cells), np.full(64, 0.5 / 64), 0, mg.Options())
    assert H.space_coarsened == [True, True, True, False, False, False]
    np.testing.assert_allclose(H.lambdas, [0.5, 0.25, 0.125, 0.0625, 0.125, 0.25])
    assert [lv.mesh.n[0] for lv in H.levels] == [8, 4, 2, 1, 1, 1, 1]


def test_plan_depends_only_on_min_lambda():
    # §5.2 (l.298): "it is sufficient to only deal with the smallest lambda": raising nu on half the
    # cells (which raises lambda_2 only) leaves the plan unchanged
    m = mesh.unit_mesh((4, 4, 4))
    half = m.cell_ijk[:, 0] < 2
    tau = np.full(32, 0.3 / 16)
    plans = []
    for nu2 in (1.0, 10.0, 1e6):
        nu = np.where(half, nu2, 1.0)
        H = mg.Hierarchy(m, np.ones(m.n_cells), nu, tau, 0, mg.Options())
        plans.append(H.space_coarsened)
    assert plans[0] == plans[1] == plans[2]


def test_vcycle_solves_the_system():
    # V-cycles (GPU-path inner sweeps) converge to the direct solution of the whole space-time system
    w = workloads.c1()
    m = mesh.Mesh(w.n, w.node_coords())
    H = mg.Hierarchy(m, w.sigma, w.nu, w.tau, w.q, mg.Options())
    F = workloads.to_oracle(w.rhs())
    X, hist = mg.solve(H, F, tol=1e-11, maxit=60)
    Xd = spla.spsolve(mg.assemble_L(H.levels[0]).tocsc(), F.ravel()).reshape(F.shape)
    assert hist[-1] <= 1e-11
    np.testing.assert_allclose(X, Xd, atol=1e-8 * np.abs(Xd).max())
    assert len(hist) - 1 <= 20


def test_vcycle_is_linear_iteration():
    # error propagation independent of f (a fixed linear iteration)
    w = workloads.small("c2")
    m = mesh.Mesh(w.n, w.node_coords())
    H = mg.Hierarchy(m, w.sigma, w.nu, w.tau, w.q, mg.Options(omega_s=0.5))
    lv = H.levels[0]
    rng = np.random.default_rng(0)
    E0 = rng.normal(size=(lv.S, lv.q + 1, lv.n))
    errs = []
    for seed in (1, 2):
        Xs = np.random.default_rng(seed).normal(size=E0.shape)
        F = mg.apply_L(lv, Xs)
        errs.append(mg.vcycle(H, 0, Xs + E0, F) - Xs)
    np.testing.assert_allclose(errs[0], errs[1], atol=1e-11)


def test_solve_is_deterministic():
    w = workloads.c1()
    m = mesh.Mesh(w.n, w.node_coords())
    H = mg.Hierarchy(m, w.sigma, w.nu, w.tau, w.q, mg.Options())
    F = workloads.to_oracle(w.rhs())
    a = mg.solve(H, F, tol=1e-8)[1]
    b = mg.solve(H, F, tol=1e-8)[1]
    assert a == b
