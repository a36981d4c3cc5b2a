"""CPU-side checks of libst.so: exported C-ABI symbols and the host setup (plan,
assembled operators) against the independent oracle assembly.  No GPU needed."""
import os
import re

import numpy as np
import pytest
import scipy.sparse as sp

import workloads
from oracle import fem, mesh, multigrid as mg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def stlib():
    from paper_1911_09548_b200 import build
    build.build()
    import paper_1911_09548_b200 as p
    return p


def header_functions():
    src = open(os.path.join(ROOT, "include", "st.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(st_\w+)\s*\(", src, re.M)))


def test_header_symbols_exported(stlib):
    lib = stlib.load()
    names = header_functions()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(stlib.EXPORTED) == names


SMALL = ["c1", "c2", "c3", "c4", "c5", "c2_lam0.1", "c2_lam10"]


def _args(w):
    return (w.dim, w.n, w.sigma, w.nu, w.tau), dict(q=w.q, coords=w.coords, omega_s=w.omega_s)


@pytest.mark.parametrize("name", SMALL)
def test_plan_matches_oracle(stlib, name):
    w = workloads.small(name)
    a, kw = _args(w)
    info = stlib.plan(*a, **kw)
    H = mg.Hierarchy(mesh.Mesh(w.n, w.node_coords()), w.sigma, w.nu, w.tau, w.q, mg.Options(omega_s=w.omega_s))
    assert info["n_levels"] == len(H.levels)
    assert info["level_n_edges"] == [lv.n for lv in H.levels]
    assert info["level_n_slabs"] == [lv.S for lv in H.levels]
    assert info["level_space_coarsened"][:-1] == [int(c) for c in H.space_coarsened]
    np.testing.assert_allclose(info["level_lambda"][:-1], H.lambdas, rtol=1e-12)


def _to_csr(rows, width, col, val, ncols):
    r = np.repeat(np.arange(rows), width)
    return sp.csr_matrix((val.ravel(), (r, col.ravel())), shape=(rows, ncols))


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_host_operators_match_oracle(stlib, name):
    # The C++ setup and the oracle assemble M, K, K_n independently (different quadrature loops and
    # summation orders): every entry agrees to <= 32 ulps of its row's largest entry (measured <= 16).
    # This is the operator-rounding model behind the parity envelope (tests/parity_util.py).
    w = workloads.small(name)
    a, kw = _args(w)
    H = mg.Hierarchy(mesh.Mesh(w.n, w.node_coords()), w.sigma, w.nu, w.tau, w.q, mg.Options(omega_s=w.omega_s))
    for lvl in sorted({0, 1, len(H.levels) - 1}):
        lv = H.levels[lvl]
        for which, ref, ncols in ((0, lv.M, lv.n), (1, lv.K, lv.n), (2, lv.Kn, lv.nn)):
            A = _to_csr(*stlib.host_matrix(lvl, which, *a, **kw), ncols)
            D = (A - ref).tocoo()
            rowmax = np.asarray(abs(ref).max(axis=1).todense()).ravel()
            ulps = np.abs(D.data) / np.spacing(rowmax[D.row]) if D.nnz else np.zeros(1)
            assert ulps.max() <= 32, (name, lvl, which, ulps.max())
        if lvl < len(H.levels) - 1 and H.P_edge[lvl] is not None:
            P = _to_csr(*stlib.host_matrix(lvl, 3, *a, **kw), H.levels[lvl + 1].n)
            assert abs(P - H.P_edge[lvl]).max() == 0.0


def test_invalid_arguments_raise(stlib):
    w = workloads.small("c1")
    with pytest.raises(stlib.StError):
        stlib.plan(w.dim, w.n, -w.sigma, w.nu, w.tau)
    with pytest.raises(stlib.StError):
        stlib.plan(w.dim, w.n, w.sigma, w.nu, w.tau, spec="SXS")
    with pytest.raises(stlib.StError):
        stlib.plan(w.dim, w.n, w.sigma, w.nu, w.tau, q=5)
