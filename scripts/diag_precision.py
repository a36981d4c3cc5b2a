"""Diagnostic: GPU vs fp64 oracle vs long-double oracle for one V-cycle on a recipe, per smoother
variant (which step of the V-cycle carries the GPU's rounding difference).

    python scripts/diag_precision.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1911_09548_b200 as p  # noqa: E402
import workloads  # noqa: E402
from oracle import mesh, multigrid as mg  # noqa: E402

MODES = {0: "auto", 1: "semi_time", 2: "full"}


def run(w, spec="SAS", mode=0, min_slabs=1, nu_s=2, nu_n=2):
    H = mg.Hierarchy(mesh.Mesh(w.n, w.node_coords()), w.sigma, w.nu, w.tau, w.q,
                     mg.Options(omega_s=w.omega_s, spec=spec, mode=MODES[mode], min_slabs=min_slabs, nu_s=nu_s,
                                nu_n=nu_n))
    rng = np.random.default_rng(11)
    F = rng.uniform(-1, 1, (w.S, w.q + 1, w.n_edges))
    X0 = rng.uniform(-1, 1, F.shape)
    X1 = mg.vcycle(H, 0, X0.copy(), F)
    Xe = mg.vcycle(H, 0, X0.astype(np.longdouble), F.astype(np.longdouble)).astype(np.float64)
    s = p.Solver.from_workload(w, spec=spec, mode=mode, min_slabs=min_slabs, nu_s=nu_s, nu_n=nu_n)
    x = torch.from_numpy(workloads.from_oracle(X0)).cuda()
    f = torch.from_numpy(workloads.from_oracle(F)).cuda()
    s.vcycle(x, f)
    Xg = workloads.to_oracle(x.cpu().numpy())
    sc = float(np.abs(Xe).max())
    e_or, e_g = float(np.abs(X1 - Xe).max()) / sc, float(np.abs(Xg - Xe).max()) / sc
    print(f"spec={spec:4s} mode={mode} min_slabs={min_slabs} nu_s={nu_s} nu_n={nu_n} levels={len(H.levels)}: "
          f"oracle {e_or:.2e}  gpu {e_g:.2e}  x{e_g / e_or:.1f}", flush=True)


if __name__ == "__main__":
    w = workloads.c4(n=8, S=128, tau=1.0 / 64)
    run(w)
    run(w, spec="S")
    run(w, spec="A")
    run(w, mode=1)
    run(w, min_slabs=64)
    run(w, spec="S", min_slabs=64)
    run(w, spec="A", min_slabs=64)
    run(w, spec="A", min_slabs=64, nu_n=1)
    run(w, spec="S", min_slabs=64, nu_s=1)
    w2 = workloads.c4(n=8, S=16, tau=1.0 / 64)
    run(w2, spec="A", min_slabs=8)
    run(w2, spec="S", min_slabs=8)
