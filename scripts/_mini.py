import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1911_09548_b200 as p, workloads
nc = 8
w = workloads.Workload("stencil", 3, (2, 2, 2), 1, np.full(16, 1/16.), np.full(nc, 2.0), np.full(nc, 0.5), rhs_seed=7)
s = p.Solver.from_workload(w)
f = torch.from_numpy(w.rhs()).cuda(); x = torch.zeros_like(f); r = torch.empty_like(f)
for step in ["residual", "vcycle"]:
    try:
        if step == "residual": s.residual(x, f, r)
        else: s.vcycle(x, f)
        torch.cuda.synchronize(); print(step, "ok", p.kernel_variants())
    except Exception as e:
        print(step, "FAILED", e)
