"""Time to solution (||f - L x|| / ||f|| <= 1e-8) on the BASELINE.json workloads at full size,
for both approximations of A_k^{-1} in the smoother S (block-Jacobi sweeps vs the inner spatial
V-cycle, R13).  Device-resident inputs; CUDA events on the solver's stream.

    python scripts/time_to_solution.py [--cases c3,c4,c5,c2_lam10] [--maxit 200]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import workloads  # noqa: E402

FULL = {"c1": lambda: workloads.c1(), "c2_lam0.1": lambda: workloads.c2(0.1), "c2": lambda: workloads.c2(1.0),
        "c2_lam10": lambda: workloads.c2(10.0), "c3": lambda: workloads.c3(), "c4": lambda: workloads.c4(),
        "c5": lambda: workloads.c5()}


def main():
    import torch
    import paper_1911_09548_b200 as p
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="c2_lam10,c3,c4,c5")
    ap.add_argument("--inner", default="jacobi,mg")
    ap.add_argument("--maxit", type=int, default=200)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--graphs", action="store_true", help="replay each V-cycle as a CUDA graph")
    ap.add_argument("--kw", default="{}", help="extra Solver keyword arguments (JSON), e.g. '{\"omega_s\": 0.4}'")
    args = ap.parse_args()
    for name in args.cases.split(","):
        w = FULL[name]()
        for inner in args.inner.split(","):
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                s = p.Solver.from_workload(w, stream=stream, inner=inner, **json.loads(args.kw))
                s.set_graphs(args.graphs)
                f = w.rhs_device()
                x = torch.zeros_like(f)
                s.vcycle(x, f)            # warm-up (first-launch costs, graph capture)
                x.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                stream.synchronize()
                e0.record(stream)
                it, hist = s.solve(x, f, tol=args.tol, maxit=args.maxit)
                e1.record(stream)
                stream.synchronize()
                ms = e0.elapsed_time(e1)
                mb = s.info()["device_bytes"] / 2 ** 20
                s.close()
            rate = (hist[-1] / hist[0]) ** (1.0 / max(it, 1))
            print(json.dumps({"case": name, "inner": inner, "kw": json.loads(args.kw), "graphs": args.graphs, "dofs": f.numel(), "iterations": it,
                              "final_rel_residual": hist[-1], "rate": rate, "ms_total": ms,
                              "ms_per_vcycle": ms / max(it, 1), "device_MiB": round(mb)}), flush=True)
            del x, f
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
