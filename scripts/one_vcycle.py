"""Run a few full-size V-cycles of a BASELINE workload (default c4) through the C-ABI: a short,
deterministic command for ncu launch lists / single-kernel captures.

    python scripts/one_vcycle.py [c4|c5|c3] [cycles]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1911_09548_b200 as p  # noqa: E402
import workloads  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    w = {"c3": workloads.c3, "c4": workloads.c4, "c5": workloads.c5}[name]()
    s = p.Solver.from_workload(w)
    f = w.rhs_device()
    x = torch.zeros_like(f)
    for _ in range(cycles):
        s.vcycle(x, f)
    torch.cuda.synchronize()
    print(name, "cycles", cycles, "launches", s.info()["kernel_launches"], "variants", sorted(p.kernel_variants()))


if __name__ == "__main__":
    main()
