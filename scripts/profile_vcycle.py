"""Per-kernel-family CUDA-event profile of full-size V-cycles on one BASELINE workload, through a
given libst.so (to compare builds, e.g. an older commit's library against the current one).

    python scripts/profile_vcycle.py [path/to/libst.so] [c4|c5|c3] [cycles]
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import workloads  # noqa: E402
from paper_1911_09548_b200 import binding as b  # noqa: E402


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else b.LIB_PATH
    name = sys.argv[2] if len(sys.argv) > 2 else "c5"
    cycles = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    lib = ctypes.CDLL(path)        # only entry points every version exports
    w = {"c3": workloads.c3, "c4": workloads.c4, "c5": workloads.c5}[name]()
    p, keep = b.make_params(w.dim, w.n, w.sigma, w.nu, w.tau, q=w.q, coords=w.coords, omega_s=w.omega_s)
    h = ctypes.c_void_p()
    assert lib.st_setup(ctypes.byref(p), ctypes.byref(h)) == 0, lib
    st = torch.cuda.Stream()
    lib.st_set_stream(h, ctypes.c_void_p(st.cuda_stream))
    f = w.rhs_device()
    x = torch.zeros_like(f)
    xp, fp = ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(f.data_ptr())
    torch.cuda.synchronize()
    lib.st_vcycle(h, xp, fp)
    st.synchronize()
    lib.st_profile(h, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(cycles):
        lib.st_vcycle(h, xp, fp)
    e1.record(st)
    st.synchronize()
    out = (b.StKstat * 64)()
    n = ctypes.c_int()
    lib.st_profile_read(h, out, 64, ctypes.byref(n))
    fams = {out[i].name.decode(): (out[i].launches, round(out[i].ms, 1)) for i in range(n.value)}
    print(os.path.basename(path), name, "ms/V-cycle %.1f" % (e0.elapsed_time(e1) / cycles), fams)
    lib.st_free(h)


if __name__ == "__main__":
    main()
