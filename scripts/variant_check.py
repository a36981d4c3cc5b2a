"""Timing + a correctness check of one libst.so build (tuning variants): per-family V-cycle profile on
c4 and the stencil residual / one V-cycle against the assembled-ELL kernels of the same build
(ST_STENCIL=0) on the full c4 configuration.

    python scripts/variant_check.py path/to/libst.so [cycles]
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import workloads  # noqa: E402
from paper_1911_09548_b200 import binding as b  # noqa: E402


def main():
    path = sys.argv[1]
    cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    lib = ctypes.CDLL(path)
    w = workloads.c4()
    p, keep = b.make_params(w.dim, w.n, w.sigma, w.nu, w.tau, q=w.q, coords=w.coords, omega_s=w.omega_s)
    st = torch.cuda.Stream()
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    f = w.rhs_device()
    x0 = torch.empty_like(f).uniform_(-1, 1, generator=g)
    outs = {}
    for stencil in ("1", "0"):
        os.environ["ST_STENCIL"] = stencil
        h = ctypes.c_void_p()
        assert lib.st_setup(ctypes.byref(p), ctypes.byref(h)) == 0
        lib.st_set_stream(h, ctypes.c_void_p(st.cuda_stream))
        r = torch.empty_like(f)
        x = x0.clone()
        vp = lambda t: ctypes.c_void_p(t.data_ptr())   # noqa: E731
        assert lib.st_residual(h, vp(x), vp(f), vp(r), None) == 0
        assert lib.st_vcycle(h, vp(x), vp(f)) == 0
        st.synchronize()
        outs[stencil] = (r.clone(), x.clone())
        if stencil == "1":
            lib.st_profile(h, 1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(cycles):
                lib.st_vcycle(h, vp(x), vp(f))
            e1.record(st)
            st.synchronize()
            out = (b.StKstat * 64)()
            n = ctypes.c_int()
            lib.st_profile_read(h, out, 64, ctypes.byref(n))
            fams = {out[i].name.decode(): round(out[i].ms / cycles, 2) for i in range(n.value)}
            ms = e0.elapsed_time(e1) / cycles
        lib.st_free(h)
    dr = float((outs["1"][0] - outs["0"][0]).abs().max() / outs["0"][0].abs().max())
    dx = float((outs["1"][1] - outs["0"][1]).abs().max() / outs["0"][1].abs().max())
    print(f"{os.path.basename(path)}: {ms:.1f} ms/V-cycle {fams} | stencil vs ELL: residual {dr:.1e}, "
          f"V-cycle {dx:.1e}", flush=True)


if __name__ == "__main__":
    main()
