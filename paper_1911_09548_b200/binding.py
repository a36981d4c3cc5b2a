"""Thin ctypes binding of libst.so (include/st.h).  Argument marshalling only.

Device vectors are torch CUDA tensors (float64, contiguous, ST layout
[edge][time node][slab]); PyTorch provides the device memory and the stream.
Every arithmetic step runs in the library's CUDA kernels.  There is no CPU
fallback: if libst.so is missing or no CUDA device is present, calls raise.
"""
import ctypes
import os
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libst.so")

LEVEL_OPS = ["st_lv_count", "st_lv_get", "st_lv_residual", "st_lv_smooth_S", "st_lv_correct_local",
             "st_lv_correct_apply", "st_lv_restrict", "st_lv_prolong", "st_lv_vcycle", "st_lv_end_values",
             "st_copy_slabs", "st_zero", "st_vec_axpy", "st_vec_sum_blocks", "st_vec_norm2", "st_sync"]
EXPORTED = ["st_setup", "st_free", "st_set_stream", "st_residual", "st_vcycle", "st_set_graphs", "st_solve",
            "st_solve_host", "st_solve_many_host", "st_info", "st_profile", "st_profile_read", "st_plan", "st_host_matrix",
            *LEVEL_OPS, "st_kernel_variants", "st_variant_name", "st_last_error"]


class StParams(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int),
                ("coords", ctypes.POINTER(ctypes.c_double)),
                ("sigma", ctypes.POINTER(ctypes.c_double)), ("nu", ctypes.POINTER(ctypes.c_double)),
                ("tau", ctypes.POINTER(ctypes.c_double)), ("n_slabs", ctypes.c_int), ("q", ctypes.c_int),
                ("spec", ctypes.c_char_p), ("omega", ctypes.c_double), ("nu_s", ctypes.c_int),
                ("omega_s", ctypes.c_double), ("nu_n", ctypes.c_int), ("omega_n", ctypes.c_double),
                ("lambda_crit", ctypes.c_double), ("mode", ctypes.c_int), ("min_slabs", ctypes.c_int),
                ("kernel_path", ctypes.c_int), ("rank", ctypes.c_int), ("nranks", ctypes.c_int),
                ("inner", ctypes.c_int), ("nu_in", ctypes.c_int), ("omega_in", ctypes.c_double)]


class StInfo(ctypes.Structure):
    _fields_ = [("n_levels", ctypes.c_int), ("q", ctypes.c_int), ("n_dofs", ctypes.c_int64),
                ("level_n_edges", ctypes.c_int * 32), ("level_n_nodes", ctypes.c_int * 32),
                ("level_n_slabs", ctypes.c_int * 32), ("level_space_coarsened", ctypes.c_int * 32),
                ("level_lambda", ctypes.c_double * 32), ("kernel_launches", ctypes.c_int64),
                ("device_bytes", ctypes.c_int64), ("level_matrix_free", ctypes.c_int * 32)]


class StLevel(ctypes.Structure):
    _fields_ = [("set", ctypes.c_int), ("level", ctypes.c_int), ("global_level", ctypes.c_int),
                ("n_slabs", ctypes.c_int), ("slab0", ctypes.c_int), ("n_edges", ctypes.c_int),
                ("n_nodes", ctypes.c_int), ("q", ctypes.c_int), ("coarsest", ctypes.c_int),
                ("space_coarsened", ctypes.c_int), ("x", ctypes.c_void_p), ("f", ctypes.c_void_p),
                ("r", ctypes.c_void_p)]


class StKstat(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_int64), ("ms", ctypes.c_double),
                ("bytes", ctypes.c_double)]


_lib = None


def load():
    """Load libst.so (raises OSError if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise OSError(f"{LIB_PATH} not built: run `python -m paper_1911_09548_b200.build` (no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, dp, ip = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)
    lib.st_setup.argtypes = [ctypes.POINTER(StParams), ctypes.POINTER(vp)]
    lib.st_free.argtypes = [vp]
    lib.st_set_stream.argtypes = [vp, vp]
    lib.st_residual.argtypes = [vp, vp, vp, vp, dp]
    lib.st_vcycle.argtypes = [vp, vp, vp]
    lib.st_set_graphs.argtypes = [vp, ctypes.c_int]
    lib.st_solve.argtypes = [vp, vp, vp, ctypes.c_double, ctypes.c_int, ip, dp]
    lib.st_solve_host.argtypes = [vp, dp, dp, ctypes.c_double, ctypes.c_int, ip, dp]
    lib.st_solve_many_host.argtypes = [vp, ctypes.c_int, ctypes.POINTER(dp), ctypes.POINTER(dp), ctypes.c_int,
                                       ctypes.c_double, ctypes.c_int, ip, dp]
    lib.st_info.argtypes = [vp, ctypes.POINTER(StInfo)]
    lib.st_profile.argtypes = [vp, ctypes.c_int]
    lib.st_profile_read.argtypes = [vp, ctypes.POINTER(StKstat), ctypes.c_int, ip]
    lib.st_plan.argtypes = [ctypes.POINTER(StParams), ctypes.POINTER(StInfo)]
    lib.st_host_matrix.argtypes = [ctypes.POINTER(StParams), ctypes.c_int, ctypes.c_int, ip, ip, ip, dp]
    i64 = ctypes.c_int64
    ci = ctypes.c_int
    lib.st_lv_count.argtypes = [vp, ci, ip]
    lib.st_lv_get.argtypes = [vp, ci, ci, ctypes.POINTER(StLevel)]
    lib.st_lv_residual.argtypes = [vp, ci, ci, vp, vp, vp, vp, dp]
    lib.st_lv_smooth_S.argtypes = [vp, ci, ci, vp, vp, vp]
    lib.st_lv_correct_local.argtypes = [vp, ci, ci, vp, vp, vp, vp]
    lib.st_lv_correct_apply.argtypes = [vp, ci, ci, vp, vp]
    lib.st_lv_restrict.argtypes = [vp, ci, ci, vp, vp]
    lib.st_lv_prolong.argtypes = [vp, ci, ci, vp, vp]
    lib.st_lv_vcycle.argtypes = [vp, ci, ci, vp, vp]
    lib.st_lv_end_values.argtypes = [vp, ci, ci, vp, vp]
    lib.st_copy_slabs.argtypes = [vp, ci, ci, ci, vp, ci, ci, vp, ci, ci, ci]
    lib.st_zero.argtypes = [vp, vp, i64]
    lib.st_vec_axpy.argtypes = [vp, i64, ctypes.c_double, vp, vp]
    lib.st_vec_sum_blocks.argtypes = [vp, i64, ci, vp, vp]
    lib.st_vec_norm2.argtypes = [vp, i64, vp, dp]
    lib.st_sync.argtypes = [vp]
    lib.st_kernel_variants.argtypes = [ctypes.POINTER(ctypes.c_uint64), ci]
    lib.st_variant_name.argtypes = [ci]
    lib.st_variant_name.restype = ctypes.c_char_p
    lib.st_last_error.restype = ctypes.c_char_p
    for name in EXPORTED[:-3] + ["st_kernel_variants"]:
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


class StError(RuntimeError):
    pass


def kernel_variants(reset=False):
    """Names of the kernel variants launched by this process (st_kernel_variants)."""
    lib = load()
    mask = ctypes.c_uint64()
    _check(lib.st_kernel_variants(ctypes.byref(mask), 1 if reset else 0))
    out, i = set(), 0
    while True:
        name = lib.st_variant_name(i)
        if name is None:
            return out
        if mask.value >> i & 1:
            out.add(name.decode())
        i += 1


def _check(rc):
    if rc != 0:
        raise StError(f"libst error {rc}: {load().st_last_error().decode()}")


def _dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def make_params(dim, n, sigma, nu, tau, q=1, coords=None, spec="SAS", omega=0.5, nu_s=2, omega_s=None,
                nu_n=2, omega_n=0.6, lambda_crit=0.1, mode=0, min_slabs=1, kernel_path=0, rank=0, nranks=1,
                inner="jacobi", nu_in=2, omega_in=0.4):
    """Fill an StParams; returns (params, keep-alive list)."""
    keep = [np.ascontiguousarray(sigma, dtype=np.float64), np.ascontiguousarray(nu, dtype=np.float64),
            np.ascontiguousarray(tau, dtype=np.float64), spec.encode()]
    p = StParams()
    p.dim = dim
    p.nx, p.ny = int(n[0]), int(n[1])
    p.nz = int(n[2]) if dim == 3 else 1
    if coords is not None:
        c = np.ascontiguousarray(coords, dtype=np.float64)
        keep.append(c)
        p.coords = _dptr(c)
    p.sigma, p.nu, p.tau = _dptr(keep[0]), _dptr(keep[1]), _dptr(keep[2])
    p.n_slabs = len(keep[2])
    p.q = q
    p.spec = keep[3]
    p.omega, p.nu_s, p.nu_n, p.omega_n = omega, nu_s, nu_n, omega_n
    p.omega_s = omega_s if omega_s is not None else (0.6 if dim == 3 else 0.5)
    p.lambda_crit, p.mode, p.min_slabs = lambda_crit, mode, min_slabs
    p.kernel_path = kernel_path
    p.rank, p.nranks = rank, nranks
    if inner not in ("jacobi", "mg"):
        raise ValueError("inner must be 'jacobi' or 'mg'")
    p.inner, p.nu_in, p.omega_in = (1 if inner == "mg" else 0), nu_in, omega_in
    return p, keep


def _info_dict(inf):
    L = inf.n_levels
    return {"n_levels": L, "q": inf.q, "n_dofs": inf.n_dofs,
            "level_n_edges": list(inf.level_n_edges[:L]), "level_n_nodes": list(inf.level_n_nodes[:L]),
            "level_n_slabs": list(inf.level_n_slabs[:L]),
            "level_space_coarsened": list(inf.level_space_coarsened[:L]),
            "level_lambda": list(inf.level_lambda[:L]),
            "kernel_launches": inf.kernel_launches, "device_bytes": inf.device_bytes,
            "level_matrix_free": list(inf.level_matrix_free[:L])}


def plan(*args, **kw):
    """Host-only hierarchy plan (st_plan): no CUDA device needed."""
    p, keep = make_params(*args, **kw)
    inf = StInfo()
    _check(load().st_plan(ctypes.byref(p), ctypes.byref(inf)))
    return _info_dict(inf)


def host_matrix(level, which, *args, **kw):
    """Host-only assembled operator (st_host_matrix) as a dense-able (rows, width, col, val) tuple."""
    p, keep = make_params(*args, **kw)
    rows, width = ctypes.c_int(), ctypes.c_int()
    lib = load()
    _check(lib.st_host_matrix(ctypes.byref(p), level, which, ctypes.byref(rows), ctypes.byref(width), None, None))
    col = np.zeros(rows.value * width.value, dtype=np.int32)
    val = np.zeros(rows.value * width.value, dtype=np.float64)
    _check(lib.st_host_matrix(ctypes.byref(p), level, which, ctypes.byref(rows), ctypes.byref(width),
                              col.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), _dptr(val)))
    return rows.value, width.value, col.reshape(rows.value, width.value), val.reshape(rows.value, width.value)


class Solver:
    """Handle over st_setup for one workload (see workloads.Workload for the fields)."""

    def __init__(self, dim, n, sigma, nu, tau, q=1, coords=None, spec="SAS", omega=0.5, nu_s=2, omega_s=None,
                 nu_n=2, omega_n=0.6, lambda_crit=0.1, mode=0, min_slabs=1, kernel_path=0, rank=0, nranks=1,
                 inner="jacobi", nu_in=2, omega_in=0.4, stream=None):
        import torch
        if not torch.cuda.is_available():
            raise StError("no CUDA device: the space-time multigrid has no CPU path")
        lib = load()
        p, self._keep = make_params(dim, n, sigma, nu, tau, q=q, coords=coords, spec=spec, omega=omega, nu_s=nu_s,
                                    omega_s=omega_s, nu_n=nu_n, omega_n=omega_n, lambda_crit=lambda_crit, mode=mode,
                                    min_slabs=min_slabs, kernel_path=kernel_path, rank=rank, nranks=nranks,
                                    inner=inner, nu_in=nu_in, omega_in=omega_in)
        self.dim, self.n, self.q = dim, tuple(n), q
        self.rank, self.nranks = rank, max(nranks, 1)
        self.S = p.n_slabs // self.nranks          # slabs of this rank's block
        h = ctypes.c_void_p()
        _check(lib.st_setup(ctypes.byref(p), ctypes.byref(h)))
        self._h = h
        self.set_stream(stream if stream is not None else torch.cuda.current_stream())
        inf = self.info()
        self.n_edges = inf["level_n_edges"][0]
        self.shape = (self.n_edges, q + 1, self.S)

    @classmethod
    def from_workload(cls, w, **kw):
        kw.setdefault("omega_s", w.omega_s)
        return cls(w.dim, w.n, w.sigma, w.nu, w.tau, q=w.q, coords=w.coords, **kw)

    def set_stream(self, stream):
        self.stream = stream
        _check(load().st_set_stream(self._h, ctypes.c_void_p(stream.cuda_stream)))

    def close(self):
        if getattr(self, "_h", None):
            load().st_free(self._h)
            self._h = None

    def __del__(self):
        if sys is None or sys.is_finalizing():
            return          # the CUDA context may already be gone; the process exit frees everything
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _chk(t):
        import torch
        if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
            raise StError("expected a contiguous float64 CUDA tensor")
        if t.data_ptr() % 16:
            raise StError("expected a 16-byte aligned tensor (the kernels use 16-byte vector loads)")
        return ctypes.c_void_p(t.data_ptr())

    def residual(self, x, f, r=None, norms=False):
        out = (ctypes.c_double * 2)()
        _check(load().st_residual(self._h, self._chk(x), self._chk(f), self._chk(r) if r is not None else None,
                                  out if norms else None))
        return (out[0], out[1]) if norms else None

    def vcycle(self, x, f):
        _check(load().st_vcycle(self._h, self._chk(x), self._chk(f)))

    def set_graphs(self, enable=True):
        """Replay the V-cycle as a captured CUDA graph per (x, f) pair (st_set_graphs)."""
        _check(load().st_set_graphs(self._h, 1 if enable else 0))

    def solve(self, x, f, tol=1e-8, maxit=100):
        it = ctypes.c_int()
        hist = (ctypes.c_double * (maxit + 1))()
        _check(load().st_solve(self._h, self._chk(x), self._chk(f), tol, maxit, ctypes.byref(it), hist))
        return it.value, list(hist[: it.value + 1])

    def solve_host(self, x, f, tol=1e-8, maxit=100):
        """x (in/out) and f: host numpy float64 arrays in ST layout."""
        assert x.dtype == np.float64 and f.dtype == np.float64 and x.flags.c_contiguous and f.flags.c_contiguous
        it = ctypes.c_int()
        hist = (ctypes.c_double * (maxit + 1))()
        _check(load().st_solve_host(self._h, _dptr(x), _dptr(f), tol, maxit, ctypes.byref(it), hist))
        return it.value, list(hist[: it.value + 1])

    def solve_many_host(self, xs, fs, tol=1e-8, maxit=100, init_from_x=False, history=True):
        """Streaming solves of independent problems (st_solve_many_host): xs (out, or in/out with
        init_from_x) and fs are lists of host float64 arrays in ST layout (page-locked memory,
        e.g. torch's pin_memory().numpy(), lets the copies overlap the solves).  Returns
        (iterations, histories) per problem."""
        n = len(fs)
        assert len(xs) == n
        for a in list(xs) + list(fs):
            assert a.dtype == np.float64 and a.flags.c_contiguous and a.size == self.n_edges * (self.q + 1) * self.S
        X = (ctypes.POINTER(ctypes.c_double) * n)(*[_dptr(a) for a in xs])
        F = (ctypes.POINTER(ctypes.c_double) * n)(*[_dptr(a) for a in fs])
        it = (ctypes.c_int * max(n, 1))()
        hist = (ctypes.c_double * max(n * (maxit + 1), 1))() if history else None
        _check(load().st_solve_many_host(self._h, n, X, F, 1 if init_from_x else 0, tol, maxit, it, hist))
        if not history:       # (tol <= 0 then runs exactly maxit cycles without norms)
            return [it[i] for i in range(n)], None
        return [it[i] for i in range(n)], [list(hist[i * (maxit + 1): i * (maxit + 1) + it[i] + 1]) for i in range(n)]

    # ---- level operations (multi-GPU driver: distributed.py) -------------------------
    def level(self, set_, level):
        out = StLevel()
        _check(load().st_lv_get(self._h, set_, level, ctypes.byref(out)))
        return out

    def n_levels(self, set_):
        n = ctypes.c_int()
        _check(load().st_lv_count(self._h, set_, ctypes.byref(n)))
        return n.value

    def lv(self, name, *args):
        """Call st_lv_<name>(handle, *args); tensors are passed as device pointers, None as NULL."""
        conv = []
        for a in args:
            if a is None:
                conv.append(None)
            elif hasattr(a, "data_ptr"):
                conv.append(ctypes.c_void_p(a.data_ptr()))
            else:
                conv.append(a)
        _check(getattr(load(), "st_lv_" + name)(self._h, *conv))

    def lv_residual_norm2(self, set_, level, x, f, prev):
        out = ctypes.c_double()
        _check(load().st_lv_residual(self._h, set_, level, ctypes.c_void_p(x.data_ptr()),
                                     ctypes.c_void_p(f.data_ptr()),
                                     ctypes.c_void_p(prev.data_ptr()) if prev is not None else None,
                                     None, ctypes.byref(out)))
        return out.value

    def copy_slabs(self, rows, ns, dst, dS, dk0, src, sS, sk0, add=False):
        _check(load().st_copy_slabs(self._h, rows, self.q, ns, ctypes.c_void_p(dst.data_ptr()), dS, dk0,
                                    ctypes.c_void_p(src.data_ptr()), sS, sk0, 1 if add else 0))

    def zero(self, t):
        _check(load().st_zero(self._h, ctypes.c_void_p(t.data_ptr()), t.numel()))

    def axpy(self, alpha, x, y):
        """y += alpha x (device tensors of equal size), st_vec_axpy."""
        assert x.numel() == y.numel()
        _check(load().st_vec_axpy(self._h, y.numel(), alpha, ctypes.c_void_p(x.data_ptr()),
                                  ctypes.c_void_p(y.data_ptr())))

    def sum_blocks(self, blocks, nb, out):
        """out = sum of the first nb rows of blocks (nb x n device tensor), st_vec_sum_blocks."""
        _check(load().st_vec_sum_blocks(self._h, out.numel(), nb, ctypes.c_void_p(blocks.data_ptr()),
                                        ctypes.c_void_p(out.data_ptr())))

    def norm2(self, v):
        """||v||_2^2 of a device tensor, st_vec_norm2."""
        out = ctypes.c_double()
        _check(load().st_vec_norm2(self._h, v.numel(), ctypes.c_void_p(v.data_ptr()), ctypes.byref(out)))
        return out.value

    def sync(self):
        _check(load().st_sync(self._h))

    def profile(self, enable=True):
        _check(load().st_profile(self._h, 1 if enable else 0))

    def profile_read(self):
        """{family: (launches, ms, algorithmic bytes)} of the launches recorded since profile(True)."""
        out = (StKstat * 64)()
        n = ctypes.c_int()
        _check(load().st_profile_read(self._h, out, 64, ctypes.byref(n)))
        return {out[i].name.decode(): (out[i].launches, out[i].ms, out[i].bytes) for i in range(min(n.value, 64))}

    def info(self):
        inf = StInfo()
        _check(load().st_info(self._h, ctypes.byref(inf)))
        return _info_dict(inf)
