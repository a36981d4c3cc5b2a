"""Seeded synthetic inputs for the BASELINE.json workloads.

Shared by the oracle-side tests and the CUDA path (this module holds none of
the method's arithmetic: it only draws meshes, coefficients, slab lengths and
right-hand sides).  Recipe:

  c1  3D 4^3 uniform,  dG(1), 16 slabs tau=1/16, sigma=nu=1, f ~ U(-1,1) seed 0
  c2  2D 64^2 uniform, dG(1), 256 slabs, tau = lam*h^2, lam in {0.1,1,10}, f seed 1
  c3  3D 32^3, dG(1), 1024 slabs tau=1/1024, sigma=1 on the core [0.25,0.75]^3 else 1e-6,
      nu=1000 with p=0.1 else 1 (seed 2, then f from the same generator)
  c4  3D 64^3, dG(1), tau=1/4096, 512 slabs per GPU (weak scaling), f seed 3
  c5  3D 48^3, interior nodes jittered U(-0.2h,0.2h) seed 4, dG(1), 2048 slabs with
      geometric tau over [1e-4,1e-2], log-uniform sigma in [1e-3,1], nu in [1,100] and f (seed 5)

Space-time vectors are returned in the C-ABI layout [edge][time node a][slab]
(shape (n_edges, q+1, S)); the oracle uses the transpose (S, q+1, n_edges).
The random stream for f is drawn in the oracle layout order (slab-major), so
the values do not depend on which side consumes them.
"""
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Workload:
    name: str
    dim: int
    n: tuple
    q: int
    tau: np.ndarray                 # (S,) slab lengths
    sigma: np.ndarray               # (n_cells,)
    nu: np.ndarray                  # (n_cells,)
    coords: np.ndarray = None       # (n_nodes, dim) or None for the uniform unit mesh
    rhs_seed: int = 0
    rhs_rng_state: dict = field(default=None, repr=False)
    omega_s: float = 0.6

    @property
    def n_cells(self):
        return int(np.prod(self.n))

    @property
    def n_nodes(self):
        return int(np.prod([v + 1 for v in self.n]))

    @property
    def n_edges(self):
        if self.dim == 2:
            nx, ny = self.n
            return nx * (ny + 1) + (nx + 1) * ny
        nx, ny, nz = self.n
        return nx * (ny + 1) * (nz + 1) + (nx + 1) * ny * (nz + 1) + (nx + 1) * (ny + 1) * nz

    @property
    def S(self):
        return len(self.tau)

    def rhs(self):
        """f ~ U(-1,1) i.i.d. per (slab, time node, edge); returned as [edge][a][slab]."""
        if self.rhs_rng_state is not None:
            rng = np.random.default_rng()
            rng.bit_generator.state = self.rhs_rng_state
        else:
            rng = np.random.default_rng(self.rhs_seed)
        f = rng.uniform(-1.0, 1.0, size=(self.S, self.q + 1, self.n_edges))
        return np.ascontiguousarray(f.transpose(2, 1, 0))

    def rhs_device(self, device="cuda"):
        """Bench-size RHS drawn on the device: the same U(-1,1) i.i.d. recipe and seed, but
        torch's generator stream (not bit-identical to rhs()); ST layout."""
        import torch
        g = torch.Generator(device=device)
        g.manual_seed(self.rhs_seed)
        f = torch.empty((self.n_edges, self.q + 1, self.S), dtype=torch.float64, device=device)
        f.uniform_(-1.0, 1.0, generator=g)
        return f

    def uniform_coords(self):
        axes = [np.linspace(0.0, 1.0, v + 1) for v in self.n]
        grids = np.meshgrid(*axes[::-1], indexing="ij")[::-1]
        return np.stack([g.ravel() for g in grids], axis=1)

    def node_coords(self):
        return self.uniform_coords() if self.coords is None else self.coords


def to_oracle(x):
    """[edge][a][slab] -> oracle layout (slab, a, edge)."""
    return np.ascontiguousarray(np.asarray(x).transpose(2, 1, 0))


def from_oracle(X):
    return np.ascontiguousarray(np.asarray(X).transpose(2, 1, 0))


def _cell_centres(n):
    axes = [(np.arange(v) + 0.5) / v for v in n]
    grids = np.meshgrid(*axes[::-1], indexing="ij")[::-1]
    return np.stack([g.ravel() for g in grids], axis=1)


def c1(n=4, S=16):
    nc = n ** 3
    return Workload("c1", 3, (n, n, n), 1, np.full(S, 1.0 / S), np.ones(nc), np.ones(nc), rhs_seed=0)


def c2(lam=1.0, n=64, S=256):
    h = 1.0 / n
    nc = n * n
    return Workload(f"c2_lam{lam:g}", 2, (n, n), 1, np.full(S, lam * h * h), np.ones(nc), np.ones(nc),
                    rhs_seed=1, omega_s=0.5)


def c3(n=32, S=1024):
    rng = np.random.default_rng(2)
    c = _cell_centres((n, n, n))
    core = np.all((c > 0.25) & (c < 0.75), axis=1)
    sigma = np.where(core, 1.0, 1e-6)
    nu = np.where(rng.uniform(size=n ** 3) < 0.1, 1000.0, 1.0)
    w = Workload("c3", 3, (n, n, n), 1, np.full(S, 1.0 / S), sigma, nu)
    w.rhs_rng_state = rng.bit_generator.state
    return w


def c4(n=64, S=512, tau=1.0 / 4096):
    nc = n ** 3
    return Workload("c4", 3, (n, n, n), 1, np.full(S, tau), np.ones(nc), np.ones(nc), rhs_seed=3)


def c5(n=48, S=2048):
    rng = np.random.default_rng(4)
    nn = (n + 1) ** 3
    jit = rng.uniform(-0.2, 0.2, size=(nn, 3))
    # omega_s = 0.45: with the 3D default 0.6 the two block-Jacobi sweeps amplify on the full
    # 48^3 jittered mesh (measured divergence, R3)
    w = Workload("c5", 3, (n, n, n), 1, np.geomspace(1e-4, 1e-2, S), None, None, omega_s=0.45)
    X = w.uniform_coords()
    inner = np.all((X > 1e-12) & (X < 1 - 1e-12), axis=1)
    X[inner] += jit[inner] / n
    w.coords = X
    rng2 = np.random.default_rng(5)
    w.sigma = np.exp(rng2.uniform(np.log(1e-3), 0.0, size=n ** 3))
    w.nu = np.exp(rng2.uniform(0.0, np.log(100.0), size=n ** 3))
    w.rhs_rng_state = rng2.bit_generator.state
    return w


def small(name):
    """Oracle-sized variants (same recipe, fewer cells/slabs) for parity tests."""
    return {
        "c1": lambda: c1(),
        "c2": lambda: c2(1.0, n=16, S=32),
        "c2_lam0.1": lambda: c2(0.1, n=16, S=32),
        "c2_lam10": lambda: c2(10.0, n=16, S=32),
        "c3": lambda: c3(n=8, S=32),
        "c4": lambda: c4(n=8, S=16, tau=1.0 / 64),
        "c4_s64": lambda: c4(n=8, S=64, tau=1.0 / 64),
        "c5": lambda: c5(n=6, S=32),
    }[name]()
