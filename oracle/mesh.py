"""Structured hexahedral (3D) / quadrilateral (2D) meshes of the unit cube/square.

Oracle (test infrastructure).  The paper's experiments (§5.1)
use refined tetrahedra; the north-star workloads (BASELINE.json configs) use
tensor-product hex/quad meshes, which this module enumerates.  Numbering
conventions (shared *by specification*, not by code, with include/st.h):

  node  (i,j[,k])            id = i + (nx+1)*(j + (ny+1)*k)
  x-edge (i,j,k), i<nx       id = i + nx*(j + (ny+1)*k)                       (block 0)
  y-edge (i,j,k), j<ny       id = Ex + i + (nx+1)*(j + ny*k)                  (block 1)
  z-edge (i,j,k), k<nz       id = Ex + Ey + i + (nx+1)*(j + (ny+1)*k)         (block 2)
  cell  (i,j,k)              id = i + nx*(j + ny*k)

Every edge is oriented from its lower to its higher node id (the +axis
direction).  Local (reference) edge order inside a 3D cell:
  x-edges (b,c) -> b + 2c ; y-edges (a,c) -> 4 + a + 2c ; z-edges (a,b) -> 8 + a + 2b
where a,b,c in {0,1} are the local offsets in x,y,z.  In 2D: x-edges b -> b,
y-edges a -> 2 + a.  Local node order: a + 2b (+ 4c).
"""
import numpy as np


class Mesh:
    def __init__(self, n, coords):
        self.n = tuple(int(v) for v in n)
        self.dim = len(self.n)
        assert self.dim in (2, 3)
        self.coords = np.asarray(coords, dtype=np.float64)
        nn = np.prod([v + 1 for v in self.n])
        assert self.coords.shape == (nn, self.dim)
        self._build()

    # -- enumeration -------------------------------------------------------
    def node_id(self, i, j, k=0):
        nx, ny = self.n[0], self.n[1]
        return i + (nx + 1) * (j + (ny + 1) * k)

    def _build(self):
        if self.dim == 2:
            nx, ny = self.n
            self.n_nodes = (nx + 1) * (ny + 1)
            self.Ex = nx * (ny + 1)
            self.Ey = (nx + 1) * ny
            self.n_edges = self.Ex + self.Ey
            self.n_cells = nx * ny
            # edge -> (start node, end node)
            en = np.zeros((self.n_edges, 2), dtype=np.int64)
            j, i = np.meshgrid(np.arange(ny + 1), np.arange(nx), indexing="ij")
            ids = i + nx * j
            en[ids.ravel(), 0] = self.node_id(i, j).ravel()
            en[ids.ravel(), 1] = self.node_id(i + 1, j).ravel()
            j, i = np.meshgrid(np.arange(ny), np.arange(nx + 1), indexing="ij")
            ids = self.Ex + i + (nx + 1) * j
            en[ids.ravel(), 0] = self.node_id(i, j).ravel()
            en[ids.ravel(), 1] = self.node_id(i, j + 1).ravel()
            self.edge_nodes = en
            j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
            i = i.ravel(); j = j.ravel()
            ce = np.zeros((self.n_cells, 4), dtype=np.int64)
            for b in range(2):
                ce[:, b] = i + nx * (j + b)
            for a in range(2):
                ce[:, 2 + a] = self.Ex + (i + a) + (nx + 1) * j
            cn = np.zeros((self.n_cells, 4), dtype=np.int64)
            for b in range(2):
                for a in range(2):
                    cn[:, a + 2 * b] = self.node_id(i + a, j + b)
            self.cell_edges = ce
            self.cell_nodes = cn
            self.cell_ijk = np.stack([i, j], axis=1)
        else:
            nx, ny, nz = self.n
            self.n_nodes = (nx + 1) * (ny + 1) * (nz + 1)
            self.Ex = nx * (ny + 1) * (nz + 1)
            self.Ey = (nx + 1) * ny * (nz + 1)
            self.Ez = (nx + 1) * (ny + 1) * nz
            self.n_edges = self.Ex + self.Ey + self.Ez
            self.n_cells = nx * ny * nz
            en = np.zeros((self.n_edges, 2), dtype=np.int64)
            k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx), indexing="ij")
            ids = (i + nx * (j + (ny + 1) * k)).ravel()
            en[ids, 0] = self.node_id(i, j, k).ravel()
            en[ids, 1] = self.node_id(i + 1, j, k).ravel()
            k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny), np.arange(nx + 1), indexing="ij")
            ids = (self.Ex + i + (nx + 1) * (j + ny * k)).ravel()
            en[ids, 0] = self.node_id(i, j, k).ravel()
            en[ids, 1] = self.node_id(i, j + 1, k).ravel()
            k, j, i = np.meshgrid(np.arange(nz), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
            ids = (self.Ex + self.Ey + i + (nx + 1) * (j + (ny + 1) * k)).ravel()
            en[ids, 0] = self.node_id(i, j, k).ravel()
            en[ids, 1] = self.node_id(i, j, k + 1).ravel()
            self.edge_nodes = en
            k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
            i = i.ravel(); j = j.ravel(); k = k.ravel()
            ce = np.zeros((self.n_cells, 12), dtype=np.int64)
            for c in range(2):
                for b in range(2):
                    ce[:, b + 2 * c] = i + nx * ((j + b) + (ny + 1) * (k + c))
            for c in range(2):
                for a in range(2):
                    ce[:, 4 + a + 2 * c] = self.Ex + (i + a) + (nx + 1) * (j + ny * (k + c))
            for b in range(2):
                for a in range(2):
                    ce[:, 8 + a + 2 * b] = self.Ex + self.Ey + (i + a) + (nx + 1) * ((j + b) + (ny + 1) * k)
            cn = np.zeros((self.n_cells, 8), dtype=np.int64)
            for c in range(2):
                for b in range(2):
                    for a in range(2):
                        cn[:, a + 2 * b + 4 * c] = self.node_id(i + a, j + b, k + c)
            self.cell_edges = ce
            self.cell_nodes = cn
            self.cell_ijk = np.stack([i, j, k], axis=1)

    # -- geometry ----------------------------------------------------------
    def longest_edge(self):
        """h_T per cell: "the length of the longest edge" (§2.2)."""
        cn = self.cell_nodes
        X = self.coords
        # the cell's edges are the local node pairs that differ in one offset bit
        pairs = []
        nloc = cn.shape[1]
        for p in range(nloc):
            for d in range(self.dim):
                if not (p >> d) & 1:
                    pairs.append((p, p | (1 << d)))
        h = np.zeros(self.n_cells)
        for p, q in pairs:
            h = np.maximum(h, np.linalg.norm(X[cn[:, q]] - X[cn[:, p]], axis=1))
        return h

    def can_coarsen(self):
        return all(v % 2 == 0 and v >= 2 for v in self.n)

    def coarsen(self):
        """Coarse mesh made of the fine nodes with all-even indices (nested for
        uniform meshes; for jittered meshes the coarse cells are the trilinear
        hexes through those nodes - DESIGN.md reading R6)."""
        assert self.can_coarsen()
        nc = tuple(v // 2 for v in self.n)
        if self.dim == 2:
            J, I = np.meshgrid(np.arange(nc[1] + 1), np.arange(nc[0] + 1), indexing="ij")
            ids = self.node_id(2 * I, 2 * J).ravel()
        else:
            K, J, I = np.meshgrid(np.arange(nc[2] + 1), np.arange(nc[1] + 1), np.arange(nc[0] + 1), indexing="ij")
            ids = self.node_id(2 * I, 2 * J, 2 * K).ravel()
        return Mesh(nc, self.coords[ids])

    def child_cells(self):
        """For each coarse cell (of self.coarsen()), the ids of its 2^dim children."""
        nc = [v // 2 for v in self.n]
        if self.dim == 2:
            J, I = np.meshgrid(np.arange(nc[1]), np.arange(nc[0]), indexing="ij")
            I = I.ravel(); J = J.ravel()
            out = [(2 * I + a) + self.n[0] * (2 * J + b) for b in range(2) for a in range(2)]
        else:
            K, J, I = np.meshgrid(np.arange(nc[2]), np.arange(nc[1]), np.arange(nc[0]), indexing="ij")
            I = I.ravel(); J = J.ravel(); K = K.ravel()
            out = [(2 * I + a) + self.n[0] * ((2 * J + b) + self.n[1] * (2 * K + c))
                   for c in range(2) for b in range(2) for a in range(2)]
        return np.stack(out, axis=1)


def unit_mesh(n):
    """Uniform mesh of (0,1)^dim with n cells per direction."""
    axes = [np.linspace(0.0, 1.0, v + 1) for v in n]
    if len(n) == 2:
        Y, X = np.meshgrid(axes[1], axes[0], indexing="ij")
        coords = np.stack([X.ravel(), Y.ravel()], axis=1)
    else:
        Z, Y, X = np.meshgrid(axes[2], axes[1], axes[0], indexing="ij")
        coords = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
    return Mesh(n, coords)


def jittered_mesh(n, jitter_uniform):
    """Uniform mesh whose *interior* nodes are moved by jitter_uniform * h_axis.

    ``jitter_uniform`` has shape (n_nodes, dim) with entries in [-a, a]
    (BASELINE config 5: a = 0.2); boundary nodes keep their position so the
    domain stays (0,1)^dim."""
    m = unit_mesh(n)
    X = m.coords.copy()
    h = np.array([1.0 / v for v in n])
    inner = np.all((X > 1e-12) & (X < 1 - 1e-12), axis=1)
    X[inner] += jitter_uniform[inner] * h
    return Mesh(n, X)
