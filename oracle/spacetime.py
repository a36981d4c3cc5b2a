"""Space-time operator, block-Jacobi smoother S and nodal correction A - oracle.

Space-time vectors are numpy arrays X of shape (S, q+1, n): slab k, time node
a, spatial dof.  (The C-ABI layout [dof][a][slab] is a transpose of this; the
tests convert.)

PAPER.md references
  L_{tau,h}          l.51-77   (block lower-bidiagonal space-time system)
  smoother S, Eq.(2) l.79-82   x <- x + omega (I (x) A^{-1}) (f - L x), omega = 1/2
  correction A, Eq.(5) l.181-188   x <- x + G Sigma_t K_n^{-1} G^T (f - L x)
  hybrid SAS         l.207-208   read right to left; post-smoothing reversed

Inner spatial solves ("sufficiently well approximated", l.84):
  mode 'exact'   : A_k^{-1}, K_n^{-1} by sparse direct factorisation (LFA assumption, l.212)
  mode 'mg'      : A_k^{-1} by one geometric V-cycle over the level's spatial chain with a
                   hybrid edge / nodal smoother (R13; the role AMS plays in l.269)
  mode 'jacobi'  : the GPU hot path's fixed linear approximations (R3/R4):
                   nu_s damped block-Jacobi sweeps on A_k (one (q+1)x(q+1) block per edge),
                   nu_n damped Jacobi sweeps on K_n, both started from zero
                   (plain diagonals; sweep z <- z + w D^{-1}(r - A z)).
"""
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import time_dg


class Level:
    """One rung of the hierarchy: mesh, spatial operators, slab lengths tau_k."""

    def __init__(self, mesh, sigma, nu, tau, q, M=None, K=None, Kn=None):
        from . import fem
        self.mesh = mesh
        self.sigma = np.asarray(sigma, float)
        self.nu = np.asarray(nu, float)
        self.tau = np.asarray(tau, float)
        self.q = q
        self.S = len(self.tau)
        if M is None:
            M, K, Kn = fem.assemble(mesh, self.sigma, self.nu)
        self.M, self.K, self.Kn = M.tocsr(), K.tocsr(), Kn.tocsr()
        self.G = fem.gradient(mesh)
        self.n = mesh.n_edges
        self.nn = mesh.n_nodes
        self.Ct, self.Mt, self.Nt = time_dg.time_matrices(q)
        self._Ainv = {}
        self._Kn_lu = None

    # -- spatial operators applied to all (slab, time-node) blocks -------------
    def spatial(self, A, X):
        """Apply spatial matrix A to every block of X (S, q+1, n_in)."""
        S, Q, n = X.shape
        Y = A @ X.reshape(S * Q, n).T
        return Y.T.reshape(S, Q, A.shape[0])

    def A_k(self, k):
        """A_k = Ct (x) M + tau_k Mt (x) K, ordering [time node a][edge]."""
        return (sp.kron(self.Ct, self.M) + self.tau[k] * sp.kron(self.Mt, self.K)).tocsc()

    def Ainv_exact(self, k):
        key = float(self.tau[k])
        if key not in self._Ainv:
            self._Ainv[key] = spla.splu(self.A_k(k))
        return self._Ainv[key]


def apply_L(lv, X, prev=None):
    """(L X)_k = sum_a (Ct M + tau_k Mt K) X_{k,a} - sum_a Nt M X_{k-1,a}  (l.51-77).

    ``prev`` is the (q+1, n) block of slab k = -1 (None: zero initial state)."""
    MX = lv.spatial(lv.M, X)
    KX = lv.spatial(lv.K, X)
    Y = np.einsum("ba,kan->kbn", lv.Ct, MX) + lv.tau[:, None, None] * np.einsum("ba,kan->kbn", lv.Mt, KX)
    Y[1:] -= np.einsum("ba,kan->kbn", lv.Nt, MX[:-1])
    if prev is not None:
        Y[0] -= lv.Nt @ (lv.M @ prev.T).T
    return Y


def residual(lv, X, F):
    return F - apply_L(lv, X)


def inv_blocks(D):
    """Inverse of every (Q x Q) block of D (shape (..., Q, Q)) in D's precision.  float64 uses
    LAPACK (np.linalg.inv); other dtypes (np.longdouble for the extended-precision reference of
    the c3 tolerance, R12) Gauss-Jordan elimination with partial pivoting."""
    if D.dtype == np.float64:
        return np.linalg.inv(D)
    A = np.array(D, copy=True)
    Q = A.shape[-1]
    B = np.broadcast_to(np.eye(Q, dtype=A.dtype), A.shape).copy()
    for c in range(Q):
        piv = np.argmax(np.abs(A[..., c:, c]), axis=-1) + c
        idx = np.indices(piv.shape)
        rows_c = A[..., c, :].copy(); rows_p = A[(*idx, piv)].copy()
        A[..., c, :] = rows_p; A[(*idx, piv)] = rows_c
        rows_c = B[..., c, :].copy(); rows_p = B[(*idx, piv)].copy()
        B[..., c, :] = rows_p; B[(*idx, piv)] = rows_c
        p = A[..., c, c][..., None].copy()
        A[..., c, :] /= p; B[..., c, :] /= p
        for r in range(Q):
            if r != c:
                fct = A[..., r, c][..., None].copy()
                A[..., r, :] -= fct * A[..., c, :]
                B[..., r, :] -= fct * B[..., c, :]
    return B


def dense_solve(A, b):
    """x = A^{-1} b by Gaussian elimination with partial pivoting in A's precision (used for the
    extended-precision coarsest forward substitution)."""
    A = np.array(A, copy=True); b = np.array(b, copy=True)
    n = A.shape[0]
    for c in range(n):
        p = c + int(np.argmax(np.abs(A[c:, c])))
        if p != c:
            A[[c, p]] = A[[p, c]]; b[[c, p]] = b[[p, c]]
        f = A[c + 1:, c] / A[c, c]
        A[c + 1:, c:] -= np.outer(f, A[c, c:])
        b[c + 1:] -= f * b[c]
    x = np.zeros_like(b)
    for c in range(n - 1, -1, -1):
        x[c] = (b[c] - A[c, c + 1:] @ x[c + 1:]) / A[c, c]
    return x


def block_jacobi_inverse(lv, k, R, nu_s, omega_s):
    """nu_s damped block-Jacobi sweeps on A_k z = R_k from z = 0.

    The Jacobi block of edge e is the (q+1)x(q+1) matrix
    D_e = Ct M_ee + tau_k Mt K_ee (all time nodes of one edge)."""
    Q = lv.q + 1
    dt = R.dtype                    # float64, or np.longdouble for the extended-precision reference
    dM = lv.M.diagonal().astype(dt); dK = lv.K.diagonal().astype(dt)
    D = lv.Ct.astype(dt)[None] * dM[:, None, None] + dt.type(lv.tau[k]) * lv.Mt.astype(dt)[None] * dK[:, None, None]   # (n, Q, Q)
    Dinv = inv_blocks(D)
    z = np.zeros((Q, lv.n), dtype=dt)
    for _ in range(nu_s):
        Az = lv.Ct @ (lv.M @ z.T).T + lv.tau[k] * (lv.Mt @ (lv.K @ z.T).T)
        d = R - Az
        z = z + omega_s * np.einsum("eab,be->ae", Dinv, d)
    return z


class SpatialChain:
    """Spatial hierarchy of one level's mesh for the inner V-cycle (reading R13): the mesh and
    its successive 2:1 coarsenings (coefficients averaged as for the outer hierarchy, R6)."""

    def __init__(self, mesh, sigma, nu, q):
        from . import fem
        self.Ct, self.Mt, _ = time_dg.time_matrices(q)
        self.Ctinv = np.linalg.inv(self.Ct)
        self.lv = []
        while True:
            M, K, Kn = fem.assemble(mesh, sigma, nu)
            G = fem.gradient(mesh).tocsr()
            d = dict(M=M.tocsr(), K=K.tocsr(), G=G, GT=G.T.tocsr(), dM=M.diagonal(), dK=K.diagonal(),
                     dN=Kn.diagonal(), n=mesh.n_edges, P=None)
            self.lv.append(d)
            if not mesh.can_coarsen():
                break
            mc = mesh.coarsen()
            ch = mesh.child_cells()
            d["P"] = fem.edge_prolongation(mesh, mc).tocsr()
            sigma, nu, mesh = sigma[ch].mean(axis=1), nu[ch].mean(axis=1), mc

    def A(self, j, tau, z):
        L = self.lv[j]
        return self.Ct @ (L["M"] @ z.T).T + tau * (self.Mt @ (L["K"] @ z.T).T)

    def edge_sweep(self, j, tau, r, z, om):
        """z + om D^{-1} (r - A z), D_e = Ct M_ee + tau Mt K_ee (R3)."""
        L = self.lv[j]
        D = self.Ct[None] * L["dM"][:, None, None] + tau * self.Mt[None] * L["dK"][:, None, None]
        return z + om * np.einsum("eab,be->ae", np.linalg.inv(D), r - self.A(j, tau, z))

    def nodal_step(self, j, tau, r, z, om):
        """Hiptmair's nodal step on the gradient space: G^T A G = Ct (x) K_n (K G = 0), one
        damped Jacobi sweep on it: z + G (om Ct^{-1} G^T (r - A z) / d_n)."""
        L = self.lv[j]
        w = (L["GT"] @ (r - self.A(j, tau, z)).T).T
        y = om * (self.Ctinv @ w) / L["dN"][None, :]
        return z + (L["G"] @ y.T).T

    def vcycle(self, j, tau, r, opts):
        """One V-cycle for A z = r (Q, n_j) from z = 0: nu_in hybrid sweeps (edge then nodal)
        before, P^T / P to the next chain level, nu_in sweeps (nodal then edge) after; the
        coarsest chain level only smooths."""
        z = np.zeros_like(r)
        for _ in range(opts.nu_in):
            z = self.edge_sweep(j, tau, r, z, opts.omega_in)
            z = self.nodal_step(j, tau, r, z, opts.omega_n)
        P = self.lv[j]["P"]
        if P is None:
            return z
        rc = (P.T @ (r - self.A(j, tau, z)).T).T
        z = z + (P @ self.vcycle(j + 1, tau, rc, opts).T).T
        for _ in range(opts.nu_in):
            z = self.nodal_step(j, tau, r, z, opts.omega_n)
            z = self.edge_sweep(j, tau, r, z, opts.omega_in)
        return z


def apply_B(lv, R, opts):
    """(I (x) A^{-1}) R with the configured inner approximation, slab by slab."""
    Z = np.zeros_like(R)
    if opts.inner == "mg" and getattr(lv, "chain", None) is None:
        lv.chain = SpatialChain(lv.mesh, lv.sigma, lv.nu, lv.q)
    for k in range(lv.S):
        if opts.inner == "exact":
            Z[k] = lv.Ainv_exact(k).solve(R[k].reshape(-1)).reshape(lv.q + 1, lv.n)
        elif opts.inner == "mg":
            Z[k] = lv.chain.vcycle(0, lv.tau[k], R[k], opts)
        else:
            Z[k] = block_jacobi_inverse(lv, k, R[k], opts.nu_s, opts.omega_s)
    return Z


def smoother_S(lv, X, F, opts):
    """Eq. (2): x <- x + omega (I (x) A_{tau,h}^{-1}) (f - L x)."""
    R = residual(lv, X, F)
    return X + opts.omega * apply_B(lv, R, opts)


def Kn_inverse(lv, W, opts):
    """K_n^{-1} (exact, on the complement of constants) or nu_n damped Jacobi sweeps."""
    if opts.inner == "exact":
        if lv._Kn_lu is None:
            lv._Kn_lu = spla.splu(lv.Kn[1:, 1:].tocsc())    # pin node 0 (Neumann K_n is singular)
        S, Q, nn = W.shape
        Z = np.zeros_like(W)
        rhs = W.reshape(S * Q, nn)[:, 1:].T
        Z.reshape(S * Q, nn)[:, 1:] = lv._Kn_lu.solve(np.ascontiguousarray(rhs)).T
        return Z
    d = lv.Kn.diagonal()
    Z = np.zeros_like(W)
    for _ in range(opts.nu_n):
        Z = Z + opts.omega_n * (W - lv.spatial(lv.Kn, Z)) / d
    return Z


def sigma_t(lv, Z):
    """Time integration Sigma_t (l.182-184): (Sigma_t y)_i = sum_{j<=i} y_j for
    q = 0.  For dG(q) (reading R2) it is the inverse of the time factor of
    G^T L G = L_t (x) K_n, i.e. forward substitution of the pure dG(q) ODE
    u' = z:  Y_k = Ct^{-1} (Z_k + Nt Y_{k-1})."""
    Y = np.zeros_like(Z)
    Ctinv = inv_blocks(lv.Ct.astype(Z.dtype))
    prev = np.zeros(Z.shape[1:], dtype=Z.dtype)
    for k in range(Z.shape[0]):
        Y[k] = Ctinv @ (Z[k] + lv.Nt @ prev)
        prev = Y[k]
    return Y


def correction_A(lv, X, F, opts):
    """Eq. (5): x <- x + G Sigma_t K_n^{-1} G^T (f - L x)."""
    R = residual(lv, X, F)
    W = lv.spatial(lv.G.T.tocsr(), R)
    Z = Kn_inverse(lv, W, opts)
    Y = sigma_t(lv, Z)
    return X + lv.spatial(lv.G, Y)


def hybrid_smooth(lv, X, F, opts, phase):
    """Apply opts.spec (e.g. 'SAS') read right to left (l.208: "SA is one
    application of A followed by an application of S"); the post phase uses
    the reversed string."""
    seq = opts.spec if phase == "pre" else opts.spec[::-1]
    for ch in reversed(seq):
        if ch == "S":
            X = smoother_S(lv, X, F, opts)
        elif ch == "A":
            X = correction_A(lv, X, F, opts)
        else:
            raise ValueError("smoother spec may only contain 'S' and 'A'")
    return X


def forward_solve(lv, F, prev=None):
    """Exact forward substitution in time: X_k = A_k^{-1} (F_k + Nt M X_{k-1})."""
    X = np.zeros_like(F)
    p = np.zeros((lv.q + 1, lv.n), dtype=F.dtype) if prev is None else prev
    for k in range(lv.S):
        rhs = F[k] + lv.Nt @ (lv.M @ p.T).T
        if F.dtype == np.float64:
            X[k] = lv.Ainv_exact(k).solve(rhs.reshape(-1)).reshape(lv.q + 1, lv.n)
        else:       # extended-precision reference: dense elimination in F's precision
            A = lv.A_k(k).toarray().astype(F.dtype)
            X[k] = dense_solve(A, rhs.reshape(-1)).reshape(lv.q + 1, lv.n)
        p = X[k]
    return X
