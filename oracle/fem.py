"""Lowest-order Nedelec (edge) FE operators on hex/quad meshes - oracle.

Definitions followed (§3, l.126-128):
    (M_h)_{ij} = \\int sigma phi_i . phi_j dx,   (K_h)_{ij} = \\int mu^{-1} curl phi_i . curl phi_j dx
and §3.3 (l.181): G the discrete gradient from the nodal H^1 space into the
Nedelec space, K_n the nodal stiffness matrix of div(sigma grad).

Reference element: the unit cube/square; edge basis of the first-kind
lowest-order Nedelec space (x-edge (b,c): l_b(y) l_c(z) e_x, l_0 = 1-t,
l_1 = t), mapped by the covariant Piola transform of the trilinear (bilinear)
geometry map.  All integrals use the tensor Gauss-Legendre rule with 3 points
per direction (reading R5): exact on affine cells, a fixed
quadrature on the jittered cells of config 5.  Coefficients sigma, nu (= mu^{-1})
are piecewise constant per cell.

Natural (homogeneous Neumann) boundary conditions: no dof is eliminated
("The problem features homogeneous Neumann boundary conditions";
the config edge counts, e.g. 300 for 4x4x4, count every edge).
"""
import numpy as np
import scipy.sparse as sp

_GP = np.array([-np.sqrt(0.6), 0.0, np.sqrt(0.6)]) * 0.5 + 0.5
_GW = np.array([5.0, 8.0, 5.0]) / 18.0


def _l(t, s):
    return 1.0 - t if s == 0 else t


def _dl(s):
    return -1.0 if s == 0 else 1.0


def quad_points(dim):
    if dim == 2:
        pts = [(x, y) for y in _GP for x in _GP]
        w = [wx * wy for wy in _GW for wx in _GW]
    else:
        pts = [(x, y, z) for z in _GP for y in _GP for x in _GP]
        w = [wx * wy * wz for wz in _GW for wy in _GW for wx in _GW]
    return np.array(pts), np.array(w)


def ref_edge_basis(dim, p):
    """Values (n_loc, dim) and reference curls (n_loc, 3 or scalar) at point p."""
    if dim == 2:
        x, y = p
        N = np.zeros((4, 2)); C = np.zeros(4)
        for b in range(2):
            N[b, 0] = _l(y, b)
            C[b] = -_dl(b)                 # curl = d_x N_y - d_y N_x
        for a in range(2):
            N[2 + a, 1] = _l(x, a)
            C[2 + a] = _dl(a)
        return N, C
    x, y, z = p
    N = np.zeros((12, 3)); C = np.zeros((12, 3))
    for c in range(2):
        for b in range(2):
            e = b + 2 * c
            N[e, 0] = _l(y, b) * _l(z, c)
            C[e] = [0.0, _l(y, b) * _dl(c), -_dl(b) * _l(z, c)]
    for c in range(2):
        for a in range(2):
            e = 4 + a + 2 * c
            N[e, 1] = _l(x, a) * _l(z, c)
            C[e] = [-_l(x, a) * _dl(c), 0.0, _dl(a) * _l(z, c)]
    for b in range(2):
        for a in range(2):
            e = 8 + a + 2 * b
            N[e, 2] = _l(x, a) * _l(y, b)
            C[e] = [_l(x, a) * _dl(b), -_dl(a) * _l(y, b), 0.0]
    return N, C


def ref_node_basis(dim, p):
    """Q1 nodal values (n_loc,) and reference gradients (n_loc, dim)."""
    nloc = 2 ** dim
    V = np.ones(nloc); D = np.ones((nloc, dim))
    for n in range(nloc):
        off = [(n >> d) & 1 for d in range(dim)]
        for d in range(dim):
            V[n] *= _l(p[d], off[d])
            for e in range(dim):
                D[n, e] *= (_dl(off[d]) if d == e else _l(p[d], off[d]))
    return V, D


def _jacobians(mesh, p):
    """J (n_cells, dim, dim) with J[r, c] = d x_r / d xhat_c, at ref point p."""
    _, D = ref_node_basis(mesh.dim, p)
    X = mesh.coords[mesh.cell_nodes]            # (cells, nloc, dim)
    return np.einsum("cnr,nk->crk", X, D)


def element_matrices(mesh, sigma, nu):
    """Per-cell edge mass Me, curl-curl Ke (n_cells, nloc_e, nloc_e) and nodal
    stiffness Kne (n_cells, nloc_n, nloc_n) of div(sigma grad)."""
    dim = mesh.dim
    pts, wts = quad_points(dim)
    ne = 4 if dim == 2 else 12
    nn = 2 ** dim
    Me = np.zeros((mesh.n_cells, ne, ne))
    Ke = np.zeros((mesh.n_cells, ne, ne))
    Kne = np.zeros((mesh.n_cells, nn, nn))
    for p, w in zip(pts, wts):
        J = _jacobians(mesh, p)
        detJ = np.linalg.det(J)
        assert np.all(detJ > 0), "degenerate or inverted cell"
        JtJ = np.einsum("crk,crl->ckl", J, J)
        JtJinv = np.linalg.inv(JtJ)
        N, C = ref_edge_basis(dim, p)
        _, Dn = ref_node_basis(dim, p)
        # covariant Piola: phi = J^{-T} Nhat  ->  phi_i.phi_j = Nhat_i^T (J^T J)^{-1} Nhat_j
        Me += (w * sigma * detJ)[:, None, None] * np.einsum("ik,ckl,jl->cij", N, JtJinv, N)
        if dim == 3:
            # curl phi = J curlhat / detJ -> curl_i.curl_j = c_i^T (J^T J) c_j / detJ^2
            Ke += (w * nu / detJ)[:, None, None] * np.einsum("ik,ckl,jl->cij", C, JtJ, C)
        else:
            Ke += (w * nu / detJ)[:, None, None] * np.outer(C, C)[None]
        Kne += (w * sigma * detJ)[:, None, None] * np.einsum("ik,ckl,jl->cij", Dn, JtJinv, Dn)
    return Me, Ke, Kne


def _assemble(dofs, Ae, n):
    nloc = dofs.shape[1]
    rows = np.repeat(dofs, nloc, axis=1).ravel()
    cols = np.tile(dofs, (1, nloc)).ravel()
    return sp.csr_matrix((Ae.ravel(), (rows, cols)), shape=(n, n))


def assemble(mesh, sigma, nu):
    """Global M_sigma, K_nu (edges x edges) and K_n (nodes x nodes), CSR."""
    Me, Ke, Kne = element_matrices(mesh, np.asarray(sigma, float), np.asarray(nu, float))
    M = _assemble(mesh.cell_edges, Me, mesh.n_edges)
    K = _assemble(mesh.cell_edges, Ke, mesh.n_edges)
    Kn = _assemble(mesh.cell_nodes, Kne, mesh.n_nodes)
    return M, K, Kn


def gradient(mesh):
    """Discrete gradient G (edges x nodes): row of edge (s -> e) is -1 at s, +1 at e
    (DOF of grad(phi_n) on an edge = phi_n(end) - phi_n(start))."""
    en = mesh.edge_nodes
    ne = mesh.n_edges
    rows = np.concatenate([np.arange(ne), np.arange(ne)])
    cols = np.concatenate([en[:, 0], en[:, 1]])
    vals = np.concatenate([-np.ones(ne), np.ones(ne)])
    return sp.csr_matrix((vals, (rows, cols)), shape=(ne, mesh.n_nodes))


def _axis_weights(f):
    """Fine index f along a transverse axis -> [(coarse index, weight)] of the
    coarse Q1 hat functions at the fine node position."""
    if f % 2 == 0:
        return [(f // 2, 1.0)]
    return [((f - 1) // 2, 0.5), ((f + 1) // 2, 0.5)]


def edge_prolongation(fine, coarse):
    """P_edge (fine edges x coarse edges): canonical Nedelec interpolation of
    the coarse edge basis on the fine edges of a uniform 2:1 refinement.

    A fine edge collinear with coarse edge c has DOF 1/2 (half the line
    integral); a fine edge on a coarse face/cell midline gets 1/2 times the
    transverse Q1 hat weights.  Weights are topological (used unchanged on
    jittered meshes, reading R6)."""
    rows, cols, vals = [], [], []
    dim = fine.dim
    nf = fine.n
    nc = coarse.n

    def eid(m, d, ijk):
        if dim == 2:
            i, j = ijk
            if d == 0:
                return i + m.n[0] * j
            return m.Ex + i + (m.n[0] + 1) * j
        i, j, k = ijk
        nx, ny = m.n[0], m.n[1]
        if d == 0:
            return i + nx * (j + (ny + 1) * k)
        if d == 1:
            return m.Ex + i + (nx + 1) * (j + ny * k)
        return m.Ex + m.Ey + i + (nx + 1) * (j + (ny + 1) * k)

    import itertools
    for d in range(dim):
        ranges = [range(nf[a] if a == d else nf[a] + 1) for a in range(dim)]
        for ijk in itertools.product(*ranges):
            ef = eid(fine, d, ijk)
            trans = [a for a in range(dim) if a != d]
            lists = [_axis_weights(ijk[a]) for a in trans]
            for combo in itertools.product(*lists):
                cidx = list(ijk)
                cidx[d] = ijk[d] // 2
                w = 0.5
                for a, (ci, wa) in zip(trans, combo):
                    cidx[a] = ci
                    w *= wa
                rows.append(ef); cols.append(eid(coarse, d, tuple(cidx))); vals.append(w)
    assert all(c == f // 2 for c, f in zip(nc, nf))
    return sp.csr_matrix((vals, (rows, cols)), shape=(fine.n_edges, coarse.n_edges))


def node_prolongation(fine, coarse):
    """P_node: Q1 interpolation (used only to pin the commuting diagram)."""
    import itertools
    rows, cols, vals = [], [], []
    dim = fine.dim
    for ijk in itertools.product(*[range(v + 1) for v in fine.n]):
        lists = [_axis_weights(f) for f in ijk]
        for combo in itertools.product(*lists):
            w = np.prod([c[1] for c in combo])
            cid = coarse.node_id(*[c[0] for c in combo])
            rows.append(fine.node_id(*ijk)); cols.append(cid); vals.append(w)
    return sp.csr_matrix((vals, (rows, cols)), shape=(fine.n_nodes, coarse.n_nodes))
