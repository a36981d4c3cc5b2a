// setup.cpp — host-side construction of the space-time level hierarchy.
//
// Everything here runs once in st_setup: mesh enumeration, lowest-order
// Nedelec element matrices (§3 l.126-128: M_h = int sigma phi.phi,
// K_h = int mu^{-1} curl phi . curl phi), the nodal stiffness of div(sigma grad)
// and the discrete gradient (§3.3 l.181), the coarsening rule Eq. (3)
// (l.105-109), spatial/time transfer operators and the dense coarsest inverse.
// Independent implementation (no code shared with oracle/); readings R1-R9 of
// DESIGN.md §0(c).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "internal.h"

namespace st {

// ---------------------------------------------------------------- small dense
static void invert(int n, const double *A, double *Ainv) {
    // Gauss-Jordan with partial pivoting, row-major
    std::vector<double> a(A, A + (size_t)n * n), b((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) b[(size_t)i * n + i] = 1.0;
    for (int c = 0; c < n; ++c) {
        int piv = c;
        for (int r = c + 1; r < n; ++r)
            if (std::fabs(a[(size_t)r * n + c]) > std::fabs(a[(size_t)piv * n + c])) piv = r;
        if (a[(size_t)piv * n + c] == 0.0) throw std::runtime_error("singular matrix in setup");
        if (piv != c)
            for (int j = 0; j < n; ++j) {
                std::swap(a[(size_t)c * n + j], a[(size_t)piv * n + j]);
                std::swap(b[(size_t)c * n + j], b[(size_t)piv * n + j]);
            }
        const double inv = 1.0 / a[(size_t)c * n + c];
        for (int j = 0; j < n; ++j) { a[(size_t)c * n + j] *= inv; b[(size_t)c * n + j] *= inv; }
        for (int r = 0; r < n; ++r) {
            if (r == c) continue;
            const double fct = a[(size_t)r * n + c];
            if (fct == 0.0) continue;
            for (int j = 0; j < n; ++j) {
                a[(size_t)r * n + j] -= fct * a[(size_t)c * n + j];
                b[(size_t)r * n + j] -= fct * b[(size_t)c * n + j];
            }
        }
    }
    std::memcpy(Ainv, b.data(), sizeof(double) * (size_t)n * n);
}

static void gauss_legendre(int n, std::vector<double> &x, std::vector<double> &w) {
    // nodes/weights on [0,1] by Newton iteration on P_n
    x.assign(n, 0.0); w.assign(n, 0.0);
    for (int i = 0; i < n; ++i) {
        double t = std::cos(M_PI * (i + 0.75) / (n + 0.5));
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = t;
            for (int k = 2; k <= n; ++k) { double p2 = ((2 * k - 1) * t * p1 - (k - 1) * p0) / k; p0 = p1; p1 = p2; }
            double dp = n * (t * p1 - p0) / (t * t - 1.0);
            double dt = p1 / dp;
            t -= dt;
            if (std::fabs(dt) < 1e-16) break;
        }
        double p0 = 1.0, p1 = t;
        for (int k = 2; k <= n; ++k) { double p2 = ((2 * k - 1) * t * p1 - (k - 1) * p0) / k; p0 = p1; p1 = p2; }
        double dp = n * (t * p1 - p0) / (t * t - 1.0);
        x[i] = 0.5 * (1.0 - t);
        w[i] = 1.0 / ((1.0 - t * t) * dp * dp);   // (2/((1-t^2)P'^2)) * 1/2
    }
}

// ------------------------------------------------------------ dG(q) in time
static double lag(int q, int a, double s) {
    if (q == 0) return 1.0;
    double v = 1.0;
    for (int m = 0; m <= q; ++m)
        if (m != a) v *= (s - (double)m / q) / ((double)(a - m) / q);
    return v;
}
static double dlag(int q, int a, double s) {
    if (q == 0) return 0.0;
    double tot = 0.0;
    for (int skip = 0; skip <= q; ++skip) {
        if (skip == a) continue;
        double term = 1.0 / ((double)(a - skip) / q);
        for (int m = 0; m <= q; ++m)
            if (m != a && m != skip) term *= (s - (double)m / q) / ((double)(a - m) / q);
        tot += term;
    }
    return tot;
}

TimeMats time_matrices(int q) {
    if (q < 0 || q > kMaxQ - 1) throw std::invalid_argument("q must be 0, 1 or 2");
    TimeMats tm{};
    const int Q = q + 1;
    tm.Q = Q;
    std::vector<double> gx, gw;
    gauss_legendre(q + 2, gx, gw);
    for (int b = 0; b < Q; ++b)
        for (int a = 0; a < Q; ++a) {
            double m = 0, c = 0;
            for (size_t i = 0; i < gx.size(); ++i) {
                m += gw[i] * lag(q, a, gx[i]) * lag(q, b, gx[i]);
                c += gw[i] * dlag(q, a, gx[i]) * lag(q, b, gx[i]);
            }
            tm.Mt[b * Q + a] = m;
            tm.Ct[b * Q + a] = c + lag(q, a, 0.0) * lag(q, b, 0.0);   // upwind jump term
            tm.Nt[b * Q + a] = lag(q, b, 0.0) * lag(q, a, 1.0);      // trace of the previous slab
        }
    invert(Q, tm.Ct, tm.Ctinv);
    for (int a = 0; a < Q; ++a) tm.g[a] = tm.Ctinv[a * Q + 0];
    // the kernels rely on the nodal structure Nt = e_0 e_q^T and (Ct^{-1} e_0)_q = 1 (R2)
    for (int b = 0; b < Q; ++b)
        for (int a = 0; a < Q; ++a) {
            double want = (b == 0 && a == q) ? 1.0 : 0.0;
            if (std::fabs(tm.Nt[b * Q + a] - want) > 1e-14) throw std::runtime_error("unexpected Nt structure");
        }
    if (std::fabs(tm.g[q] - 1.0) > 1e-12) throw std::runtime_error("unexpected Ct^{-1} e0");
    return tm;
}

// -------------------------------------------------------------------- mesh
HostMesh make_mesh(int dim, const int n[3], const double *coords) {
    HostMesh m;
    m.dim = dim;
    const int nx = n[0], ny = n[1], nz = dim == 3 ? n[2] : 1;
    m.n[0] = nx; m.n[1] = ny; m.n[2] = dim == 3 ? nz : 1;
    auto nid = [&](int i, int j, int k) { return i + (nx + 1) * (j + (ny + 1) * k); };
    if (dim == 2) {
        m.n_nodes = (nx + 1) * (ny + 1);
        m.Ex = nx * (ny + 1); m.Ey = (nx + 1) * ny;
        m.n_edges = m.Ex + m.Ey;
        m.n_cells = nx * ny;
    } else {
        m.n_nodes = (nx + 1) * (ny + 1) * (nz + 1);
        m.Ex = nx * (ny + 1) * (nz + 1); m.Ey = (nx + 1) * ny * (nz + 1);
        m.n_edges = m.Ex + m.Ey + (nx + 1) * (ny + 1) * nz;
        m.n_cells = nx * ny * nz;
    }
    m.coords.resize((size_t)m.n_nodes * dim);
    if (coords) {
        std::memcpy(m.coords.data(), coords, sizeof(double) * m.coords.size());
    } else {
        const int kmax = dim == 3 ? nz : 0;
        for (int k = 0; k <= kmax; ++k)
            for (int j = 0; j <= ny; ++j)
                for (int i = 0; i <= nx; ++i) {
                    double *X = &m.coords[(size_t)nid(i, j, k) * dim];
                    X[0] = (double)i / nx; X[1] = (double)j / ny;
                    if (dim == 3) X[2] = (double)k / nz;
                }
    }
    m.edge_nodes.resize((size_t)2 * m.n_edges);
    const int kk = dim == 3 ? nz : 0;
    // x-edges
    for (int k = 0; k <= kk; ++k)
        for (int j = 0; j <= ny; ++j)
            for (int i = 0; i < nx; ++i) {
                int e = i + nx * (j + (ny + 1) * k);
                m.edge_nodes[2 * e] = nid(i, j, k); m.edge_nodes[2 * e + 1] = nid(i + 1, j, k);
            }
    for (int k = 0; k <= kk; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i <= nx; ++i) {
                int e = m.Ex + i + (nx + 1) * (j + ny * k);
                m.edge_nodes[2 * e] = nid(i, j, k); m.edge_nodes[2 * e + 1] = nid(i, j + 1, k);
            }
    if (dim == 3)
        for (int k = 0; k < nz; ++k)
            for (int j = 0; j <= ny; ++j)
                for (int i = 0; i <= nx; ++i) {
                    int e = m.Ex + m.Ey + i + (nx + 1) * (j + (ny + 1) * k);
                    m.edge_nodes[2 * e] = nid(i, j, k); m.edge_nodes[2 * e + 1] = nid(i, j, k + 1);
                }
    const int ne = dim == 3 ? 12 : 4, nn = dim == 3 ? 8 : 4;
    m.cell_edges.resize((size_t)ne * m.n_cells);
    m.cell_nodes.resize((size_t)nn * m.n_cells);
    for (int k = 0; k < (dim == 3 ? nz : 1); ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                const int c = i + nx * (j + ny * k);
                int *E = &m.cell_edges[(size_t)ne * c];
                int *N = &m.cell_nodes[(size_t)nn * c];
                if (dim == 2) {
                    for (int b = 0; b < 2; ++b) E[b] = i + nx * (j + b);
                    for (int a = 0; a < 2; ++a) E[2 + a] = m.Ex + (i + a) + (nx + 1) * j;
                    for (int b = 0; b < 2; ++b)
                        for (int a = 0; a < 2; ++a) N[a + 2 * b] = nid(i + a, j + b, 0);
                } else {
                    for (int c2 = 0; c2 < 2; ++c2)
                        for (int b = 0; b < 2; ++b) E[b + 2 * c2] = i + nx * ((j + b) + (ny + 1) * (k + c2));
                    for (int c2 = 0; c2 < 2; ++c2)
                        for (int a = 0; a < 2; ++a) E[4 + a + 2 * c2] = m.Ex + (i + a) + (nx + 1) * (j + ny * (k + c2));
                    for (int b = 0; b < 2; ++b)
                        for (int a = 0; a < 2; ++a)
                            E[8 + a + 2 * b] = m.Ex + m.Ey + (i + a) + (nx + 1) * ((j + b) + (ny + 1) * k);
                    for (int c2 = 0; c2 < 2; ++c2)
                        for (int b = 0; b < 2; ++b)
                            for (int a = 0; a < 2; ++a) N[a + 2 * b + 4 * c2] = nid(i + a, j + b, k + c2);
                }
            }
    return m;
}

// ------------------------------------------------------- element integrals
static inline double l01(int s, double t) { return s ? t : 1.0 - t; }
static inline double d01(int s) { return s ? 1.0 : -1.0; }

// Reference Nedelec basis (values N[e][3], curls C[e][3]; 2D: C[e][0] = scalar curl)
static void edge_basis(int dim, const double *p, double N[12][3], double C[12][3]) {
    std::memset(N, 0, sizeof(double) * 36);
    std::memset(C, 0, sizeof(double) * 36);
    if (dim == 2) {
        const double x = p[0], y = p[1];
        for (int b = 0; b < 2; ++b) { N[b][0] = l01(b, y); C[b][0] = -d01(b); }
        for (int a = 0; a < 2; ++a) { N[2 + a][1] = l01(a, x); C[2 + a][0] = d01(a); }
        return;
    }
    const double x = p[0], y = p[1], z = p[2];
    for (int c = 0; c < 2; ++c)
        for (int b = 0; b < 2; ++b) {
            int e = b + 2 * c;
            N[e][0] = l01(b, y) * l01(c, z);
            C[e][1] = l01(b, y) * d01(c);
            C[e][2] = -d01(b) * l01(c, z);
        }
    for (int c = 0; c < 2; ++c)
        for (int a = 0; a < 2; ++a) {
            int e = 4 + a + 2 * c;
            N[e][1] = l01(a, x) * l01(c, z);
            C[e][0] = -l01(a, x) * d01(c);
            C[e][2] = d01(a) * l01(c, z);
        }
    for (int b = 0; b < 2; ++b)
        for (int a = 0; a < 2; ++a) {
            int e = 8 + a + 2 * b;
            N[e][2] = l01(a, x) * l01(b, y);
            C[e][0] = l01(a, x) * d01(b);
            C[e][1] = -d01(a) * l01(b, y);
        }
}

static void node_grads(int dim, const double *p, double D[8][3]) {
    const int nl = 1 << dim;
    for (int n = 0; n < nl; ++n)
        for (int e = 0; e < dim; ++e) {
            double v = 1.0;
            for (int d = 0; d < dim; ++d) {
                int o = (n >> d) & 1;
                v *= (d == e) ? d01(o) : l01(o, p[d]);
            }
            D[n][e] = v;
        }
}

// 2x2 / 3x3 inverse by cofactors (exact zeros stay exact on axis-aligned cells)
static double inv_small(int d, const double *A, double *B) {
    if (d == 2) {
        double det = A[0] * A[3] - A[1] * A[2];
        B[0] = A[3] / det; B[1] = -A[1] / det; B[2] = -A[2] / det; B[3] = A[0] / det;
        return det;
    }
    double c00 = A[4] * A[8] - A[5] * A[7], c01 = A[5] * A[6] - A[3] * A[8], c02 = A[3] * A[7] - A[4] * A[6];
    double det = A[0] * c00 + A[1] * c01 + A[2] * c02;
    B[0] = c00 / det; B[3] = c01 / det; B[6] = c02 / det;
    B[1] = (A[2] * A[7] - A[1] * A[8]) / det; B[4] = (A[0] * A[8] - A[2] * A[6]) / det; B[7] = (A[1] * A[6] - A[0] * A[7]) / det;
    B[2] = (A[1] * A[5] - A[2] * A[4]) / det; B[5] = (A[2] * A[3] - A[0] * A[5]) / det; B[8] = (A[0] * A[4] - A[1] * A[3]) / det;
    return det;
}

// Element matrices of cell c: Me, Ke (ne x ne), Kne (nn x nn); 3-point Gauss per direction (R5)
static void element(const HostMesh &m, int c, double sigma, double nu, double *Me, double *Ke, double *Kne) {
    const int d = m.dim, ne = d == 3 ? 12 : 4, nn = 1 << d;
    static const double gp[3] = {0.5 - 0.5 * std::sqrt(0.6), 0.5, 0.5 + 0.5 * std::sqrt(0.6)};
    static const double gw[3] = {5.0 / 18.0, 8.0 / 18.0, 5.0 / 18.0};
    std::fill(Me, Me + ne * ne, 0.0);
    std::fill(Ke, Ke + ne * ne, 0.0);
    std::fill(Kne, Kne + nn * nn, 0.0);
    const int nq = d == 3 ? 27 : 9;
    for (int iq = 0; iq < nq; ++iq) {
        int ix = iq % 3, iy = (iq / 3) % 3, iz = iq / 9;
        double p[3] = {gp[ix], gp[iy], gp[iz]};
        double w = gw[ix] * gw[iy] * (d == 3 ? gw[iz] : 1.0);
        double D[8][3];
        node_grads(d, p, D);
        // J[r*d + k] = dx_r / dxhat_k, summed over the cell's edges in direction k from
        // coordinate differences (exact zeros on axis-aligned cells, so no spurious
        // ~1e-20 couplings survive in M for uniform meshes)
        double J[9] = {0};
        for (int n = 0; n < nn; ++n)
            for (int k = 0; k < d; ++k) {
                if ((n >> k) & 1) continue;
                const int n1 = n | (1 << k);
                double w = 1.0;                  // transverse Q1 weights of this edge at p
                for (int a = 0; a < d; ++a)
                    if (a != k) w *= l01((n >> a) & 1, p[a]);
                const double *X0 = &m.coords[(size_t)m.cell_nodes[(size_t)nn * c + n] * d];
                const double *X1 = &m.coords[(size_t)m.cell_nodes[(size_t)nn * c + n1] * d];
                for (int r = 0; r < d; ++r) J[r * d + k] += (X1[r] - X0[r]) * w;
            }
        double JtJ[9] = {0}, G[9];
        for (int a = 0; a < d; ++a)
            for (int b = 0; b < d; ++b)
                for (int r = 0; r < d; ++r) JtJ[a * d + b] += J[r * d + a] * J[r * d + b];
        double Jinv[9];
        double det = inv_small(d, J, Jinv);
        if (!(det > 0)) throw std::runtime_error("inverted or degenerate cell");
        inv_small(d, JtJ, G);   // (J^T J)^{-1}
        double N[12][3], C[12][3];
        edge_basis(d, p, N, C);
        for (int i = 0; i < ne; ++i)
            for (int j = 0; j < ne; ++j) {
                double mv = 0, kv = 0;
                for (int a = 0; a < d; ++a)
                    for (int b = 0; b < d; ++b) mv += N[i][a] * G[a * d + b] * N[j][b];
                if (d == 3) {
                    for (int a = 0; a < 3; ++a)
                        for (int b = 0; b < 3; ++b) kv += C[i][a] * JtJ[a * 3 + b] * C[j][b];
                } else {
                    kv = C[i][0] * C[j][0];
                }
                Me[i * ne + j] += w * sigma * det * mv;
                Ke[i * ne + j] += w * nu / det * kv;
            }
        for (int i = 0; i < nn; ++i)
            for (int j = 0; j < nn; ++j) {
                double v = 0;
                for (int a = 0; a < d; ++a)
                    for (int b = 0; b < d; ++b) v += D[i][a] * G[a * d + b] * D[j][b];
                Kne[i * nn + j] += w * sigma * det * v;
            }
    }
}

// ------------------------------------------------------------ ELL assembly
struct RowAcc {
    int cap;
    std::vector<int> col, cnt;
    std::vector<double> val;
    RowAcc(int rows, int cap_) : cap(cap_), col((size_t)rows * cap_, -1), cnt(rows, 0), val((size_t)rows * cap_, 0.0) {}
    void add(int r, int c, double v) {
        int *C = &col[(size_t)r * cap];
        for (int s = 0; s < cnt[r]; ++s)
            if (C[s] == c) { val[(size_t)r * cap + s] += v; return; }
        if (cnt[r] == cap) throw std::runtime_error("ELL row capacity exceeded");
        C[cnt[r]] = c; val[(size_t)r * cap + cnt[r]] = v; ++cnt[r];
    }
    // compress: sort columns, drop exact zeros, pad with (pad_col(r), 0)
    HostELL finish(bool square) {
        HostELL E;
        E.rows = (int)cnt.size();
        int width = 0;
        std::vector<std::vector<std::pair<int, double>>> rows(E.rows);
        for (int r = 0; r < E.rows; ++r) {
            for (int s = 0; s < cnt[r]; ++s) {
                double v = val[(size_t)r * cap + s];
                if (v != 0.0) rows[r].push_back({col[(size_t)r * cap + s], v});
            }
            std::sort(rows[r].begin(), rows[r].end());
            width = std::max(width, (int)rows[r].size());
        }
        E.width = std::max(width, 1);
        E.col.assign((size_t)E.rows * E.width, 0);
        E.val.assign((size_t)E.rows * E.width, 0.0);
        for (int r = 0; r < E.rows; ++r) {
            for (int s = 0; s < E.width; ++s) {
                if (s < (int)rows[r].size()) {
                    E.col[(size_t)r * E.width + s] = rows[r][s].first;
                    E.val[(size_t)r * E.width + s] = rows[r][s].second;
                } else {
                    E.col[(size_t)r * E.width + s] = square ? r : 0;
                }
            }
        }
        return E;
    }
};

static std::vector<double> ell_diag(const HostELL &E) {
    std::vector<double> d(E.rows, 0.0);
    for (int r = 0; r < E.rows; ++r)
        for (int s = 0; s < E.width; ++s)
            if (E.col[(size_t)r * E.width + s] == r) d[r] += E.val[(size_t)r * E.width + s];
    return d;
}

void assemble(HostLevel &L) {
    const HostMesh &m = L.mesh;
    const int d = m.dim, ne = d == 3 ? 12 : 4, nn = 1 << d;
    RowAcc M(m.n_edges, d == 3 ? 40 : 8), K(m.n_edges, d == 3 ? 40 : 8), Kn(m.n_nodes, d == 3 ? 27 : 9);
    std::vector<double> Me(144), Ke(144), Kne(64);
    for (int c = 0; c < m.n_cells; ++c) {
        element(m, c, L.sigma[c], L.nu[c], Me.data(), Ke.data(), Kne.data());
        const int *E = &m.cell_edges[(size_t)ne * c];
        const int *N = &m.cell_nodes[(size_t)nn * c];
        for (int i = 0; i < ne; ++i)
            for (int j = 0; j < ne; ++j) {
                M.add(E[i], E[j], Me[i * ne + j]);
                K.add(E[i], E[j], Ke[i * ne + j]);
            }
        for (int i = 0; i < nn; ++i)
            for (int j = 0; j < nn; ++j) Kn.add(N[i], N[j], Kne[i * nn + j]);
    }
    L.M = M.finish(true);
    L.K = K.finish(true);
    L.Kn = Kn.finish(true);
    // merged M/K pattern (one gather feeds both products)
    {
        RowAcc mk(m.n_edges, L.M.width + L.K.width), kk(m.n_edges, L.M.width + L.K.width);
        for (int r = 0; r < m.n_edges; ++r) {
            for (int s = 0; s < L.K.width; ++s) {
                const double v = L.K.val[(size_t)r * L.K.width + s];
                if (v != 0.0) { mk.add(r, L.K.col[(size_t)r * L.K.width + s], 0.0); kk.add(r, L.K.col[(size_t)r * L.K.width + s], v); }
            }
            for (int s = 0; s < L.M.width; ++s) {
                const double v = L.M.val[(size_t)r * L.M.width + s];
                if (v != 0.0) { mk.add(r, L.M.col[(size_t)r * L.M.width + s], v); kk.add(r, L.M.col[(size_t)r * L.M.width + s], 0.0); }
            }
        }
        // same insertion order in both accumulators -> identical column lists; keep every slot
        // (a zero M value must not drop a K entry), sorted by column
        const int cap = mk.cap;
        int width = 0;
        for (int r = 0; r < m.n_edges; ++r) width = std::max(width, mk.cnt[r]);
        L.MK.rows = m.n_edges; L.MK.width = std::max(width, 1);
        L.MK.col.assign((size_t)L.MK.rows * L.MK.width, 0);
        L.MK.val.assign((size_t)L.MK.rows * L.MK.width, 0.0);
        L.MKk.assign((size_t)L.MK.rows * L.MK.width, 0.0);
        std::vector<std::pair<int, std::pair<double, double>>> row;
        for (int r = 0; r < m.n_edges; ++r) {
            row.clear();
            for (int s = 0; s < mk.cnt[r]; ++s)
                row.push_back({mk.col[(size_t)r * cap + s], {mk.val[(size_t)r * cap + s], kk.val[(size_t)r * cap + s]}});
            std::sort(row.begin(), row.end());
            for (int s = 0; s < L.MK.width; ++s) {
                const size_t o = (size_t)r * L.MK.width + s;
                if (s < (int)row.size()) { L.MK.col[o] = row[s].first; L.MK.val[o] = row[s].second.first; L.MKk[o] = row[s].second.second; }
                else L.MK.col[o] = r;
            }
        }
    }
    L.dM = ell_diag(L.M);
    L.dK = ell_diag(L.K);
    L.dN = ell_diag(L.Kn);
    // G^T incidence (node -> +-incident edges)
    RowAcc gt(m.n_nodes, d == 3 ? 6 : 4);
    for (int e = 0; e < m.n_edges; ++e) {
        gt.add(m.edge_nodes[2 * e], 2 * e + 1, 1.0);       // start node: -1
        gt.add(m.edge_nodes[2 * e + 1], 2 * e, 1.0);       // end node: +1
    }
    HostELL GT;
    GT.rows = m.n_nodes;
    GT.width = d == 3 ? 6 : 4;
    GT.col.assign((size_t)GT.rows * GT.width, -1);
    GT.val.clear();
    for (int r = 0; r < m.n_nodes; ++r) {
        std::vector<int> cs(&gt.col[(size_t)r * gt.cap], &gt.col[(size_t)r * gt.cap] + gt.cnt[r]);
        std::sort(cs.begin(), cs.end());
        for (size_t s = 0; s < cs.size(); ++s) GT.col[(size_t)r * GT.width + s] = cs[s];
    }
    L.GT = GT;
    // G^T M_sigma: since K G = 0, G^T (f - L x) = G^T f - (Ct (x) G^T M) x + (Nt (x) G^T M) x_prev
    // (fused nodal residual)
    RowAcc gm(m.n_nodes, GT.width * L.M.width);
    for (int n = 0; n < m.n_nodes; ++n)
        for (int s = 0; s < GT.width; ++s) {
            const int code = GT.col[(size_t)n * GT.width + s];
            if (code < 0) break;
            const int e = code >> 1;
            const double sg = (code & 1) ? -1.0 : 1.0;
            for (int t = 0; t < L.M.width; ++t) {
                const double v = L.M.val[(size_t)e * L.M.width + t];
                if (v != 0.0) gm.add(n, L.M.col[(size_t)e * L.M.width + t], sg * v);
            }
        }
    L.GtM = gm.finish(false);
}

// ------------------------------------------------------------- transfers
static int edge_id(const HostMesh &m, int dir, const int *ijk) {
    const int nx = m.n[0], ny = m.n[1];
    if (m.dim == 2) {
        if (dir == 0) return ijk[0] + nx * ijk[1];
        return m.Ex + ijk[0] + (nx + 1) * ijk[1];
    }
    if (dir == 0) return ijk[0] + nx * (ijk[1] + (ny + 1) * ijk[2]);
    if (dir == 1) return m.Ex + ijk[0] + (nx + 1) * (ijk[1] + ny * ijk[2]);
    return m.Ex + m.Ey + ijk[0] + (nx + 1) * (ijk[1] + (ny + 1) * ijk[2]);
}

// Canonical Nedelec interpolation of coarse edge functions on the fine edges
// of a 2:1 refinement (R6): weight 1/2 x (Q1 hat weights across the edge).
static void build_transfers(const HostMesh &f, const HostMesh &c, HostELL &Pg, HostELL &Rg) {
    const int d = f.dim;
    RowAcc P(f.n_edges, d == 3 ? 4 : 2), R(c.n_edges, d == 3 ? 18 : 6);
    for (int dir = 0; dir < d; ++dir) {
        int lim[3];
        for (int a = 0; a < 3; ++a) lim[a] = a < d ? (a == dir ? f.n[a] : f.n[a] + 1) : 1;
        for (int k = 0; k < lim[2]; ++k)
            for (int j = 0; j < lim[1]; ++j)
                for (int i = 0; i < lim[0]; ++i) {
                    int ijk[3] = {i, j, k};
                    const int ef = edge_id(f, dir, ijk);
                    // transverse axes: list of (coarse index, weight)
                    int cidx[3][2]; double cw[3][2]; int cnt[3];
                    for (int a = 0; a < d; ++a) {
                        if (a == dir) { cidx[a][0] = ijk[a] / 2; cw[a][0] = 0.5; cnt[a] = 1; continue; }
                        if (ijk[a] % 2 == 0) { cidx[a][0] = ijk[a] / 2; cw[a][0] = 1.0; cnt[a] = 1; }
                        else { cidx[a][0] = (ijk[a] - 1) / 2; cidx[a][1] = (ijk[a] + 1) / 2; cw[a][0] = cw[a][1] = 0.5; cnt[a] = 2; }
                    }
                    if (d == 2) { cnt[2] = 1; cidx[2][0] = 0; cw[2][0] = 1.0; }
                    for (int s0 = 0; s0 < cnt[0]; ++s0)
                        for (int s1 = 0; s1 < cnt[1]; ++s1)
                            for (int s2 = 0; s2 < cnt[2]; ++s2) {
                                int cc[3] = {cidx[0][s0], cidx[1][s1], cidx[2][s2]};
                                double w = cw[0][s0] * cw[1][s1] * cw[2][s2];
                                const int ec = edge_id(c, dir, cc);
                                P.add(ef, ec, w);
                                R.add(ec, ef, w);
                            }
                }
    }
    Pg = P.finish(false);
    Rg = R.finish(false);
}

static void coarsen_mesh(const HostLevel &F, HostLevel &C) {
    const HostMesh &f = F.mesh;
    const int d = f.dim;
    int nc[3] = {f.n[0] / 2, f.n[1] / 2, d == 3 ? f.n[2] / 2 : 1};
    std::vector<double> X;
    const int nxc = nc[0], nyc = nc[1], nzc = d == 3 ? nc[2] : 0;
    for (int k = 0; k <= nzc; ++k)
        for (int j = 0; j <= nyc; ++j)
            for (int i = 0; i <= nxc; ++i) {
                int fid = 2 * i + (f.n[0] + 1) * (2 * j + (f.n[1] + 1) * 2 * k);
                for (int a = 0; a < d; ++a) X.push_back(f.coords[(size_t)fid * d + a]);
            }
    C.mesh = make_mesh(d, nc, X.data());
    const int ncc = C.mesh.n_cells, nch = 1 << d;
    C.sigma.assign(ncc, 0.0); C.nu.assign(ncc, 0.0); C.ratio_min.assign(ncc, 0.0);
    for (int k = 0; k < (d == 3 ? nc[2] : 1); ++k)
        for (int j = 0; j < nc[1]; ++j)
            for (int i = 0; i < nc[0]; ++i) {
                const int cc = i + nc[0] * (j + nc[1] * k);
                double s = 0, n = 0, r = 1e300;
                for (int ch = 0; ch < nch; ++ch) {
                    int a = ch & 1, b = (ch >> 1) & 1, c2 = (ch >> 2) & 1;
                    int fc = (2 * i + a) + f.n[0] * ((2 * j + b) + f.n[1] * (2 * k + c2));
                    s += F.sigma[fc]; n += F.nu[fc]; r = std::min(r, F.ratio_min[fc]);
                }
                C.sigma[cc] = s / nch; C.nu[cc] = n / nch; C.ratio_min[cc] = r;
            }
}

static double level_lambda(const HostLevel &L) {
    // Eq. (3): min over cells of min_{x in T}(beta/alpha) * tau / h_T^2, h_T = longest edge (l.109)
    const HostMesh &m = L.mesh;
    const int d = m.dim, ne = d == 3 ? 12 : 4;
    double tmin = *std::min_element(L.tau.begin(), L.tau.end());
    double lam = 1e300;
    for (int c = 0; c < m.n_cells; ++c) {
        double h2 = 0;
        for (int i = 0; i < ne; ++i) {
            int e = m.cell_edges[(size_t)ne * c + i];
            const double *A = &m.coords[(size_t)m.edge_nodes[2 * e] * d];
            const double *B = &m.coords[(size_t)m.edge_nodes[2 * e + 1] * d];
            double l2 = 0;
            for (int a = 0; a < d; ++a) l2 += (B[a] - A[a]) * (B[a] - A[a]);
            h2 = std::max(h2, l2);
        }
        lam = std::min(lam, L.ratio_min[c] * tmin / h2);
    }
    return lam;
}

// Row schedules for L1 reuse: the rows of a small box of nodes
// (3D 4x2x2, 2D 8x4) are processed by one CTA, so the columns they share are
// fetched from L2 once per CTA.  Edge (dir, node) belongs to the box of its
// start node; within a box: node order, then direction.
static void box_schedule(const HostMesh &m, HostLevel &L) {
    const int d = m.dim;
    int B[3] = {d == 3 ? 4 : 8, d == 3 ? 2 : 4, d == 3 ? 2 : 1};
    if (const char *e = std::getenv("ST_BOX")) {   // tuning knob: "bx,by,bz"
        int a = 0, b = 0, c = 0;
        if (std::sscanf(e, "%d,%d,%d", &a, &b, &c) == 3 && a > 0 && b > 0 && c > 0) { B[0] = a; B[1] = b; B[2] = d == 3 ? c : 1; }
    }
    const int nn[3] = {m.n[0] + 1, m.n[1] + 1, d == 3 ? m.n[2] + 1 : 1};
    const int nb[3] = {(nn[0] + B[0] - 1) / B[0], (nn[1] + B[1] - 1) / B[1], (nn[2] + B[2] - 1) / B[2]};
    L.sched_e.clear(); L.bptr_e.assign(1, 0); L.sched_n.clear(); L.bptr_n.assign(1, 0);
    const int nx = m.n[0], ny = m.n[1], nz = d == 3 ? m.n[2] : 0;
    for (int bk = 0; bk < nb[2]; ++bk)
        for (int bj = 0; bj < nb[1]; ++bj)
            for (int bi = 0; bi < nb[0]; ++bi) {
                for (int k = bk * B[2]; k < std::min(nn[2], (bk + 1) * B[2]); ++k)
                    for (int j = bj * B[1]; j < std::min(nn[1], (bj + 1) * B[1]); ++j)
                        for (int i = bi * B[0]; i < std::min(nn[0], (bi + 1) * B[0]); ++i) {
                            L.sched_n.push_back(i + (nx + 1) * (j + (ny + 1) * k));
                            if (i < nx) L.sched_e.push_back(i + nx * (j + (ny + 1) * k));
                            if (j < ny) L.sched_e.push_back(m.Ex + i + (nx + 1) * (j + ny * k));
                            if (d == 3 && k < nz) L.sched_e.push_back(m.Ex + m.Ey + i + (nx + 1) * (j + (ny + 1) * k));
                        }
                L.bptr_e.push_back((int)L.sched_e.size());
                L.bptr_n.push_back((int)L.sched_n.size());
            }
}

// A level is "uniform" when every cell is the same axis-aligned box (then the
// matrix-free pencil march applies).  Exact comparison against the
// lattice i*hx, j*hy, k*hz built from the corner coordinates.
static void detect_uniform(HostLevel &L) {
    const HostMesh &m = L.mesh;
    const int d = m.dim;
    L.uniform = false;
    if (d != 3) return;
    const int nx = m.n[0], ny = m.n[1], nz = m.n[2];
    const double *X0 = &m.coords[0];
    const double *X1 = &m.coords[(size_t)(nx + (nx + 1) * (ny + (ny + 1) * nz)) * 3];
    const double h[3] = {(X1[0] - X0[0]) / nx, (X1[1] - X0[1]) / ny, (X1[2] - X0[2]) / nz};
    for (int k = 0; k <= nz; ++k)
        for (int j = 0; j <= ny; ++j)
            for (int i = 0; i <= nx; ++i) {
                const double *X = &m.coords[(size_t)(i + (nx + 1) * (j + (ny + 1) * k)) * 3];
                const double want[3] = {X0[0] + i * h[0], X0[1] + j * h[1], X0[2] + k * h[2]};
                for (int a = 0; a < 3; ++a)
                    if (std::fabs(X[a] - want[a]) > 1e-13 * (std::fabs(h[a]) * (m.n[a]) + std::fabs(X0[a]))) return;
            }
    L.uniform = true;
    for (int a = 0; a < 3; ++a) L.hbox[a] = h[a];
}

// Structured stencil table (stencil.cuh): on a uniform hex level, every edge row's merged (M, K)
// entries are mapped to structural slots; rows of one (direction, boundary class) must carry
// bitwise identical coefficients, M must vanish off the parallel block (axis-aligned cells), and a
// slot whose neighbour does not exist must be zero for the whole class.  Returns false (the level
// keeps the ELL kernels) when any of this fails, e.g. for per-cell varying coefficients.
// K_n of a uniform hex level as a 27-point node stencil per boundary class (nstencil.cuh): every
// node of a class must carry the class representative's coefficients (to a few ulps, as for the
// edge table) and every nonzero slot must point at an existing node
bool build_node_tab(const HostLevel &L, NodeTab &tab) {
    const HostMesh &m = L.mesh;
    if (m.dim != 3 || !L.uniform || L.Kn.rows != m.n_nodes) return false;
    const int nx = m.n[0], ny = m.n[1], nz = m.n[2];
    const int W = L.Kn.width;
    std::memset(&tab, 0, sizeof(tab));
    bool seen[kSnClasses] = {};
    double row[kSnSlots];
    for (int r = 0; r < m.n_nodes; ++r) {
        const int i = r % (nx + 1), j = (r / (nx + 1)) % (ny + 1), l = r / ((nx + 1) * (ny + 1));
        const int cls = 9 * st_cls(i, nx) + 3 * st_cls(j, ny) + st_cls(l, nz);
        for (int s2 = 0; s2 < kSnSlots; ++s2) row[s2] = 0.0;
        bool has[kSnSlots] = {};
        for (int s = 0; s < W; ++s) {
            const size_t o = (size_t)r * W + s;
            const double v = L.Kn.val[o];
            if (v == 0.0) continue;                        // padding / exact zeros
            const int c = L.Kn.col[o];
            const int i2 = c % (nx + 1), j2 = (c / (nx + 1)) % (ny + 1), l2 = c / ((nx + 1) * (ny + 1));
            const int di = i2 - i, dj = j2 - j, dl = l2 - l;
            if (std::abs(di) > 1 || std::abs(dj) > 1 || std::abs(dl) > 1) return false;
            const int sl = 9 * (di + 1) + 3 * (dj + 1) + (dl + 1);
            if (has[sl]) return false;
            has[sl] = true;
            row[sl] = v;
        }
        double *t = tab.c[cls];
        if (!seen[cls]) {
            seen[cls] = true;
            for (int s2 = 0; s2 < kSnSlots; ++s2) t[s2] = row[s2];
        } else {
            double sc = 0.0;
            for (int s2 = 0; s2 < kSnSlots; ++s2) sc = std::max(sc, std::fabs(row[s2]));
            const double tol = 8.0 * std::nextafter(sc, 2.0 * sc + 1.0) - 8.0 * sc;
            // (an entry that is zero in exact arithmetic may come out as a few ulps of the row scale
            // on a non-dyadic mesh, so zero-ness is compared through the same tolerance)
            for (int s2 = 0; s2 < kSnSlots; ++s2)
                if (std::fabs(t[s2] - row[s2]) > tol) return false;
        }
        for (int s2 = 0; s2 < kSnSlots; ++s2) {
            if (t[s2] == 0.0) continue;
            const int di = s2 / 9 - 1, dj = (s2 / 3) % 3 - 1, dl = s2 % 3 - 1;
            if (i + di < 0 || i + di > nx || j + dj < 0 || j + dj > ny || l + dl < 0 || l + dl > nz) return false;
        }
    }
    for (int c = 0; c < kSnClasses; ++c) tab.dinv[c] = tab.c[c][13] != 0.0 ? 1.0 / tab.c[c][13] : 0.0;
    return true;
}

bool build_stencil_tab(const HostLevel &L, StencilTab &tab) {
    const HostMesh &m = L.mesh;
    if (m.dim != 3 || !L.uniform || L.MK.rows != m.n_edges) return false;
    const int nx = m.n[0], ny = m.n[1], nz = m.n[2];
    const int W = L.MK.width;
    std::memset(&tab, 0, sizeof(tab));
    bool seen[3][kStClasses] = {};
    auto decode = [&](int e, int &T, int &i, int &j, int &l) {
        if (e < m.Ex) { T = 0; i = e % nx; j = (e / nx) % (ny + 1); l = e / (nx * (ny + 1)); }
        else if (e < m.Ex + m.Ey) { const int f = e - m.Ex; T = 1; i = f % (nx + 1); j = (f / (nx + 1)) % ny; l = f / ((nx + 1) * ny); }
        else { const int f = e - m.Ex - m.Ey; T = 2; i = f % (nx + 1); j = (f / (nx + 1)) % (ny + 1); l = f / ((nx + 1) * (ny + 1)); }
    };
    auto exists = [&](int T, int i, int j, int l) {
        if (i < 0 || j < 0 || l < 0 || i > nx || j > ny || l > nz) return false;
        return T == 0 ? i < nx : (T == 1 ? j < ny : l < nz);
    };
    double2 row[kStSlots];
    bool has[kStSlots];
    for (int r = 0; r < m.n_edges; ++r) {
        int T, i, j, l;
        decode(r, T, i, j, l);
        const int cls = T == 0 ? 3 * st_cls(j, ny) + st_cls(l, nz)
                               : (T == 1 ? 3 * st_cls(i, nx) + st_cls(l, nz) : 3 * st_cls(i, nx) + st_cls(j, ny));
        for (int s2 = 0; s2 < kStSlots; ++s2) { row[s2] = make_double2(0.0, 0.0); has[s2] = false; }
        for (int s = 0; s < W; ++s) {
            const size_t o = (size_t)r * W + s;
            const double mv = L.MK.val[o], kv = L.MKk[o];
            if (mv == 0.0 && kv == 0.0) continue;        // padding (col = row, value 0)
            int T2, i2, j2, l2;
            decode(L.MK.col[o], T2, i2, j2, l2);
            const int o0 = i2 - i, o1 = j2 - j, o2 = l2 - l;
            const int oT = T == 0 ? o0 : (T == 1 ? o1 : o2);
            const int oT2 = T2 == 0 ? o0 : (T2 == 1 ? o1 : o2);
            const int t3 = 3 - T - T2;
            const int o3 = t3 == 0 ? o0 : (t3 == 1 ? o1 : o2);
            if (T2 == T) {
                if (oT != 0) return false;
                for (int a = 0; a < 3; ++a)
                    if (a != T && std::abs(a == 0 ? o0 : (a == 1 ? o1 : o2)) > 1) return false;
            } else {
                if (oT < 0 || oT > 1 || oT2 < -1 || oT2 > 0 || o3 < -1 || o3 > 1) return false;
                if (mv != 0.0) return false;                 // M couples parallel edges only here
            }
            const int sl = st_slot(T, T2, o0, o1, o2);
            if (has[sl]) return false;
            has[sl] = true;
            row[sl] = make_double2(mv, kv);
        }
        // the first row of a class is its representative; every other row must agree with it to a
        // few ulps of the row's scale (cells of a uniform but non-dyadic mesh, e.g. h = 1/3, get
        // coordinate differences that round differently, so their element matrices differ by ulps)
        double2 *t = tab.c[T][cls];
        if (!seen[T][cls]) {
            seen[T][cls] = true;
            for (int s2 = 0; s2 < kStSlots; ++s2) t[s2] = row[s2];
        } else {
            double sm = 0.0, sk = 0.0;
            for (int s2 = 0; s2 < kStSlots; ++s2) { sm = std::max(sm, std::fabs(row[s2].x)); sk = std::max(sk, std::fabs(row[s2].y)); }
            const double tm = 8.0 * std::nextafter(sm, 2.0 * sm + 1.0) - 8.0 * sm, tk = 8.0 * std::nextafter(sk, 2.0 * sk + 1.0) - 8.0 * sk;
            for (int s2 = 0; s2 < kStSlots; ++s2)
                if (std::fabs(t[s2].x - row[s2].x) > tm || std::fabs(t[s2].y - row[s2].y) > tk ||
                    ((t[s2].x == 0.0) != (row[s2].x == 0.0)) || ((t[s2].y == 0.0) != (row[s2].y == 0.0)))
                    return false;
        }
    }
    // every nonzero slot of a class must point at an existing edge for every row of the class
    for (int r = 0; r < m.n_edges; ++r) {
        int T, i, j, l;
        decode(r, T, i, j, l);
        const int cls = T == 0 ? 3 * st_cls(j, ny) + st_cls(l, nz)
                               : (T == 1 ? 3 * st_cls(i, nx) + st_cls(l, nz) : 3 * st_cls(i, nx) + st_cls(j, ny));
        for (int T2 = 0; T2 < 3; ++T2)
            for (int o0 = -1; o0 <= 1; ++o0)
                for (int o1 = -1; o1 <= 1; ++o1)
                    for (int o2 = -1; o2 <= 1; ++o2) {
                        const int oT = T == 0 ? o0 : (T == 1 ? o1 : o2);
                        const int oT2 = T2 == 0 ? o0 : (T2 == 1 ? o1 : o2);
                        if (T2 == T ? oT != 0 : (oT < 0 || oT2 > 0)) continue;
                        const double2 c = tab.c[T][cls][st_slot(T, T2, o0, o1, o2)];
                        if ((c.x != 0.0 || c.y != 0.0) && !exists(T2, i + o0, j + o1, l + o2)) return false;
                    }
    }
    return true;
}

// Spatial coarsening chain of the finest mesh for the inner V-cycle (R13): chain[i] is the
// mesh coarsened i times (coefficients averaged as for the outer hierarchy, R6), with the
// transfers chain[i] -> chain[i+1] in chain[i].Pg / Rg.  Every outer level's mesh is one of
// them (outer level l sits at chain index = number of space coarsenings above it).
void build_chain(const HostLevel &L0, std::vector<HostLevel> &chain) {
    chain.clear();
    chain.emplace_back();
    chain[0].mesh = L0.mesh; chain[0].sigma = L0.sigma; chain[0].nu = L0.nu; chain[0].ratio_min = L0.ratio_min;
    for (size_t i = 0;; ++i) {
        HostLevel &C = chain[i];
        assemble(C);
        box_schedule(C.mesh, C);
        const HostMesh &m = C.mesh;
        bool can = true;
        for (int a = 0; a < m.dim; ++a) can = can && (m.n[a] % 2 == 0) && m.n[a] >= 2;
        if (!can) break;
        HostLevel N;
        coarsen_mesh(C, N);
        build_transfers(C.mesh, N.mesh, C.Pg, C.Rg);
        C.space_coarsened = true;
        chain.push_back(std::move(N));
    }
}

void build_hierarchy(const st_params &p, const Options &o, const TimeMats &tm, std::vector<HostLevel> &levels) {
    const int Q = tm.Q, q = Q - 1;
    levels.clear();
    levels.emplace_back();
    {
        HostLevel &L = levels.back();
        int n[3] = {p.nx, p.ny, p.nz};
        L.mesh = make_mesh(p.dim, n, p.coords);
        L.sigma.assign(p.sigma, p.sigma + L.mesh.n_cells);
        L.nu.assign(p.nu, p.nu + L.mesh.n_cells);
        L.ratio_min.resize(L.mesh.n_cells);
        for (int c = 0; c < L.mesh.n_cells; ++c) L.ratio_min[c] = L.nu[c] / L.sigma[c];
        L.tau.assign(p.tau, p.tau + p.n_slabs);
    }
    for (int lvl = 0;; ++lvl) {
        HostLevel &L = levels[lvl];
        assemble(L);
        box_schedule(L.mesh, L);
        detect_uniform(L);
        const int S = (int)L.tau.size();
        L.lambda = level_lambda(L);
        if (S <= o.min_slabs || S % 2) break;
        const HostMesh &m = L.mesh;
        bool can = true;
        for (int a = 0; a < m.dim; ++a) can = can && (m.n[a] % 2 == 0) && m.n[a] >= 2;
        bool cs = false;
        if (o.mode == 0) cs = L.lambda >= o.lambda_crit && can;
        else if (o.mode == 2) cs = lvl == 0 && can;
        L.space_coarsened = cs;
        // time transfer matrices per coarse slab (R7): Pt[(j*Q + b)][a] = phi_a(position of fine node (j,b))
        L.Pt.assign((size_t)(S / 2) * 2 * Q * Q, 0.0);
        for (int K = 0; K < S / 2; ++K) {
            const double th = L.tau[2 * K] / (L.tau[2 * K] + L.tau[2 * K + 1]);
            for (int j = 0; j < 2; ++j)
                for (int b = 0; b < Q; ++b) {
                    const double sb = q == 0 ? 0.0 : (double)b / q;
                    const double pos = j == 0 ? th * sb : th + (1.0 - th) * sb;
                    for (int a = 0; a < Q; ++a)
                        L.Pt[(size_t)K * 2 * Q * Q + (j * Q + b) * Q + a] = lag(q, a, pos);
                }
        }
        HostLevel C;
        if (cs) {
            coarsen_mesh(L, C);
            build_transfers(L.mesh, C.mesh, L.Pg, L.Rg);
        } else {
            C.mesh = L.mesh; C.sigma = L.sigma; C.nu = L.nu; C.ratio_min = L.ratio_min;
        }
        C.tau.resize(S / 2);
        for (int K = 0; K < S / 2; ++K) C.tau[K] = L.tau[2 * K] + L.tau[2 * K + 1];
        levels.push_back(std::move(C));
    }
    // coarsest level: dense inverse of A_k = Ct (x) M + tau_k Mt (x) K, index a*n + e (R8)
    HostLevel &Lc = levels.back();
    const int n = Lc.mesh.n_edges, N = Q * n, S = (int)Lc.tau.size();
    if ((double)N * N * S > 64.0e6) throw std::length_error("coarsest level too large for the dense solve");
    Lc.Ainv.assign((size_t)S * N * N, 0.0);
    std::vector<double> A((size_t)N * N);
    for (int k = 0; k < S; ++k) {
        std::fill(A.begin(), A.end(), 0.0);
        for (int e = 0; e < n; ++e) {
            for (int s = 0; s < Lc.M.width; ++s) {
                int c = Lc.M.col[(size_t)e * Lc.M.width + s]; double v = Lc.M.val[(size_t)e * Lc.M.width + s];
                for (int b = 0; b < Q; ++b)
                    for (int a = 0; a < Q; ++a) A[(size_t)(b * n + e) * N + a * n + c] += tm.Ct[b * Q + a] * v;
            }
            for (int s = 0; s < Lc.K.width; ++s) {
                int c = Lc.K.col[(size_t)e * Lc.K.width + s]; double v = Lc.K.val[(size_t)e * Lc.K.width + s];
                for (int b = 0; b < Q; ++b)
                    for (int a = 0; a < Q; ++a) A[(size_t)(b * n + e) * N + a * n + c] += Lc.tau[k] * tm.Mt[b * Q + a] * v;
            }
        }
        invert(N, A.data(), &Lc.Ainv[(size_t)k * N * N]);
    }
}

}  // namespace st
