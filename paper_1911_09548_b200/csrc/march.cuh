// march.cuh — matrix-free space-time operator for uniform (axis-aligned, equal box)
// hex levels: the pencil march (kernel "march").
//
// Lanes of a warp own consecutive slabs (lane 0 = halo slab k0-1, whose mass image
// feeds the upwind coupling of lane 1 through a shuffle); a warp marches along x
// over the nodes (i, j, k) of one pencil (j, k) and produces the rows of the x-, y-
// and z-edge starting at each node.  Per-cell coefficients sigma (mass) and nu
// (curl-curl) enter through
//   M_sigma  on a box cell: x-edges  sigma (hy hz / hx) (M1 (x) M1)   (M1 = [[1/3,1/6],[1/6,1/3]])
//   K_nu = C^T M_f C: face fluxes F = C x (circulation of the 4 edges), face mass per
//          cell and normal n: nu (h_n / (h_a h_b)) M1 between the cell's two faces of
//          normal n, then edges gather +-P of their 4 faces.
// (§3 l.126-128 for M_h, K_h; the factorisation is exact for lowest-order
// Nedelec on affine cells, checked against the assembled ELL operator by the parity
// tests.)  Carried state of the march window (per time node a): Y and Z at x = i
// (read one step ahead), Y(i-1,j,.), Z(i-1,.,k), the x-normal fluxes at i-1 and i,
// and the z-/y-normal face values P at i-1.  New loads per node: 9 X + 6 Y + 6 Z.
#pragma once

namespace st {

// Grid3 (internal.h): nx, ny, nz, Ex, Ey; mx = hy hz/hx, my = hx hz/hy, mz = hx hy/hz;
// wx = hx/(hy hz), wy = hy/(hx hz), wz = hz/(hx hy); per-cell sigma, nu.

__device__ __forceinline__ int xid(const Grid3 &g, int i, int j, int k) { return i + g.nx * (j + (g.ny + 1) * k); }
__device__ __forceinline__ int yid(const Grid3 &g, int i, int j, int k) { return g.Ex + i + (g.nx + 1) * (j + g.ny * k); }
__device__ __forceinline__ int zid(const Grid3 &g, int i, int j, int k) {
    return g.Ex + g.Ey + i + (g.nx + 1) * (j + (g.ny + 1) * k);
}
__device__ __forceinline__ bool cell_ok(const Grid3 &g, int i, int j, int k) {
    return i >= 0 && j >= 0 && k >= 0 && i < g.nx && j < g.ny && k < g.nz;
}
__device__ __forceinline__ double csig(const Grid3 &g, int i, int j, int k) {
    return cell_ok(g, i, j, k) ? __ldg(g.sigma + i + g.nx * (j + g.ny * k)) : 0.0;
}
__device__ __forceinline__ double cnu(const Grid3 &g, int i, int j, int k) {
    return cell_ok(g, i, j, k) ? __ldg(g.nu + i + g.nx * (j + g.ny * k)) : 0.0;
}

// value loader for one lane: slab ks (ks < 0: the slab before the rank's first one)
struct Lane {
    const double *x;
    const double *prev;   // end values of slab -1 (or null = zero initial state)
    int S, QS, ks, q;
    __device__ __forceinline__ double ld(int row, int a, bool ok) const {
        if (!ok) return 0.0;
        if (ks >= 0) return __ldg(x + (size_t)row * QS + a * S + ks);
        return (a == q && prev) ? __ldg(prev + row) : 0.0;
    }
};

constexpr double M1d = 1.0 / 3.0, M1o = 1.0 / 6.0;
__device__ __forceinline__ double m1(int u, int v) { return u == v ? M1d : M1o; }

// Per time node a: the carried window and one march step.
struct Win {
    double Yc[2][3];   // Y(i, j+dj, k+dk), dj in {-1,0}, dk in {-1,0,1}
    double Yp[3];      // Y(i-1, j, k+dk)
    double Zc[3][2];   // Z(i, j+dj, k+dk), dj in {-1,0,1}, dk in {-1,0}
    double Zp[3];      // Z(i-1, j+dj, k)
    double Fxc[2][2];  // Fx(i, j+dj, k+dk), dj, dk in {-1,0}
    double Fxp[2][2];  // Fx(i-1, ...)
    double Pzp, Pyp;   // Pz(i-1, j, k), Py(i-1, j, k)
};

// loads of the Y / Z values at x-position ii into (Yv, Zv)
__device__ __forceinline__ void load_yz(const Grid3 &g, const Lane &ln, int a, int ii, int j, int k,
                                        double (&Yv)[2][3], double (&Zv)[3][2]) {
    const bool iok = ii >= 0 && ii <= g.nx;
#pragma unroll
    for (int dj = -1; dj <= 0; ++dj)
#pragma unroll
        for (int dk = -1; dk <= 1; ++dk) {
            const int jj = j + dj, kk = k + dk;
            const bool ok = iok && jj >= 0 && jj < g.ny && kk >= 0 && kk <= g.nz;
            Yv[dj + 1][dk + 1] = ln.ld(ok ? yid(g, ii, jj, kk) : 0, a, ok);
        }
#pragma unroll
    for (int dj = -1; dj <= 1; ++dj)
#pragma unroll
        for (int dk = -1; dk <= 0; ++dk) {
            const int jj = j + dj, kk = k + dk;
            const bool ok = iok && jj >= 0 && jj <= g.ny && kk >= 0 && kk < g.nz;
            Zv[dj + 1][dk + 1] = ln.ld(ok ? zid(g, ii, jj, kk) : 0, a, ok);
        }
}

// Fx at x-position ii from the Y/Z values there: Fx(ii, j+dj, k+dk) = Z(j+dj+1,k+dk) - Z(j+dj,k+dk) - Y(j+dj,k+dk+1) + Y(j+dj,k+dk)
__device__ __forceinline__ void fx_from(const double (&Yv)[2][3], const double (&Zv)[3][2], double (&F)[2][2]) {
#pragma unroll
    for (int dj = 0; dj < 2; ++dj)
#pragma unroll
        for (int dk = 0; dk < 2; ++dk) F[dj][dk] = Zv[dj + 1][dk] - Zv[dj][dk] - Yv[dj][dk + 1] + Yv[dj][dk];
}

// cell coefficients around the current node, index [di][dj][dk] with di = 0 -> i-1, 1 -> i
struct Cells {
    double s[2][2][2], n[2][2][2];
};

// Values a march step needs from memory: X at x-position i, Y and Z one position ahead.
struct StepLoads {
    double Xc[3][3];   // X(i, j+dj, k+dk)
    double Yn[2][3];   // Y(i+1, j+dj, k+dk), dj in {-1,0}
    double Zn[3][2];   // Z(i+1, j+dj, k+dk), dk in {-1,0}
};

__device__ __forceinline__ void load_step(const Grid3 &g, const Lane &ln, int a, int i, int j, int k, StepLoads &L) {
    const bool xok_i = i < g.nx;
#pragma unroll
    for (int dj = -1; dj <= 1; ++dj)
#pragma unroll
        for (int dk = -1; dk <= 1; ++dk) {
            const int jj = j + dj, kk = k + dk;
            const bool ok = xok_i && jj >= 0 && jj <= g.ny && kk >= 0 && kk <= g.nz;
            L.Xc[dj + 1][dk + 1] = ln.ld(ok ? xid(g, i, jj, kk) : 0, a, ok);
        }
    load_yz(g, ln, a, i + 1, j, k, L.Yn, L.Zn);
}

// One step at node (i, j, k) for time node a from the loaded values: spatial images
// MX, MY, MZ, KX, KY, KZ of the three edges starting at the node; advances the window.
__device__ __forceinline__ void step(const Grid3 &g, const Cells &c, const StepLoads &L, Win &w, double out[6]) {
    const auto &Xc = L.Xc;
    const auto &Yn = L.Yn;
    const auto &Zn = L.Zn;
    // face fluxes at x-position i
    double Fz[2][3];   // Fz(i, j+dj, k+dk), dj in {-1,0}, dk in {-1,0,1}
#pragma unroll
    for (int dj = 0; dj < 2; ++dj)
#pragma unroll
        for (int dk = 0; dk < 3; ++dk) Fz[dj][dk] = Xc[dj][dk] + Yn[dj][dk] - Xc[dj + 1][dk] - w.Yc[dj][dk];
    double Fy[3][2];   // Fy(i, j+dj, k+dk), dj in {-1,0,1}, dk in {-1,0}
#pragma unroll
    for (int dj = 0; dj < 3; ++dj)
#pragma unroll
        for (int dk = 0; dk < 2; ++dk) Fy[dj][dk] = Xc[dj][dk + 1] - Xc[dj][dk] - Zn[dj][dk] + w.Zc[dj][dk];
    double Fxn[2][2];
    fx_from(Yn, Zn, Fxn);
    // face mass: P = sum over the two cells sharing the face along its normal
    double Pz[2], Py[2], Px[2][2];
#pragma unroll
    for (int dj = 0; dj < 2; ++dj)   // Pz(i, j-1+dj, k): cells (i, j-1+dj, k-1), (i, j-1+dj, k)
        Pz[dj] = g.wz * (c.n[1][dj][0] * (M1o * Fz[dj][0] + M1d * Fz[dj][1]) +
                         c.n[1][dj][1] * (M1d * Fz[dj][1] + M1o * Fz[dj][2]));
#pragma unroll
    for (int dk = 0; dk < 2; ++dk)   // Py(i, j, k-1+dk): cells (i, j-1, k-1+dk), (i, j, k-1+dk)
        Py[dk] = g.wy * (c.n[1][0][dk] * (M1o * Fy[0][dk] + M1d * Fy[1][dk]) +
                         c.n[1][1][dk] * (M1d * Fy[1][dk] + M1o * Fy[2][dk]));
#pragma unroll
    for (int dj = 0; dj < 2; ++dj)   // Px(i, j-1+dj, k-1+dk): cells (i-1, ..), (i, ..)
#pragma unroll
        for (int dk = 0; dk < 2; ++dk)
            Px[dj][dk] = g.wx * (c.n[0][dj][dk] * (M1o * w.Fxp[dj][dk] + M1d * w.Fxc[dj][dk]) +
                                 c.n[1][dj][dk] * (M1d * w.Fxc[dj][dk] + M1o * Fxn[dj][dk]));
    // curl-curl images (C^T P)
    out[3] = Pz[1] - Pz[0] + Py[0] - Py[1];                 // KX(i,j,k)
    out[4] = w.Pzp - Pz[1] + Px[1][1] - Px[1][0];           // KY(i,j,k)
    out[5] = Px[0][1] - Px[1][1] + Py[1] - w.Pyp;           // KZ(i,j,k)
    // mass images
    double mxv = 0.0;   // cells (i, j-1+b, k-1+cc): local position of X(i,j,k) is (1-b, 1-cc)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
            double t = 0.0;
#pragma unroll
            for (int b2 = 0; b2 < 2; ++b2)
#pragma unroll
                for (int c2 = 0; c2 < 2; ++c2) t += m1(1 - b, b2) * m1(1 - cc, c2) * Xc[b + b2][cc + c2];
            mxv += c.s[1][b][cc] * t;
        }
    out[0] = g.mx * mxv;
    double myv = 0.0;   // cells (i-1+aa, j, k-1+cc): Y(i-1+aa+a2, j, k-1+cc+c2)
#pragma unroll
    for (int aa = 0; aa < 2; ++aa)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
            double t = 0.0;
#pragma unroll
            for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
                for (int c2 = 0; c2 < 2; ++c2) {
                    const int ix = aa + a2, kz = cc + c2;   // 0 -> i-1, 1 -> i, 2 -> i+1
                    const double yv = ix == 0 ? w.Yp[kz] : (ix == 1 ? w.Yc[1][kz] : Yn[1][kz]);
                    t += m1(1 - aa, a2) * m1(1 - cc, c2) * yv;
                }
            myv += c.s[aa][1][cc] * t;
        }
    out[1] = g.my * myv;
    double mzv = 0.0;   // cells (i-1+aa, j-1+b, k): Z(i-1+aa+a2, j-1+b+b2, k)
#pragma unroll
    for (int aa = 0; aa < 2; ++aa)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            double t = 0.0;
#pragma unroll
            for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
                for (int b2 = 0; b2 < 2; ++b2) {
                    const int ix = aa + a2, jy = b + b2;
                    const double zv = ix == 0 ? w.Zp[jy] : (ix == 1 ? w.Zc[jy][1] : Zn[jy][1]);
                    t += m1(1 - aa, a2) * m1(1 - b, b2) * zv;
                }
            mzv += c.s[aa][b][1] * t;
        }
    out[2] = g.mz * mzv;
    // advance the window to i+1
#pragma unroll
    for (int dk = 0; dk < 3; ++dk) w.Yp[dk] = w.Yc[1][dk];
#pragma unroll
    for (int dj = 0; dj < 3; ++dj) w.Zp[dj] = w.Zc[dj][1];
#pragma unroll
    for (int dj = 0; dj < 2; ++dj)
#pragma unroll
        for (int dk = 0; dk < 3; ++dk) w.Yc[dj][dk] = Yn[dj][dk];
#pragma unroll
    for (int dj = 0; dj < 3; ++dj)
#pragma unroll
        for (int dk = 0; dk < 2; ++dk) w.Zc[dj][dk] = Zn[dj][dk];
#pragma unroll
    for (int dj = 0; dj < 2; ++dj)
#pragma unroll
        for (int dk = 0; dk < 2; ++dk) { w.Fxp[dj][dk] = w.Fxc[dj][dk]; w.Fxc[dj][dk] = Fxn[dj][dk]; }
    w.Pzp = Pz[1];
    w.Pyp = Py[1];
}

__device__ __forceinline__ void win_init(const Grid3 &g, const Lane &ln, int a, int j, int k, Win &w) {
    load_yz(g, ln, a, 0, j, k, w.Yc, w.Zc);
    fx_from(w.Yc, w.Zc, w.Fxc);
#pragma unroll
    for (int t = 0; t < 3; ++t) { w.Yp[t] = 0.0; w.Zp[t] = 0.0; }
#pragma unroll
    for (int dj = 0; dj < 2; ++dj)
#pragma unroll
        for (int dk = 0; dk < 2; ++dk) w.Fxp[dj][dk] = 0.0;
    w.Pzp = 0.0;
    w.Pyp = 0.0;
}


// all 8 cells around node (i, j, k) re-read each step (warp-broadcast L1 hits) instead of
// carried in registers: the window then fits 168 registers without spills
__device__ __forceinline__ void load_cells2(const Grid3 &g, int i, int j, int k, Cells &c) {
#pragma unroll
    for (int di = 0; di < 2; ++di)
#pragma unroll
        for (int dj = 0; dj < 2; ++dj)
#pragma unroll
            for (int dk = 0; dk < 2; ++dk) {
                c.s[di][dj][dk] = csig(g, i - 1 + di, j - 1 + dj, k - 1 + dk);
                c.n[di][dj][dk] = cnu(g, i - 1 + di, j - 1 + dj, k - 1 + dk);
            }
}

}  // namespace st
