// stencil.cuh — structured stencil march for uniform hexahedral levels (included by kernels.cu,
// inside namespace st, after the helpers it uses).
//
// The space-time operator of PAPER.md l.51-77, (L x)_k = (Ct(x)M + tau_k Mt(x)K) x_k - (Nt(x)M) x_{k-1},
// with the lowest-order Nedelec mass M_sigma and curl-curl K_nu of l.126-128 on a level whose cells
// are all the same axis-aligned box and whose coefficients are uniform.  On such a level the 33
// (M, K) coefficients of an edge row depend only on the row's direction and on which of its 4
// cells exist (boundary class), so they live in a 14 KB kernel-parameter table (constant bank 0;
// the interior class is read at compile-time offsets into uniform registers) and the column of
// every coefficient follows from the structured numbering of include/st.h: no ELL indices at all.
//
// Register reuse (the point of this kernel): a warp marches a pencil of nodes (i, j)
// along z for 16 slabs x 2 time nodes (lane = (slab, time node a)).  At z-level s it loads the 21
// edges the pencil's rows need from that level (6 x-edges, 6 y-edges, 9 z-edges) ONCE and pushes
// their contributions into the open row accumulators of levels s-1, s, s+1 (X, Y rows) and s-1, s
// (Z rows); the rows of level s-1 are then complete and leave through the epilogue.  That is 21
// vector loads per node and lane instead of 3 x 33 for three ELL rows: 4.7x fewer L1 wavefronts.
// A CTA is a tile of kStTI x kStTJ pencils of one slab chunk so that the halo edges neighbouring
// pencils share are L1 hits.
//
// Upwind coupling (residual only): time node 0 of slab k needs (M x_q) of slab k-1; inside a warp
// that is the m accumulator of the lane (k-1, q), one shuffle.  For the first slab of the warp the
// march also accumulates (M x_q) of the slab before the chunk from warp-uniform (broadcast) loads of
// its 15 mass-coupled neighbours per level (or of the previous rank's end values `prev`).
//
// Epilogue per row: the lane holds (M x_a, K x_a) of its own time node a; it forms the
// contributions of x_a to (A x)_b for both b and swaps the partner's share with one shuffle (the
// (Q x Q) time blocks Ct, Mt of R1 are applied this way, as is the Jacobi block inverse D^{-1}).
#pragma once

struct StGeo {
    int nx, ny, nz, Ex, Ey;
    int S, tiles_i, n_tiles, n_chunks;
};

constexpr int kStTI = 4, kStTJ = 2;            // pencils per CTA (one warp each)
constexpr int kStWarps = kStTI * kStTJ;
constexpr int kStInterior = 4;                 // class (1, 1): both transverse coordinates inside

template <bool FAST>
__device__ __forceinline__ double2 st_coef(const StencilTab &tab, int T, int cls, int slot) {
    if (FAST) return tab.c[T][kStInterior][slot];
    return tab.c[T][cls][slot];
}

// open accumulators of the lane's time node a: (M x_a, K x_a) per row type and open level
// (X, Y rows: levels s-1, s, s+1; Z rows: s-1, s); StPrev: M x_q of the slab before the chunk
struct StAcc {
    double xm[3], xk[3], ym[3], yk[3], zm[2], zk[2];
};
struct StPrev {
    double x[3], y[3], z[2];
};

// per-pencil row offsets of the 21 in-plane neighbours (clamped into the mesh: a neighbour that
// does not exist has a zero coefficient in every class that reaches it)
struct StPencil {
    int i, j;
    bool ok;
    unsigned ox[2][3], oy[3][2], oz[3][3];
};

__device__ __forceinline__ int st_clamp(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__device__ __forceinline__ void st_pencil(const StGeo &g, int tile, int warp, StPencil &P) {
    const int ti = tile % g.tiles_i, tj = tile / g.tiles_i;
    P.i = ti * kStTI + warp % kStTI;
    P.j = tj * kStTJ + warp / kStTI;
    P.ok = P.i <= g.nx && P.j <= g.ny;
    const int i = P.ok ? P.i : 0, j = P.ok ? P.j : 0;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) P.ox[a][b] = st_clamp(i - 1 + a, 0, g.nx - 1) + g.nx * st_clamp(j - 1 + b, 0, g.ny);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) P.oy[a][b] = st_clamp(i - 1 + a, 0, g.nx) + (g.nx + 1) * st_clamp(j - 1 + b, 0, g.ny - 1);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) P.oz[a][b] = st_clamp(i - 1 + a, 0, g.nx) + (g.nx + 1) * st_clamp(j - 1 + b, 0, g.ny);
}

// element (row, a, k) of a space-time vector at byte row * rowbytes from the lane base
__device__ __forceinline__ double st_ld(const char *base, unsigned row, unsigned rowbytes) {
    return __ldg(reinterpret_cast<const double *>(base + (size_t)row * rowbytes));
}

// Push the inputs of z-level s into the open rows.  xin[a][b]: x-edge (i-1+a, j-1+b, s); yin[a][b]:
// y-edge (i-1+a, j-1+b, s); zin[a][b]: z-edge (i-1+a, j-1+b, s).  clsX[d] / clsY[d]: class of the
// X / Y row at level s-1+d, clsZ: class of the pencil's Z rows.
template <bool FAST, bool ZIN>
__device__ __forceinline__ void st_push(const StencilTab &tab, const double (&xin)[2][3], const double (&yin)[3][2],
                                        const double (&zin)[3][3], const int (&clsX)[3], const int (&clsY)[3],
                                        int clsZ, StAcc &A) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const int o2 = 1 - d;                  // input level s relative to the row level s-1+d
        // X rows: x-neighbours (i, j-1+b) o = (0, b-1, o2)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            const double2 c = st_coef<FAST>(tab, 0, clsX[d], st_slot(0, 0, 0, b - 1, o2));
            A.xm[d] = fma(c.x, xin[1][b], A.xm[d]);
            A.xk[d] = fma(c.y, xin[1][b], A.xk[d]);
        }
        // X rows: y-neighbours (i-1+a, j-1+b), a in {1,2}, b in {0,1}
#pragma unroll
        for (int a = 1; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b)
                A.xk[d] = fma(st_coef<FAST>(tab, 0, clsX[d], st_slot(0, 1, a - 1, b - 1, o2)).y, yin[a][b], A.xk[d]);
        // X rows: z-neighbours (i-1+a, j-1+b) with o2 in {-1, 0} (d in {1, 2}), a in {1,2}
        if (ZIN && d >= 1) {
#pragma unroll
            for (int a = 1; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b)
                    A.xk[d] = fma(st_coef<FAST>(tab, 0, clsX[d], st_slot(0, 2, a - 1, b - 1, o2)).y, zin[a][b], A.xk[d]);
        }
        // Y rows: x-neighbours (i-1+a, j-1+b), a in {0,1}, b in {1,2}
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 1; b < 3; ++b)
                A.yk[d] = fma(st_coef<FAST>(tab, 1, clsY[d], st_slot(1, 0, a - 1, b - 1, o2)).y, xin[a][b], A.yk[d]);
        // Y rows: y-neighbours (i-1+a, j)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double2 c = st_coef<FAST>(tab, 1, clsY[d], st_slot(1, 1, a - 1, 0, o2));
            A.ym[d] = fma(c.x, yin[a][1], A.ym[d]);
            A.yk[d] = fma(c.y, yin[a][1], A.yk[d]);
        }
        // Y rows: z-neighbours (i-1+a, j-1+b), b in {1,2}
        if (ZIN && d >= 1) {
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 1; b < 3; ++b)
                    A.yk[d] = fma(st_coef<FAST>(tab, 1, clsY[d], st_slot(1, 2, a - 1, b - 1, o2)).y, zin[a][b], A.yk[d]);
        }
    }
    // Z rows at level s-1+e: x- and y-neighbours at o2 = 1 - e in {0, 1}
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int o2 = 1 - e;
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b)
                A.zk[e] = fma(st_coef<FAST>(tab, 2, clsZ, st_slot(2, 0, a - 1, b - 1, o2)).y, xin[a][b], A.zk[e]);
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b)
                A.zk[e] = fma(st_coef<FAST>(tab, 2, clsZ, st_slot(2, 1, a - 1, b - 1, o2)).y, yin[a][b], A.zk[e]);
    }
    // Z row at level s: z-neighbours of the same level only
    if (ZIN) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                const double2 c = st_coef<FAST>(tab, 2, clsZ, st_slot(2, 2, a - 1, b - 1, 0));
                A.zm[1] = fma(c.x, zin[a][b], A.zm[1]);
                A.zk[1] = fma(c.y, zin[a][b], A.zk[1]);
            }
    }
}

// the mass-coupled part of st_push for the slab before the chunk (time node q only)
template <bool FAST, bool ZIN>
__device__ __forceinline__ void st_push_prev(const StencilTab &tab, const double (&xp)[3], const double (&yp)[3],
                                             const double (&zp)[3][3], const int (&clsX)[3], const int (&clsY)[3],
                                             int clsZ, StPrev &B) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const int o2 = 1 - d;
#pragma unroll
        for (int b = 0; b < 3; ++b)
            B.x[d] = fma(st_coef<FAST>(tab, 0, clsX[d], st_slot(0, 0, 0, b - 1, o2)).x, xp[b], B.x[d]);
#pragma unroll
        for (int a = 0; a < 3; ++a)
            B.y[d] = fma(st_coef<FAST>(tab, 1, clsY[d], st_slot(1, 1, a - 1, 0, o2)).x, yp[a], B.y[d]);
    }
    if (ZIN) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b)
                B.z[1] = fma(st_coef<FAST>(tab, 2, clsZ, st_slot(2, 2, a - 1, b - 1, 0)).x, zp[a][b], B.z[1]);
    }
}

// Lane context: time node a, slab k, tau_k, and the column a of the time matrices
// (cm[b] = Ct[b][a], ck[b] = tau_k Mt[b][a]: the contribution of x_a to (A x)_b per unit M x_a, K x_a)
template <int Q>
struct StLane {
    static constexpr int SPW = 32 / Q;         // slabs per warp
    int a, k;
    double t, cm[Q], ck[Q];
};

template <int Q>
__device__ __forceinline__ void st_lane(const KT &kt, const double *__restrict__ tau, int chunk, StLane<Q> &L) {
    const int lane = threadIdx.x & 31;
    L.a = lane % Q;
    L.k = chunk * StLane<Q>::SPW + lane / Q;
    L.t = __ldg(tau + L.k);
#pragma unroll
    for (int b = 0; b < Q; ++b) {
        double c = kt.Ct[b * Q], m = kt.Mt[b * Q];
#pragma unroll
        for (int a = 1; a < Q; ++a)
            if (L.a == a) { c = kt.Ct[b * Q + a]; m = kt.Mt[b * Q + a]; }
        L.cm[b] = c;
        L.ck[b] = L.t * m;
    }
}

// sum over the Q lanes of a slab of their per-b contributions v[b], for the own b = a
template <int Q>
__device__ __forceinline__ double st_gather(const StLane<Q> &L, const double (&v)[Q]) {
    if constexpr (Q == 1) {
        return v[0];
    } else {
        const double own = L.a ? v[1] : v[0], other = L.a ? v[0] : v[1];
        return own + __shfl_xor_sync(0xffffffffu, other, 1);
    }
}

// column a of the Jacobi block D = Ct dm + tau Mt dk and of its inverse (R3)
template <int Q>
__device__ __forceinline__ void st_block(const KT &kt, const StLane<Q> &L, double dm, double dk, double (&Dcol)[Q],
                                         double (&Icol)[Q]) {
    if constexpr (Q == 1) {
        Dcol[0] = kt.Ct[0] * dm + L.t * kt.Mt[0] * dk;
        Icol[0] = 1.0 / Dcol[0];
    } else {
        const double d00 = kt.Ct[0] * dm + L.t * kt.Mt[0] * dk, d01 = kt.Ct[1] * dm + L.t * kt.Mt[1] * dk;
        const double d10 = kt.Ct[2] * dm + L.t * kt.Mt[2] * dk, d11 = kt.Ct[3] * dm + L.t * kt.Mt[3] * dk;
        const double inv = 1.0 / (d00 * d11 - d01 * d10);
        Dcol[0] = L.a ? d01 : d00;
        Dcol[1] = L.a ? d11 : d10;
        Icol[0] = (L.a ? -d01 : d11) * inv;
        Icol[1] = (L.a ? d00 : -d10) * inv;
    }
}

// the march over one pencil; Op supplies pre(T, row) (own-row loads of the rows that complete at
// this step, issued before the step's gathers) and emit<FAST>(T, row, cls, m, k, mprev)
template <int Q, bool PREVM, class Op>
__device__ __forceinline__ void st_march(const StGeo &g, const StencilTab &tab, const StPencil &P, const char *base,
                                         unsigned rowbytes, const char *pbase, unsigned prowbytes, Op &op) {
    StAcc A;
    StPrev B;
#pragma unroll
    for (int d = 0; d < 3; ++d) { A.xm[d] = A.xk[d] = A.ym[d] = A.yk[d] = 0.0; B.x[d] = B.y[d] = 0.0; }
    A.zm[0] = A.zk[0] = A.zm[1] = A.zk[1] = 0.0;
    B.z[0] = B.z[1] = 0.0;
    const int i = P.i, j = P.j;
    const int ci = st_cls(i, g.nx), cj = st_cls(j, g.ny);
    const bool inner_pencil = ci == 1 && cj == 1;
    const int clsZ = 3 * ci + cj;
    const unsigned px_step = (unsigned)(g.nx * (g.ny + 1)), py_step = (unsigned)((g.nx + 1) * g.ny);
    const unsigned pz_step = (unsigned)((g.nx + 1) * (g.ny + 1));
    for (int s = 0; s <= g.nz + 1; ++s) {
        const int l = s - 1;                   // level of the rows that complete at this step
        const unsigned rX = (unsigned)(i + g.nx * (j + (g.ny + 1) * l));
        const unsigned rY = (unsigned)(g.Ex + i + (g.nx + 1) * (j + g.ny * l));
        const unsigned rZ = (unsigned)(g.Ex + g.Ey + i + (g.nx + 1) * (j + (g.ny + 1) * l));
        const bool eX = s >= 1 && i < g.nx, eY = s >= 1 && j < g.ny, eZ = s >= 1 && l < g.nz;
        if (eX) op.pre(0, rX);
        if (eY) op.pre(1, rY);
        if (eZ) op.pre(2, rZ);
        const bool fast = inner_pencil && s >= 2 && s <= g.nz - 2;
        if (s <= g.nz) {
            const unsigned bx = px_step * s, by = g.Ex + py_step * s, bz = g.Ex + g.Ey + pz_step * s;
            double xin[2][3], yin[3][2], zin[3][3];
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) xin[a][b] = st_ld(base, bx + P.ox[a][b], rowbytes);
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 2; ++b) yin[a][b] = st_ld(base, by + P.oy[a][b], rowbytes);
            const bool zin_ok = s < g.nz;
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) zin[a][b] = zin_ok ? st_ld(base, bz + P.oz[a][b], rowbytes) : 0.0;
            double xp[3], yp[3], zp[3][3];
            if (PREVM) {
#pragma unroll
                for (int b = 0; b < 3; ++b) xp[b] = st_ld(pbase, bx + P.ox[1][b], prowbytes);
#pragma unroll
                for (int a = 0; a < 3; ++a) yp[a] = st_ld(pbase, by + P.oy[a][1], prowbytes);
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int b = 0; b < 3; ++b) zp[a][b] = zin_ok ? st_ld(pbase, bz + P.oz[a][b], prowbytes) : 0.0;
            }
            if (fast) {
                const int dummy[3] = {0, 0, 0};
                st_push<true, true>(tab, xin, yin, zin, dummy, dummy, clsZ, A);
                if (PREVM) st_push_prev<true, true>(tab, xp, yp, zp, dummy, dummy, clsZ, B);
            } else {
                int clsX[3], clsY[3];
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    const int cl = st_cls(s - 1 + d, g.nz);
                    clsX[d] = 3 * cj + cl;
                    clsY[d] = 3 * ci + cl;
                }
                if (zin_ok) {
                    st_push<false, true>(tab, xin, yin, zin, clsX, clsY, clsZ, A);
                    if (PREVM) st_push_prev<false, true>(tab, xp, yp, zp, clsX, clsY, clsZ, B);
                } else {
                    st_push<false, false>(tab, xin, yin, zin, clsX, clsY, clsZ, A);
                    if (PREVM) st_push_prev<false, false>(tab, xp, yp, zp, clsX, clsY, clsZ, B);
                }
            }
        }
        if (s >= 1) {
            const int cl = st_cls(l, g.nz);
            if (fast) {
                if (eX) op.template emit<true>(0, rX, kStInterior, A.xm[0], A.xk[0], B.x[0]);
                if (eY) op.template emit<true>(1, rY, kStInterior, A.ym[0], A.yk[0], B.y[0]);
                if (eZ) op.template emit<true>(2, rZ, kStInterior, A.zm[0], A.zk[0], B.z[0]);
            } else {
                if (eX) op.template emit<false>(0, rX, 3 * cj + cl, A.xm[0], A.xk[0], B.x[0]);
                if (eY) op.template emit<false>(1, rY, 3 * ci + cl, A.ym[0], A.yk[0], B.y[0]);
                if (eZ) op.template emit<false>(2, rZ, clsZ, A.zm[0], A.zk[0], B.z[0]);
            }
        }
        A.xm[0] = A.xm[1]; A.xm[1] = A.xm[2]; A.xm[2] = 0.0;
        A.xk[0] = A.xk[1]; A.xk[1] = A.xk[2]; A.xk[2] = 0.0;
        A.ym[0] = A.ym[1]; A.ym[1] = A.ym[2]; A.ym[2] = 0.0;
        A.yk[0] = A.yk[1]; A.yk[1] = A.yk[2]; A.yk[2] = 0.0;
        A.zm[0] = A.zm[1]; A.zm[1] = 0.0;
        A.zk[0] = A.zk[1]; A.zk[1] = 0.0;
        if (PREVM) {
            B.x[0] = B.x[1]; B.x[1] = B.x[2]; B.x[2] = 0.0;
            B.y[0] = B.y[1]; B.y[1] = B.y[2]; B.y[2] = 0.0;
            B.z[0] = B.z[1]; B.z[1] = 0.0;
        }
    }
}

// ------------------------------------------------------------------ kernels
// Residual epilogue: r = f - L x; z = omega_s D^{-1} r (the first
// block-Jacobi sweep of Eq. (2) from zero, l.79-82); |r|^2 partials.
template <int Q, bool R_OUT, bool Z_OUT, bool NORM>
struct StResOp {
    const StencilTab &tab;
    const KT &kt;
    const StLane<Q> &L;
    const char *fb;                 // f + (a*S + k) elements, in bytes
    char *rb, *zb;
    unsigned rowbytes;
    double omega_s;
    bool first;                     // lane of the chunk's first slab
    double nrm;
    double fv[3];
    __device__ __forceinline__ void pre(int T, unsigned row) { fv[T] = st_ld(fb, row, rowbytes); }
    template <bool FAST>
    __device__ __forceinline__ void emit(int T, unsigned row, int cls, double m, double k, double mprev) {
        double u[Q];
#pragma unroll
        for (int b = 0; b < Q; ++b) u[b] = L.cm[b] * m + L.ck[b] * k;
        const double ax = st_gather<Q>(L, u);
        // upwind coupling on time node 0: (M x_q)(k-1) from lane (k-1, q), right before this lane
        const double up = __shfl_up_sync(0xffffffffu, m, 1);
        const double mp = L.a != 0 ? 0.0 : (first ? mprev : up);
        const double rr = fv[T] - ax + mp;
        const size_t off = (size_t)row * rowbytes;
        if (R_OUT) *reinterpret_cast<double *>(rb + off) = rr;
        if (Z_OUT) {
            const double2 dd = st_coef<FAST>(tab, T, cls, st_slot(T, T, 0, 0, 0));
            double Dc[Q], Ic[Q], v[Q];
            st_block<Q>(kt, L, dd.x, dd.y, Dc, Ic);
#pragma unroll
            for (int b = 0; b < Q; ++b) v[b] = Ic[b] * rr;
            *reinterpret_cast<double *>(zb + off) = omega_s * st_gather<Q>(L, v);
        }
        if (NORM) nrm = fma(rr, rr, nrm);
    }
};

template <int Q, bool R_OUT, bool Z_OUT, bool NORM>
__global__ void __launch_bounds__(32 * kStWarps, 2)
k_st_residual(StGeo g, const __grid_constant__ StencilTab tab, const double *__restrict__ tau,
              const double *__restrict__ x, const double *__restrict__ f, const double *__restrict__ prev,
              double *__restrict__ r, double *__restrict__ z, double omega_s, KT kt, double *__restrict__ partial) {
    const int chunk = blockIdx.x / g.n_tiles, tile = blockIdx.x - chunk * g.n_tiles;
    StLane<Q> L;
    st_lane<Q>(kt, tau, chunk, L);
    StPencil P;
    st_pencil(g, tile, threadIdx.x >> 5, P);
    const unsigned rowbytes = (unsigned)(8u * Q * g.S);
    const size_t lane_off = ((size_t)L.a * g.S + L.k) * 8;
    StResOp<Q, R_OUT, Z_OUT, NORM> op{tab, kt, L, reinterpret_cast<const char *>(f) + lane_off,
                                      reinterpret_cast<char *>(r) + lane_off, reinterpret_cast<char *>(z) + lane_off,
                                      rowbytes, omega_s, (threadIdx.x & 31) < Q, 0.0, {0.0, 0.0, 0.0}};
    if (P.ok) {
        const char *base = reinterpret_cast<const char *>(x) + lane_off;
        const int k0 = chunk * StLane<Q>::SPW;
        if (k0 > 0) {
            // warp-uniform (broadcast) loads of x_q at slab k0 - 1
            const char *pb = reinterpret_cast<const char *>(x) + ((size_t)(Q - 1) * g.S + k0 - 1) * 8;
            st_march<Q, true>(g, tab, P, base, rowbytes, pb, rowbytes, op);
        } else if (prev) {
            st_march<Q, true>(g, tab, P, base, rowbytes, reinterpret_cast<const char *>(prev), 8u, op);
        } else {
            st_march<Q, false>(g, tab, P, base, rowbytes, nullptr, 0u, op);
        }
    }
    if (NORM) {
        __shared__ double sh[kStWarps];
        const double s = block_reduce_sum(op.nrm, sh);
        if (threadIdx.x == 0) partial[blockIdx.x] = s;
    }
}

// Block-Jacobi sweep epilogue on A_k (the inner approximation of Eq. (2), R3):
// znew = z + omega_s D^{-1} (r - A_k z); RECON: r = D z / omega_s; LAST: x += omega znew.
template <int Q, bool LAST, bool RECON>
struct StSweepOp {
    const StencilTab &tab;
    const KT &kt;
    const StLane<Q> &L;
    const char *zb, *rb;
    char *ob;
    unsigned rowbytes;
    double omega_s, omega;
    double zv[3], rv[3], xv[3];
    __device__ __forceinline__ void pre(int T, unsigned row) {
        const size_t off = (size_t)row * rowbytes;
        zv[T] = __ldg(reinterpret_cast<const double *>(zb + off));
        if (!RECON) rv[T] = __ldg(reinterpret_cast<const double *>(rb + off));
        if (LAST) xv[T] = *reinterpret_cast<const double *>(ob + off);
    }
    template <bool FAST>
    __device__ __forceinline__ void emit(int T, unsigned row, int cls, double m, double k, double) {
        const double2 dd = st_coef<FAST>(tab, T, cls, st_slot(T, T, 0, 0, 0));
        double Dc[Q], Ic[Q], c[Q], v[Q];
        st_block<Q>(kt, L, dd.x, dd.y, Dc, Ic);
        // d = r - A z, with r = D z / omega_s (RECON) or read
#pragma unroll
        for (int b = 0; b < Q; ++b) c[b] = (RECON ? Dc[b] * zv[T] / omega_s : 0.0) - (L.cm[b] * m + L.ck[b] * k);
        const double d = st_gather<Q>(L, c) + (RECON ? 0.0 : rv[T]);
#pragma unroll
        for (int b = 0; b < Q; ++b) v[b] = Ic[b] * d;
        const double res = zv[T] + omega_s * st_gather<Q>(L, v);
        double *o = reinterpret_cast<double *>(ob + (size_t)row * rowbytes);
        if (LAST) *o = xv[T] + omega * res;
        else *o = res;
    }
};

template <int Q, bool LAST, bool RECON>
__global__ void __launch_bounds__(32 * kStWarps, 2)
k_st_sweep(StGeo g, const __grid_constant__ StencilTab tab, const double *__restrict__ tau,
           const double *__restrict__ z, const double *__restrict__ r, double *out, double omega_s, double omega,
           KT kt) {
    const int chunk = blockIdx.x / g.n_tiles, tile = blockIdx.x - chunk * g.n_tiles;
    StLane<Q> L;
    st_lane<Q>(kt, tau, chunk, L);
    StPencil P;
    st_pencil(g, tile, threadIdx.x >> 5, P);
    if (!P.ok) return;
    const unsigned rowbytes = (unsigned)(8u * Q * g.S);
    const size_t lane_off = ((size_t)L.a * g.S + L.k) * 8;
    StSweepOp<Q, LAST, RECON> op{tab, kt, L, reinterpret_cast<const char *>(z) + lane_off,
                                 reinterpret_cast<const char *>(r) + lane_off, reinterpret_cast<char *>(out) + lane_off,
                                 rowbytes, omega_s, omega, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    st_march<Q, false>(g, tab, P, reinterpret_cast<const char *>(z) + lane_off, rowbytes, nullptr, 0u, op);
}
