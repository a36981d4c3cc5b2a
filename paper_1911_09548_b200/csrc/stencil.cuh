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
// along z for 32 slabs (lane = slab; all q+1 time nodes of the slab in the lane).  At z-level s it
// reads the 21 edges the pencil's rows need from that level (6 x-edges, 6 y-edges, 9 z-edges) ONCE
// and pushes their contributions into the open row accumulators of levels s-1, s, s+1 (X, Y rows)
// and s-1, s (Z rows); the rows of level s-1 are then complete and leave through the epilogue:
// 21 operand reads per node and slab instead of 3 x 33 for three ELL rows, every coefficient load
// shared by the q+1 time nodes, and the (q+1) x (q+1) time blocks of R1 applied in registers.
// A CTA is a tile of TI x TJ pencils of one slab chunk (StTile); its z-levels are staged in shared
// memory by TMA (below), halo included, so neighbouring pencils share every operand fetch.
//
// Upwind coupling (residual only): time node 0 of slab k needs (M x_q) of slab k-1: inside a warp
// the mass accumulator of lane k-1 (one shuffle); for the first slab of each 32-slab chunk a small
// gather pass (k_st_coupling: 9 mass entries per row and chunk, or the previous rank's end values
// `prev` for chunk 0) runs before the march.
#pragma once

struct StGeo {
    int nx, ny, nz, Ex, Ey;
    int S, tiles_i, n_tiles, n_chunks;
};

// CTA tile: TI x TJ pencils (one warp each) of one 32-slab chunk
template <int TI_, int TJ_>
struct StTile {
    static constexpr int TI = TI_, TJ = TJ_, Warps = TI_ * TJ_;
    static constexpr int BX = (TI_ + 1) * (TJ_ + 2);            // staged x-edge blocks per level
    static constexpr int BY = (TI_ + 2) * (TJ_ + 1);
    static constexpr int BZ = (TI_ + 2) * (TJ_ + 2);
};
// 12 warps at <= 168 registers (3 warps per scheduler; 13-16 warps would cap at 128 registers).
// Measured per c4 V-cycle (65 x 65 pencils per level-0 z-plane), residual / sweep family: 4 x 2 pencils
// (8 warps, 224 registers) 34.0 ms sweep; 4 x 3: 32.1 / 25.3; 3 x 4: 32.0 / 25.2; 6 x 2: 31.3 / 24.7
// (66 x 66 covered instead of 68 x 66); 4 x 4 (16 warps, 128 registers, 4-140 B spills): 33.6 / 26.8;
// 7 x 2 (14 warps, 128 registers): 35.8 / 29.9
#ifndef ST_TILE_I
#define ST_TILE_I 6
#define ST_TILE_J 2
#endif
using StTileRes = StTile<ST_TILE_I, ST_TILE_J>;
using StTileSweep = StTile<ST_TILE_I, ST_TILE_J>;
// the mass-only march (k_st_res_mass) carries half the accumulators and is latency-bound: 20 warps at 96
// registers (measured per c4 V-cycle: 9.37 ms at 4 x 3, 8.52 at 4 x 4, 7.75 at 5 x 4, 8.90 at 6 x 4)
#ifndef ST_MTILE_I
#define ST_MTILE_I 5
#define ST_MTILE_J 4
#endif
using StTileMass = StTile<ST_MTILE_I, ST_MTILE_J>;
constexpr int kStSPW = 32;                     // slabs per warp (lane = slab)
constexpr int kStInterior = 4;                 // class (1, 1): both transverse coordinates inside

template <bool FAST>
__device__ __forceinline__ double2 st_coef(const StencilTab &tab, int T, int cls, int slot) {
    if (FAST) return tab.c[T][kStInterior][slot];
    return tab.c[T][cls][slot];
}

// open accumulators (M x_b, K x_b) per row type, open level and time node b
// (X, Y rows: levels s-1, s, s+1; Z rows: s-1, s)
template <int Q>
struct StAcc {
    double xm[3][Q], xk[3][Q], ym[3][Q], yk[3][Q], zm[2][Q], zk[2][Q];
};

// Push the inputs of z-level s into the open rows.  xin[a][b][q]: x-edge (i-1+a, j-1+b, s), time
// node q; yin: y-edges (i-1+a, j-1+b, s); zin: z-edges (i-1+a, j-1+b, s).  clsX[d] / clsY[d]:
// class of the X / Y row at level s-1+d, clsZ: class of the pencil's Z rows.
#ifndef ST_PHASES
#define ST_PHASES 1
#endif
// compiler-only barrier: keeps the shared-memory reads of the next input group after the FMAs of
// this one, so that only one group of operands is live at a time (register budget -> warps/SM)
__device__ __forceinline__ void st_phase() {
#if ST_PHASES
    asm volatile("" ::: "memory");
#endif
}

// xs / ys / zs: the warp's x-, y-, z-edge input blocks of the staged level, element (a, b, q) at
// [(b * row + a) * Blk + q * 32] with row = the tile-box i extent of the edge type
// MK = false: mass part only (the nodal residual's mass form, k_st_res_mass); the curl-curl FMAs and
// the inputs only they read are compiled out
template <int Q, class Tl, bool FAST, bool ZIN, bool MK = true>
__device__ __forceinline__ void st_push(const StencilTab &tab, const double *xs, const double *ys, const double *zs,
                                        const int (&clsX)[3], const int (&clsY)[3], int clsZ, StAcc<Q> &A) {
    constexpr int Blk = Q * kStSPW;
    double xin[2][3][Q], yin[3][2][Q], zin[3][3][Q];
    // input groups (one index a of an edge type): loads ...
    auto ldx = [&](int a) {
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
            for (int q = 0; q < Q; ++q) xin[a][b][q] = xs[(b * (Tl::TI + 1) + a) * Blk + q * kStSPW];
    };
    auto ldy = [&](int a) {
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int q = 0; q < Q; ++q) yin[a][b][q] = ys[(b * (Tl::TI + 2) + a) * Blk + q * kStSPW];
    };
    auto ldz = [&](int a) {
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
            for (int q = 0; q < Q; ++q) zin[a][b][q] = zs[(b * (Tl::TI + 2) + a) * Blk + q * kStSPW];
    };
    // ... and FMAs.  Loop order: input outermost, then the open levels d and time nodes q innermost,
    // so that consecutive FMAs go to independent accumulators (latency of the fp64 pipe)
    // ---- x-edge inputs xin[a][b] = x-edge (i-1+a, j-1+b)
    auto fx = [&](int a) {
#pragma unroll
        for (int b = 0; b < 3; ++b) {
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const int o2 = 1 - d;
                if (a == 1) {                                   // X rows: o = (0, b-1, o2)
                    const double2 c = st_coef<FAST>(tab, 0, clsX[d], st_slot(0, 0, 0, b - 1, o2));
#pragma unroll
                    for (int q = 0; q < Q; ++q) {
                        A.xm[d][q] = fma(c.x, xin[a][b][q], A.xm[d][q]);
                        if (MK) A.xk[d][q] = fma(c.y, xin[a][b][q], A.xk[d][q]);
                    }
                }
                if (MK && b >= 1) {                             // Y rows: o = (a-1, b-1, o2)
                    const double c = st_coef<FAST>(tab, 1, clsY[d], st_slot(1, 0, a - 1, b - 1, o2)).y;
#pragma unroll
                    for (int q = 0; q < Q; ++q) A.yk[d][q] = fma(c, xin[a][b][q], A.yk[d][q]);
                }
            }
#pragma unroll
            for (int e = 0; e < 2; ++e) {                       // Z rows at s-1+e: o = (a-1, b-1, 1-e)
                if (!MK) break;
                const double c = st_coef<FAST>(tab, 2, clsZ, st_slot(2, 0, a - 1, b - 1, 1 - e)).y;
#pragma unroll
                for (int q = 0; q < Q; ++q) A.zk[e][q] = fma(c, xin[a][b][q], A.zk[e][q]);
            }
        }
    };
    // ---- y-edge inputs yin[a][b] = y-edge (i-1+a, j-1+b)
    auto fy = [&](int a) {
#pragma unroll
        for (int b = 0; b < 2; ++b) {
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const int o2 = 1 - d;
                if (MK && a >= 1) {                             // X rows: o = (a-1, b-1, o2)
                    const double c = st_coef<FAST>(tab, 0, clsX[d], st_slot(0, 1, a - 1, b - 1, o2)).y;
#pragma unroll
                    for (int q = 0; q < Q; ++q) A.xk[d][q] = fma(c, yin[a][b][q], A.xk[d][q]);
                }
                if (b == 1) {                                   // Y rows: o = (a-1, 0, o2)
                    const double2 c = st_coef<FAST>(tab, 1, clsY[d], st_slot(1, 1, a - 1, 0, o2));
#pragma unroll
                    for (int q = 0; q < Q; ++q) {
                        A.ym[d][q] = fma(c.x, yin[a][b][q], A.ym[d][q]);
                        if (MK) A.yk[d][q] = fma(c.y, yin[a][b][q], A.yk[d][q]);
                    }
                }
            }
#pragma unroll
            for (int e = 0; e < 2; ++e) {                       // Z rows: o = (a-1, b-1, 1-e)
                if (!MK) break;
                const double c = st_coef<FAST>(tab, 2, clsZ, st_slot(2, 1, a - 1, b - 1, 1 - e)).y;
#pragma unroll
                for (int q = 0; q < Q; ++q) A.zk[e][q] = fma(c, yin[a][b][q], A.zk[e][q]);
            }
        }
    };
    // ---- z-edge inputs zin[a][b] = z-edge (i-1+a, j-1+b) from level s to s+1
    auto fz = [&](int a) {
#pragma unroll
        for (int b = 0; b < 3; ++b) {
#pragma unroll
            for (int d = 1; d < 3; ++d) {                       // X, Y rows at s, s+1: o2 = 1 - d
                const int o2 = 1 - d;
                if (MK && a >= 1) {
                    const double c = st_coef<FAST>(tab, 0, clsX[d], st_slot(0, 2, a - 1, b - 1, o2)).y;
#pragma unroll
                    for (int q = 0; q < Q; ++q) A.xk[d][q] = fma(c, zin[a][b][q], A.xk[d][q]);
                }
                if (MK && b >= 1) {
                    const double c = st_coef<FAST>(tab, 1, clsY[d], st_slot(1, 2, a - 1, b - 1, o2)).y;
#pragma unroll
                    for (int q = 0; q < Q; ++q) A.yk[d][q] = fma(c, zin[a][b][q], A.yk[d][q]);
                }
            }
            const double2 c = st_coef<FAST>(tab, 2, clsZ, st_slot(2, 2, a - 1, b - 1, 0));   // Z row at s
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                A.zm[1][q] = fma(c.x, zin[a][b][q], A.zm[1][q]);
                if (MK) A.zk[1][q] = fma(c.y, zin[a][b][q], A.zk[1][q]);
            }
        }
    };
#if ST_PHASES == 2
    // one group ahead: the shared-memory reads of group g + 1 are issued before the FMAs of group g
    // (at most two groups of <= 3 inputs live; the order of the FMAs on every accumulator is that
    // of the three-phase form below)
    ldx(0);
    ldx(1); st_phase(); fx(0);
    ldy(0); st_phase(); fx(1);
    ldy(1); st_phase(); fy(0);
    ldy(2); st_phase(); fy(1);
    if (ZIN) ldz(0);
    st_phase(); fy(2);
    if (ZIN) {
        ldz(1); st_phase(); fz(0);
        ldz(2); st_phase(); fz(1);
        st_phase(); fz(2);
    }
#elif ST_PHASES == 3
    // two groups ahead
    ldx(0); ldx(1);
    ldy(0); st_phase(); fx(0);
    ldy(1); st_phase(); fx(1);
    ldy(2); st_phase(); fy(0);
    if (ZIN) ldz(0);
    st_phase(); fy(1);
    if (ZIN) ldz(1);
    st_phase(); fy(2);
    if (ZIN) {
        ldz(2); st_phase(); fz(0);
        st_phase(); fz(1);
        st_phase(); fz(2);
    }
#else
    ldx(0); ldx(1);
    fx(0); fx(1);
    st_phase();
    ldy(0); ldy(1); ldy(2);
    fy(0); fy(1); fy(2);
    if (ZIN) {
        st_phase();
        ldz(0); ldz(1); ldz(2);
        fz(0); fz(1); fz(2);
    }
#endif
}

// ------------------------------------------------------------- TMA staging
// Each z-level's inputs of the whole CTA tile are staged in shared memory by three 5-D TMA tile
// loads (cp.async.bulk.tensor, one elected thread, completion on an mbarrier), kStNB levels ahead
// of the march.  Tensor view of an edge block of a space-time vector (innermost first):
// (slab, time node, i, j, z-level); box (32, Q, tile i extent, tile j extent, 1) with the tile's
// one-edge halo.  Out-of-range box elements (mesh boundary, the z-level above the top) are
// zero-filled by the TMA unit, so the march needs no index clamping: every missing neighbour reads
// 0 and has a zero coefficient anyway.  The box lands as [j][i][time node][slab]: a warp reads its
// 21 x (q+1) inputs with conflict-free 8-byte LDS (lane = slab) at compile-time offsets.
#ifndef ST_NB
#define ST_NB 3
#endif
constexpr int kStNB = ST_NB;                                // staged z-levels in flight
template <int Q, class Tl>
struct StCfg {
    static constexpr int Blk = Q * kStSPW;                              // doubles per edge block
    static constexpr int Level = (Tl::BX + Tl::BY + Tl::BZ) * Blk;      // doubles per staged level
    static_assert((Tl::BX * Blk * 8) % 128 == 0 && (Tl::BY * Blk * 8) % 128 == 0 && (Level * 8) % 128 == 0,
                  "TMA destinations must stay 128-byte aligned");
};

struct StMaps {
    CUtensorMap x, y, z;            // the input vector's x-, y-, z-edge blocks
};

template <int Q, class Tl>
struct alignas(128) StSmem {
    double buf[kStNB][StCfg<Q, Tl>::Level];
    unsigned long long full[kStNB];
    unsigned done[kStNB];           // warps finished with the level in each buffer (last-arriver refill)
};

// Buffer release without a CTA barrier: every warp, once done with the level in buffer nb, counts
// itself in; the last warp to arrive resets the count and issues the TMA refill, so no warp waits
// for the slowest one (a warp that runs ahead blocks only on the full barrier of a level not yet
// landed).  Measured on c4 (ms per V-cycle, two runs each): sweep 24.8 / 25.0 vs 25.1 / 25.1 with a
// CTA barrier, node scan 4.56 / 4.59 vs 5.0 / 4.98, but residual 48.2 / 48.1 vs 46.9 / 46.7 -- so
// the residual keeps the barrier (and thread 0 refilling).
template <int Warps>
__device__ __forceinline__ bool st_release(unsigned *done) {
    __syncwarp();
    unsigned last = 0;
    if ((threadIdx.x & 31) == 0) {
        __threadfence_block();          // this warp's reads of the buffer are performed before the count
        last = atomicAdd(done, 1u) == Warps - 1;
        if (last) {
            __threadfence_block();      // ... and the refill's TMA is issued after every warp's count
            *done = 0;
        }
    }
    return __shfl_sync(0xffffffffu, last, 0) != 0;
}

__device__ __forceinline__ unsigned st_smem_addr(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void st_mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(st_smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void st_mbar_expect(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(st_smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void st_mbar_wait(unsigned long long *bar, unsigned parity) {
    const unsigned a = st_smem_addr(bar);
    unsigned ok = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void st_tma_5d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3, int c4,
                                          unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
        "%6}], [%7];" ::"r"(st_smem_addr(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
        "r"(st_smem_addr(bar))
        : "memory");
}

// issue the staging of z-level s into buffer s % kStNB (one thread)
template <int Q, class Tl>
__device__ __forceinline__ void st_stage(const StGeo &g, const StMaps &maps, StSmem<Q, Tl> &sm, int s, int i0, int j0,
                                         int k0) {
    using C = StCfg<Q, Tl>;
    const int nb = s % kStNB;
    const bool zin = s < g.nz;
    constexpr unsigned bx = Tl::BX * C::Blk * 8, by = Tl::BY * C::Blk * 8, bz = Tl::BZ * C::Blk * 8;
    const unsigned bytes = bx + by + (zin ? bz : 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    st_mbar_expect(&sm.full[nb], bytes);
    double *b = sm.buf[nb];
    st_tma_5d(b, &maps.x, k0, 0, i0 - 1, j0 - 1, s, &sm.full[nb]);
    st_tma_5d(b + Tl::BX * C::Blk, &maps.y, k0, 0, i0 - 1, j0 - 1, s, &sm.full[nb]);
    if (zin) st_tma_5d(b + (Tl::BX + Tl::BY) * C::Blk, &maps.z, k0, 0, i0 - 1, j0 - 1, s, &sm.full[nb]);
}

// Lane constants: slab k, tau_k, and per row type T the Jacobi block D = Ct dM + tau_k Mt dK of the
// interior class and its inverse (R3), row-major (Q x Q)
template <int Q>
struct StLane {
    int k;
    double t;
    double tMt[Q * Q];              // tau_k Mt
};

template <int Q>
__device__ __forceinline__ void st_lane(const KT &kt, const double *__restrict__ tau, int chunk, StLane<Q> &L) {
    L.k = chunk * kStSPW + (threadIdx.x & 31);
    L.t = __ldg(tau + L.k);
#pragma unroll
    for (int i = 0; i < Q * Q; ++i) L.tMt[i] = L.t * kt.Mt[i];
}

// D = Ct dm + tau Mt dk and D^{-1} (row-major)
template <int Q>
__device__ __forceinline__ void st_block(const KT &kt, const StLane<Q> &L, double dm, double dk, double (&D)[Q * Q],
                                         double (&Di)[Q * Q]) {
#pragma unroll
    for (int i = 0; i < Q * Q; ++i) D[i] = kt.Ct[i] * dm + L.tMt[i] * dk;
    if constexpr (Q == 1) {
        Di[0] = 1.0 / D[0];
    } else {
        const double inv = 1.0 / (D[0] * D[3] - D[1] * D[2]);
        Di[0] = D[3] * inv; Di[1] = -D[1] * inv; Di[2] = -D[2] * inv; Di[3] = D[0] * inv;
    }
}

// per-CTA table of the interior-class blocks: [T][D..., D^{-1}...][lane]
template <int Q>
struct StBlockTab {
    double v[3][2 * Q * Q][32];
};

template <int Q>
__device__ __forceinline__ void st_block_table(const StencilTab &tab, const KT &kt, const StLane<Q> &L,
                                               StBlockTab<Q> &bt) {
    if ((threadIdx.x >> 5) == 0) {
#pragma unroll
        for (int T = 0; T < 3; ++T) {
            const double2 dd = tab.c[T][kStInterior][st_slot(T, T, 0, 0, 0)];
            double D[Q * Q], Di[Q * Q];
            st_block<Q>(kt, L, dd.x, dd.y, D, Di);
#pragma unroll
            for (int i = 0; i < Q * Q; ++i) { bt.v[T][i][threadIdx.x] = D[i]; bt.v[T][Q * Q + i][threadIdx.x] = Di[i]; }
        }
    }
}

template <int Q, bool FAST>
__device__ __forceinline__ void st_row_block(const StencilTab &tab, const KT &kt, const StLane<Q> &L,
                                             const StBlockTab<Q> &bt, int T, int cls, double (&D)[Q * Q],
                                             double (&Di)[Q * Q]) {
    if (FAST) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int i = 0; i < Q * Q; ++i) { D[i] = bt.v[T][i][lane]; Di[i] = bt.v[T][Q * Q + i][lane]; }
    } else {
        const double2 dd = st_coef<false>(tab, T, cls, st_slot(T, T, 0, 0, 0));
        st_block<Q>(kt, L, dd.x, dd.y, D, Di);
    }
}

// (A x)_b = sum_a Ct[b][a] (M x_a) + tau Mt[b][a] (K x_a)   (PAPER.md l.51-77 with the R1 blocks)
template <int Q>
__device__ __forceinline__ void st_time(const KT &kt, const StLane<Q> &L, const double (&m)[Q], const double (&k)[Q],
                                        double (&ax)[Q]) {
#pragma unroll
    for (int b = 0; b < Q; ++b) {
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < Q; ++a) acc = fma(kt.Ct[b * Q + a], m[a], fma(L.tMt[b * Q + a], k[a], acc));
        ax[b] = acc;
    }
}

// The march of one CTA tile (one pencil per warp) over all z-levels.  Op supplies
// pre(T, row, own) (own-row values of the rows completing at this step; own = the staged block of
// the row at its level) and emit<FAST>(T, row, cls, m[Q], k[Q]); every warp reaches every
// barrier (also warps whose pencil lies outside the mesh).
template <int Q, class Tl, bool LAST_REFILL, class Op, bool MK = true>
__device__ __forceinline__ void st_march(const StGeo &g, const StencilTab &tab, const StMaps &maps, StSmem<Q, Tl> &sm,
                                         int tile, int chunk, Op &op) {
    using C = StCfg<Q, Tl>;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ti = tile % g.tiles_i, tj = tile / g.tiles_i;
    const int i0 = ti * Tl::TI, j0 = tj * Tl::TJ;
    const int wi = warp % Tl::TI, wj = warp / Tl::TI;
    const int i = i0 + wi, j = j0 + wj;
    const bool ok = i <= g.nx && j <= g.ny;
    const int k0 = chunk * kStSPW;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int b = 0; b < kStNB; ++b) { st_mbar_init(&sm.full[b], 1); sm.done[b] = 0; }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int s = 0; s < kStNB && s <= g.nz; ++s) st_stage<Q, Tl>(g, maps, sm, s, i0, j0, k0);
    StAcc<Q> A;
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int q = 0; q < Q; ++q) A.xm[d][q] = A.xk[d][q] = A.ym[d][q] = A.yk[d][q] = 0.0;
#pragma unroll
    for (int q = 0; q < Q; ++q) A.zm[0][q] = A.zk[0][q] = A.zm[1][q] = A.zk[1][q] = 0.0;
    const int ci = st_cls(i, g.nx), cj = st_cls(j, g.ny);
    const bool inner_pencil = ci == 1 && cj == 1;
    const int clsZ = 3 * ci + cj;
    // the warp's block offsets inside a staged level (doubles)
    const int ox = (wj * (Tl::TI + 1) + wi) * C::Blk + lane;
    const int oy = Tl::BX * C::Blk + (wj * (Tl::TI + 2) + wi) * C::Blk + lane;
    const int oz = (Tl::BX + Tl::BY) * C::Blk + (wj * (Tl::TI + 2) + wi) * C::Blk + lane;
    for (int s = 0; s <= g.nz + 1; ++s) {
        const int l = s - 1;                   // level of the rows that complete at this step
        const unsigned rX = (unsigned)(i + g.nx * (j + (g.ny + 1) * l));
        const unsigned rY = (unsigned)(g.Ex + i + (g.nx + 1) * (j + g.ny * l));
        const unsigned rZ = (unsigned)(g.Ex + g.Ey + i + (g.nx + 1) * (j + (g.ny + 1) * l));
        const bool eX = ok && s >= 1 && i < g.nx, eY = ok && s >= 1 && j < g.ny, eZ = ok && s >= 1 && l < g.nz;
        const double *lb = sm.buf[(s + kStNB - 1) % kStNB];         // level s-1 (own values)
        if (eX) op.pre(0, rX, lb + ox + C::Blk * ((Tl::TI + 1) + 1));
        if (eY) op.pre(1, rY, lb + oy + C::Blk * ((Tl::TI + 2) + 1));
        if (eZ) op.pre(2, rZ, lb + oz + C::Blk * ((Tl::TI + 2) + 1));
        const bool fast = inner_pencil && s >= 2 && s <= g.nz - 2;
        if (s <= g.nz) {
            const int nb = s % kStNB;
            st_mbar_wait(&sm.full[nb], (unsigned)((s / kStNB) & 1));
            const double *bb = sm.buf[nb];
            const bool zin_ok = s < g.nz;
            if (fast) {
                const int dummy[3] = {0, 0, 0};
                st_push<Q, Tl, true, true, MK>(tab, bb + ox, bb + oy, bb + oz, dummy, dummy, clsZ, A);
            } else {
                int clsX[3], clsY[3];
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    const int cl = st_cls(s - 1 + d, g.nz);
                    clsX[d] = 3 * cj + cl;
                    clsY[d] = 3 * ci + cl;
                }
                if (zin_ok) {
                    st_push<Q, Tl, false, true, MK>(tab, bb + ox, bb + oy, bb + oz, clsX, clsY, clsZ, A);
                } else {
                    st_push<Q, Tl, false, false, MK>(tab, bb + ox, bb + oy, bb + oz, clsX, clsY, clsZ, A);
                }
            }
        }
        if (s >= 1) {
            const int cl = st_cls(l, g.nz);
            if (fast) {
                if (eX) op.template emit<true>(0, rX, kStInterior, A.xm[0], A.xk[0]);
                if (eY) op.template emit<true>(1, rY, kStInterior, A.ym[0], A.yk[0]);
                if (eZ) op.template emit<true>(2, rZ, kStInterior, A.zm[0], A.zk[0]);
            } else {
                if (eX) op.template emit<false>(0, rX, 3 * cj + cl, A.xm[0], A.xk[0]);
                if (eY) op.template emit<false>(1, rY, 3 * ci + cl, A.ym[0], A.yk[0]);
                if (eZ) op.template emit<false>(2, rZ, clsZ, A.zm[0], A.zk[0]);
            }
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            A.xm[0][q] = A.xm[1][q]; A.xm[1][q] = A.xm[2][q]; A.xm[2][q] = 0.0;
            A.xk[0][q] = A.xk[1][q]; A.xk[1][q] = A.xk[2][q]; A.xk[2][q] = 0.0;
            A.ym[0][q] = A.ym[1][q]; A.ym[1][q] = A.ym[2][q]; A.ym[2][q] = 0.0;
            A.yk[0][q] = A.yk[1][q]; A.yk[1][q] = A.yk[2][q]; A.yk[2][q] = 0.0;
            A.zm[0][q] = A.zm[1][q]; A.zm[1][q] = 0.0;
            A.zk[0][q] = A.zk[1][q]; A.zk[1][q] = 0.0;
        }
        // this warp is done with level s-1 (own values): once every warp is, refill its buffer
        // with level s-1+kStNB
        if (LAST_REFILL) {
            if (s >= 1 && s - 1 + kStNB <= g.nz && st_release<Tl::Warps>(&sm.done[(s - 1) % kStNB]) &&
                (threadIdx.x & 31) == 0)
                st_stage<Q, Tl>(g, maps, sm, s - 1 + kStNB, i0, j0, k0);
        } else {
            __syncthreads();
            if (threadIdx.x == 0 && s >= 1 && s - 1 + kStNB <= g.nz)
                st_stage<Q, Tl>(g, maps, sm, s - 1 + kStNB, i0, j0, k0);
        }
    }
}

// ------------------------------------------------------------------ kernels
// element (row, b, k) of a space-time vector: row * rowbytes + b * S * 8 + k * 8 from the base
struct StRow {
    size_t off;                     // row * rowbytes + k * 8
    size_t bstride;                 // S * 8
};

// Residual epilogue: r = f - L x; z = omega_s D^{-1} r (the first
// block-Jacobi sweep of Eq. (2) from zero, l.79-82); |r|^2 partials.
template <int Q, bool R_OUT, bool Z_OUT, bool NORM>
struct StResOp {
    const StencilTab &tab;
    const KT &kt;
    const StLane<Q> &L;
    const StBlockTab<Q> &bt;
    const char *fb;                 // f + k elements, in bytes
    char *rb, *zb;
    unsigned rowbytes;
    size_t bstride;
    double omega_s;
    bool first;                     // lane of the chunk's first slab
    const double *cpl;              // (M x_q) of the slab before this chunk, per row (k_st_coupling), or null
    double nrm;
    double fv[3][Q], cv[3];
    __device__ __forceinline__ void pre(int T, unsigned row, const double *) {
        const char *p = fb + (size_t)row * rowbytes;
#pragma unroll
        for (int b = 0; b < Q; ++b) fv[T][b] = __ldg(reinterpret_cast<const double *>(p + b * bstride));
        cv[T] = first && cpl ? __ldg(cpl + row) : 0.0;     // null: no coupling (zero initial state, x = 0)
    }
    template <bool FAST>
    __device__ __forceinline__ void emit(int T, unsigned row, int cls, const double (&m)[Q], const double (&k)[Q]) {
        double ax[Q], rr[Q];
        st_time<Q>(kt, L, m, k, ax);
        // upwind coupling on time node 0: (M x_q)(k-1), lane k-1's mass accumulator of node q
        const double up = __shfl_up_sync(0xffffffffu, m[Q - 1], 1);
        const double mp = first ? cv[T] : up;
#pragma unroll
        for (int b = 0; b < Q; ++b) rr[b] = fv[T][b] - ax[b] + (b == 0 ? mp : 0.0);
        const size_t off = (size_t)row * rowbytes;
        if (R_OUT)
#pragma unroll
            for (int b = 0; b < Q; ++b) *reinterpret_cast<double *>(rb + off + b * bstride) = rr[b];
        if (Z_OUT) {
            double D[Q * Q], Di[Q * Q];
            st_row_block<Q, FAST>(tab, kt, L, bt, T, cls, D, Di);
#pragma unroll
            for (int b = 0; b < Q; ++b) {
                double acc = 0.0;
#pragma unroll
                for (int a = 0; a < Q; ++a) acc = fma(Di[b * Q + a], rr[a], acc);
                *reinterpret_cast<double *>(zb + off + b * bstride) = omega_s * acc;
            }
        }
        if (NORM)
#pragma unroll
            for (int b = 0; b < Q; ++b) nrm = fma(rr[b], rr[b], nrm);
    }
};

// cpl: the coupling of each chunk's first slab from k_st_coupling ([chunk][row]), or null when there
// is none (a single chunk and the zero initial state)
template <int Q, bool R_OUT, bool Z_OUT, bool NORM, class Tl = StTileRes>
__global__ void __launch_bounds__(32 * Tl::Warps, 1)
k_st_residual(StGeo g, const __grid_constant__ StencilTab tab, const __grid_constant__ StMaps maps,
              const double *__restrict__ cpl, const double *__restrict__ tau, const double *__restrict__ f,
              double *__restrict__ r, double *__restrict__ z, double omega_s, KT kt, double *__restrict__ partial) {
    extern __shared__ __align__(128) unsigned char st_dyn[];
    StSmem<Q, Tl> &sm = *reinterpret_cast<StSmem<Q, Tl> *>(st_dyn + ((128u - (st_smem_addr(st_dyn) & 127u)) & 127u));
    __shared__ StBlockTab<Q> bt;
    const int chunk = blockIdx.x / g.n_tiles, tile = blockIdx.x - chunk * g.n_tiles;
    StLane<Q> L;
    st_lane<Q>(kt, tau, chunk, L);
    st_block_table<Q>(tab, kt, L, bt);            // (the march's first barrier publishes it)
    const unsigned rowbytes = (unsigned)(8u * Q * g.S);
    const size_t lane_off = (size_t)L.k * 8;
    StResOp<Q, R_OUT, Z_OUT, NORM> op{tab, kt, L, bt, reinterpret_cast<const char *>(f) + lane_off,
                                           reinterpret_cast<char *>(r) + lane_off,
                                           reinterpret_cast<char *>(z) + lane_off, rowbytes, (size_t)g.S * 8, omega_s,
                                           (threadIdx.x & 31) == 0,
                                           cpl ? cpl + (size_t)chunk * (g.Ex + g.Ey + (size_t)(g.nx + 1) * (g.ny + 1) * g.nz)
                                               : nullptr,
                                           0.0, {}, {}};
    st_march<Q, Tl, false>(g, tab, maps, sm, tile, chunk, op);
    if (NORM) {
        __shared__ double sh[Tl::Warps];
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
    const StBlockTab<Q> &bt;
    const char *rb;
    char *ob;
    unsigned rowbytes;
    size_t bstride;
    double omega_s, omega;
    double *bsl;                    // LAST: x_q of this lane's slab for the next chunk's coupling (lane 31), or null
    double zv[3][Q], rv[3][Q], xv[3][Q];
    __device__ __forceinline__ void pre(int T, unsigned row, const double *own) {
        const size_t off = (size_t)row * rowbytes;
#pragma unroll
        for (int b = 0; b < Q; ++b) {
            zv[T][b] = own[b * kStSPW];                     // staged z of the row (level s-1)
            if (!RECON) rv[T][b] = __ldg(reinterpret_cast<const double *>(rb + off + b * bstride));
            if (LAST) xv[T][b] = *reinterpret_cast<const double *>(ob + off + b * bstride);
        }
    }
    template <bool FAST>
    __device__ __forceinline__ void emit(int T, unsigned row, int cls, const double (&m)[Q], const double (&k)[Q]) {
        double D[Q * Q], Di[Q * Q], az[Q], d[Q];
        st_row_block<Q, FAST>(tab, kt, L, bt, T, cls, D, Di);
        st_time<Q>(kt, L, m, k, az);
        // RECON: r = D z / omega_s, so z + omega_s D^{-1} (r - A z) = 2 z - omega_s D^{-1} A z (no
        // division, D itself unused); otherwise d = r - A z with r read
#pragma unroll
        for (int b = 0; b < Q; ++b) d[b] = RECON ? az[b] : rv[T][b] - az[b];
        const size_t off = (size_t)row * rowbytes;
#pragma unroll
        for (int b = 0; b < Q; ++b) {
            double y = 0.0;
#pragma unroll
            for (int a = 0; a < Q; ++a) y = fma(Di[b * Q + a], d[a], y);
            const double res = RECON ? fma(-omega_s, y, 2.0 * zv[T][b]) : fma(omega_s, y, zv[T][b]);
            double *o = reinterpret_cast<double *>(ob + off + b * bstride);
            if (LAST) {
                const double xn = fma(omega, res, xv[T][b]);
                *o = xn;
                if (b == Q - 1 && bsl) bsl[row] = xn;       // the chunk's last slab (lane 31 only)
            } else {
                *o = res;
            }
        }
    }
};

template <int Q, bool LAST, bool RECON, class Tl = StTileSweep>
__global__ void __launch_bounds__(32 * Tl::Warps, 1)
k_st_sweep(StGeo g, const __grid_constant__ StencilTab tab, const __grid_constant__ StMaps maps,
           const double *__restrict__ tau, const double *__restrict__ r, double *out, double omega_s, double omega,
           KT kt, double *__restrict__ bslab) {
    extern __shared__ __align__(128) unsigned char st_dyn[];
    StSmem<Q, Tl> &sm = *reinterpret_cast<StSmem<Q, Tl> *>(st_dyn + ((128u - (st_smem_addr(st_dyn) & 127u)) & 127u));
    __shared__ StBlockTab<Q> bt;
    const int chunk = blockIdx.x / g.n_tiles, tile = blockIdx.x - chunk * g.n_tiles;
    StLane<Q> L;
    st_lane<Q>(kt, tau, chunk, L);
    st_block_table<Q>(tab, kt, L, bt);
    const unsigned rowbytes = (unsigned)(8u * Q * g.S);
    const size_t lane_off = (size_t)L.k * 8;
    // LAST: lane 31 holds the slab before chunk + 1; it records x_q there for that chunk's coupling
    // (bslab[(chunk + 1) * n_edges + row], the layout of k_st_bslab)
    const size_t n_edges = (size_t)g.Ex + g.Ey + (size_t)(g.nx + 1) * (g.ny + 1) * g.nz;
    double *bsl = (LAST && bslab && (threadIdx.x & 31) == 31 && chunk + 1 < g.n_chunks)
                      ? bslab + (size_t)(chunk + 1) * n_edges : nullptr;
    StSweepOp<Q, LAST, RECON> op{tab, kt, L, bt, reinterpret_cast<const char *>(r) + lane_off,
                                 reinterpret_cast<char *>(out) + lane_off, rowbytes, (size_t)g.S * 8, omega_s, omega,
                                 bsl, {}, {}, {}};
    st_march<Q, Tl, true>(g, tab, maps, sm, tile, chunk, op);
}

// Mass form of the nodal residual's edge pass (Eq. (5); R17):
// u = f - (Ct (x) M) x + (Nt (x) M) x_{k-1}, so that G^T u = G^T (f - L x) because K G = 0 (the
// curl-curl part of L x lies in the kernel of G^T).  The march with the curl-curl FMAs compiled out:
// 15 of the 21 inputs and ~60 of the ~290 FMAs per node-level.
template <int Q>
struct StResMassOp {
    const KT &kt;
    const char *fb;
    char *ub;
    unsigned rowbytes;
    size_t bstride;
    bool first;
    const double *cpl;
    double fv[3][Q], cv[3];
    __device__ __forceinline__ void pre(int T, unsigned row, const double *) {
        const char *p = fb + (size_t)row * rowbytes;
#pragma unroll
        for (int b = 0; b < Q; ++b) fv[T][b] = __ldg(reinterpret_cast<const double *>(p + b * bstride));
        cv[T] = first && cpl ? __ldg(cpl + row) : 0.0;
    }
    template <bool FAST>
    __device__ __forceinline__ void emit(int T, unsigned row, int, const double (&m)[Q], const double (&)[Q]) {
        const double up = __shfl_up_sync(0xffffffffu, m[Q - 1], 1);
        const double mp = first ? cv[T] : up;
        const size_t off = (size_t)row * rowbytes;
#pragma unroll
        for (int b = 0; b < Q; ++b) {
            double acc = fv[T][b] + (b == 0 ? mp : 0.0);
#pragma unroll
            for (int a = 0; a < Q; ++a) acc = fma(-kt.Ct[b * Q + a], m[a], acc);
            *reinterpret_cast<double *>(ub + off + b * bstride) = acc;
        }
    }
};

template <int Q, class Tl = StTileMass>
__global__ void __launch_bounds__(32 * Tl::Warps, 1)
k_st_res_mass(StGeo g, const __grid_constant__ StencilTab tab, const __grid_constant__ StMaps maps,
              const double *__restrict__ cpl, const double *__restrict__ f, double *__restrict__ u, KT kt) {
    extern __shared__ __align__(128) unsigned char st_dyn[];
    StSmem<Q, Tl> &sm = *reinterpret_cast<StSmem<Q, Tl> *>(st_dyn + ((128u - (st_smem_addr(st_dyn) & 127u)) & 127u));
    const int chunk = blockIdx.x / g.n_tiles, tile = blockIdx.x - chunk * g.n_tiles;
    const unsigned rowbytes = (unsigned)(8u * Q * g.S);
    const size_t lane_off = ((size_t)chunk * kStSPW + (threadIdx.x & 31)) * 8;
    StResMassOp<Q> op{kt, reinterpret_cast<const char *>(f) + lane_off, reinterpret_cast<char *>(u) + lane_off,
                      rowbytes, (size_t)g.S * 8, (threadIdx.x & 31) == 0,
                      cpl ? cpl + (size_t)chunk * (g.Ex + g.Ey + (size_t)(g.nx + 1) * (g.ny + 1) * g.nz) : nullptr,
                      {}, {}};
    st_march<Q, Tl, false, StResMassOp<Q>, false>(g, tab, maps, sm, tile, chunk, op);
}

// The upwind coupling of each chunk's first slab (N_t = e_0 e_q^T): (M x_q) of the
// slab before the chunk (chunk c >= 1: slab 32c - 1; chunk 0: the previous rank's end values `prev`,
// or nothing), out[c * n_edges + row].  The values x_q(32c - 1) come from a compact [chunk][row]
// array b: written as a side output by the kernels that last wrote x (the stencil sweep, the G
// update, the prolongation: api.cpp tracks for which x it is current), else copied by k_st_bslab
// (one strided 8-byte read per value).  k_st_coupling applies the 9-slot mass ELL to it.
template <int Q>
__global__ void __launch_bounds__(256) k_st_bslab(int n_edges, int S, int n_chunks, const double *__restrict__ x,
                                                   double *__restrict__ b) {
    const long long id = (long long)n_edges + blockIdx.x * (long long)blockDim.x + threadIdx.x;   // chunks >= 1
    if (id >= (long long)n_edges * n_chunks) return;
    const int c = (int)(id / n_edges), row = (int)(id - (long long)c * n_edges);
    b[id] = __ldg(x + (size_t)row * Q * S + (size_t)(Q - 1) * S + (size_t)c * kStSPW - 1);
}

// one thread per row: the 9-slot mass ELL row is read once into registers, then applied to every
// chunk's slice of b (the warp's 32 consecutive rows gather neighbouring columns: coalesced); a
// thread per (row, chunk) re-streams the ELL once per chunk (measured 0.35 vs ~0.1 ms per c4 launch)
__global__ void __launch_bounds__(256) k_st_coupling(int n_edges, int n_chunks, DevELL M, const double *__restrict__ b,
                                                      const double *__restrict__ prev, double *__restrict__ out) {
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n_edges) return;
    constexpr int W = 9;                        // uniform-hex mass stencil (checked by the launcher)
    double v[W];
    int col[W];
    const Ent *e = M.e + (size_t)row * M.width;
#pragma unroll
    for (int s = 0; s < W; ++s) {
        if (s < M.width) ld_ent(e + s, v[s], col[s]);
        else { v[s] = 0.0; col[s] = row; }
    }
    for (int c = 0; c < n_chunks; ++c) {
        const double *src = c == 0 ? prev : b + (size_t)c * n_edges;
        double acc = 0.0;
        if (src)
#pragma unroll
            for (int s = 0; s < W; ++s) acc = fma(v[s], __ldg(src + col[s]), acc);
        out[(size_t)c * n_edges + row] = acc;
    }
}
