// nstencil.cuh — structured node march for the last nodal Jacobi sweep of the auxiliary correction
// fused with the time integration Sigma_t (Eq. (5); R2/R4), on the
// same class-uniform hex levels as stencil.cuh (included by kernels.cu after it, inside namespace st).
//
// The nodal operator K_n = G^T M_sigma G of a uniform level is a 27-point node stencil whose
// coefficients depend only on the node's boundary class (each coordinate at 0 / inside / at n:
// 27 classes), so they live in a 5.8 KB kernel-parameter table (NodeTab) and the neighbour of
// every coefficient follows from the node numbering of include/st.h.  A warp marches a pencil of
// nodes (i, j) along z for one 32-slab chunk (lane = slab); the CTA tile's z-levels of the input
// z_n, halo included, are staged in shared memory by 5-D TMA loads (zero fill outside the mesh)
// kSnNB levels ahead (the edge march's scheme; deeper, as a node level is little work).  Per node and slab:
//   z2 = z + omega_n (w - K_n z) / d_n      (MODE 1: w = d_n z / omega_n, i.e. z2 = 2 z - omega_n K_n z / d_n)
//   u  = Ct^{-1} z2,  s = u_q,  y = u + g e_{k-1},  e the prefix sum of s over the slabs
// The prefix sum runs over the 32 slabs of the chunk (warp scan); each chunk's total goes to
// ctot[chunk][node], and the chunk carries (exclusive prefix over the chunks, k_sn_carry) are added
// by the G update (x += G (y + g carry)), so every chunk is independent: no serial walk over the
// slab chunks as in the ELL k_node_scan.
#pragma once

// (NodeTab, kSnClasses / kSnSlots / kSnInterior: internal.h)

struct SnGeo {
    int nx, ny, nz;
    int S, tiles_i, n_tiles, n_chunks, n_nodes;
};

template <int TI_, int TJ_>
struct SnTile {
    static constexpr int TI = TI_, TJ = TJ_, Warps = TI_ * TJ_;
    static constexpr int B = (TI_ + 2) * (TJ_ + 2);     // staged node blocks per level
};
using SnTileT = SnTile<4, 4>;

template <int Q, class Tl>
struct SnCfg {
    static constexpr int Blk = Q * kStSPW;
    static constexpr int Level = Tl::B * Blk;
    static_assert((Level * 8) % 128 == 0, "TMA destinations must stay 128-byte aligned");
};

// staged z-levels in flight: a node level is ~1/10 of an edge level's work, so three levels ahead
// (the edge march's depth) leave the TMA latency exposed (10 % of the issued instructions were the
// mbarrier spin in the ncu capture); 6 x 18 KB still fits two CTAs per SM
#ifndef SN_NB
#define SN_NB 6
#endif
constexpr int kSnNB = SN_NB;

template <int Q, class Tl>
struct alignas(128) SnSmem {
    double buf[kSnNB][SnCfg<Q, Tl>::Level];
    unsigned long long full[kSnNB];
    unsigned done[kSnNB];
};

template <bool FAST>
__device__ __forceinline__ double sn_coef(const NodeTab &tab, int cls, int slot) {
    if (FAST) return tab.c[kSnInterior][slot];
    return tab.c[cls][slot];
}

// push the 3 x 3 node inputs of z-level s into the open rows of levels s-1+d (d = 0, 1, 2)
template <int Q, class Tl, bool FAST>
__device__ __forceinline__ void sn_push(const NodeTab &tab, const double *v, const int (&cls)[3], double (&acc)[3][Q]) {
    constexpr int Blk = Q * kStSPW;
    double in[3][3][Q];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
            for (int q = 0; q < Q; ++q) in[a][b][q] = v[(b * (Tl::TI + 2) + a) * Blk + q * kStSPW];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const double c = sn_coef<FAST>(tab, cls[d], 9 * a + 3 * b + (2 - d));   // dl = 1 - d
#pragma unroll
                for (int q = 0; q < Q; ++q) acc[d][q] = fma(c, in[a][b][q], acc[d][q]);
            }
}

template <int Q, class Tl>
__device__ __forceinline__ void sn_stage(const SnGeo &g, const CUtensorMap *map, SnSmem<Q, Tl> &sm, int s, int i0, int j0,
                                         int k0) {
    constexpr unsigned bytes = SnCfg<Q, Tl>::Level * 8;
    const int nb = s % kSnNB;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    st_mbar_expect(&sm.full[nb], bytes);
    st_tma_5d(sm.buf[nb], map, k0, 0, i0 - 1, j0 - 1, s, &sm.full[nb]);
}

template <int Q, int MODE, class Tl = SnTileT>
__global__ void __launch_bounds__(32 * Tl::Warps, 2)
k_sn_scan(SnGeo g, const __grid_constant__ NodeTab tab, const __grid_constant__ CUtensorMap mapz,
          const double *__restrict__ w, double omega_n, KT kt, double *__restrict__ y,
          double *__restrict__ ctot) {
    using C = SnCfg<Q, Tl>;
    extern __shared__ __align__(128) unsigned char sn_dyn[];
    SnSmem<Q, Tl> &sm = *reinterpret_cast<SnSmem<Q, Tl> *>(sn_dyn + ((128u - (st_smem_addr(sn_dyn) & 127u)) & 127u));
    const int chunk = blockIdx.x / g.n_tiles, tile = blockIdx.x - chunk * g.n_tiles;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i0 = (tile % g.tiles_i) * Tl::TI, j0 = (tile / g.tiles_i) * Tl::TJ;
    const int wi = warp % Tl::TI, wj = warp / Tl::TI;
    const int i = i0 + wi, j = j0 + wj;
    const bool ok = i <= g.nx && j <= g.ny;
    const int k0 = chunk * kStSPW;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int b = 0; b < kSnNB; ++b) { st_mbar_init(&sm.full[b], 1); sm.done[b] = 0; }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int s = 0; s < kSnNB && s <= g.nz; ++s) sn_stage<Q, Tl>(g, &mapz, sm, s, i0, j0, k0);
    double acc[3][Q];
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int q = 0; q < Q; ++q) acc[d][q] = 0.0;
    const int ci = st_cls(i, g.nx), cj = st_cls(j, g.ny);
    const bool inner_pencil = ci == 1 && cj == 1;
    const int ow = (wj * (Tl::TI + 2) + wi) * C::Blk + lane;                        // warp's 3 x 3 input window
    const int oo = ow + C::Blk * ((Tl::TI + 2) + 1);                                 // its own node
    const size_t QS = (size_t)Q * g.S, k = (size_t)k0 + lane;
    for (int s = 0; s <= g.nz + 1; ++s) {
        if (s <= g.nz) {
            const int nb = s % kSnNB;
            st_mbar_wait(&sm.full[nb], (unsigned)((s / kSnNB) & 1));
            if (ok) {
                const double *v = sm.buf[nb] + ow;
                if (inner_pencil && s >= 2 && s <= g.nz - 2) {
                    const int dummy[3] = {0, 0, 0};
                    sn_push<Q, Tl, true>(tab, v, dummy, acc);
                } else {
                    int cls[3];
#pragma unroll
                    for (int d = 0; d < 3; ++d) cls[d] = 9 * ci + 3 * cj + st_cls(s - 1 + d, g.nz);
                    sn_push<Q, Tl, false>(tab, v, cls, acc);
                }
            }
        }
        if (s >= 1 && ok) {
            const int l = s - 1;
            const size_t row = (size_t)i + (size_t)(g.nx + 1) * (j + (size_t)(g.ny + 1) * l);
            const double *own = sm.buf[(s + kSnNB - 1) % kSnNB] + oo;
            const double inv = omega_n * tab.dinv[9 * ci + 3 * cj + st_cls(l, g.nz)];   // omega_n / d_n
            double z2[Q], u[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const double zq = own[q * kStSPW];
                if (MODE == 1) z2[q] = fma(-inv, acc[0][q], 2.0 * zq);
                else z2[q] = fma(inv, __ldg(w + row * QS + q * g.S + k) - acc[0][q], zq);
            }
#pragma unroll
            for (int a = 0; a < Q; ++a) {
                double t = 0.0;
#pragma unroll
                for (int b = 0; b < Q; ++b) t = fma(kt.Ctinv[a * Q + b], z2[b], t);
                u[a] = t;
            }
            const double sl = u[Q - 1];
            double incl = sl;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const double e = incl - sl;                    // integrated value before slab k (in the chunk)
#pragma unroll
            for (int a = 0; a < Q; ++a) y[row * QS + a * g.S + k] = fma(kt.g[a], e, u[a]);
            if (lane == 31) ctot[(size_t)chunk * g.n_nodes + row] = incl;
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            acc[0][q] = acc[1][q];
            acc[1][q] = acc[2][q];
            acc[2][q] = 0.0;
        }
        // last-arriver refill of the buffer of level s-1 (stencil.cuh, st_release)
        if (s >= 1 && s - 1 + kSnNB <= g.nz && st_release<Tl::Warps>(&sm.done[(s - 1) % kSnNB]) && lane == 0)
            sn_stage<Q, Tl>(g, &mapz, sm, s - 1 + kSnNB, i0, j0, k0);
    }
}

// chunk carries: cc[c][node] = sum of the chunk totals before chunk c; tot (optional) = all chunks
// (the rank's block total for the multi-GPU carry, R2)
__global__ void __launch_bounds__(256) k_sn_carry(int n_nodes, int n_chunks, const double *__restrict__ ctot,
                                                   double *__restrict__ cc, double *__restrict__ tot) {
    const int node = blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= n_nodes) return;
    double acc = 0.0;
    for (int c = 0; c < n_chunks; ++c) {
        cc[(size_t)c * n_nodes + node] = acc;
        acc += __ldg(ctot + (size_t)c * n_nodes + node);
    }
    if (tot) tot[node] = acc;
}
