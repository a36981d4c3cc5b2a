// kernels.cu — sm_100a fp64 kernels of the space-time V-cycle.
//
// Layout: every space-time vector is v[row][a][k] with the slab
// index k contiguous.  Edge-row kernels map one thread to one (row, slab):
// consecutive lanes of a warp own consecutive slabs of the same row, so the
// ELL column/value loads of that row are warp-broadcast, every vector load is
// a coalesced 256-byte segment, and the upwind trace x[col][q][k-1] of the
// previous slab is the neighbouring lane's element (L1 hit).
//
// Operators:
//   residual       r = f - L x, (L x)_k = (Ct(x)M + tau_k Mt(x)K) x_k - Nt(x)M x_{k-1}   l.51-77
//   smoother S     x += omega * B r, B = nu_s damped block-Jacobi sweeps on A_k            Eq.(2) l.79-82
//   correction A   x += G Sigma_t Bn G^T r, Bn = nu_n Jacobi sweeps on K_n                 Eq.(5) l.180-188
//   transfers      R = P^T, P = P_t (x) P_edge                                            l.84, l.93-109
// The nodal time basis makes Nt = e_0 e_q^T (only time node 0 of slab k sees the
// end value of slab k-1) and (Ct^{-1} e_0)_q = 1, checked in setup (R2).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "internal.h"
#include "march.cuh"

namespace st {

// ------------------------------------------------------------ variant log
// Which kernel instantiations / code paths have run in this process (st_kernel_variants): lets
// the parity tests prove that the paths the bench takes (4 slabs per lane, several slab chunks
// per row, multi-chunk Sigma_t carries, ...) were the ones compared with the oracle.
static const char *const kVariantNames[] = {
    "residual/dict", "residual/plain", "residual/plain-fold", "residual/spl1", "residual/spl2",
    "residual/chunked", "sweep/dict", "sweep/plain", "sweep/spl1", "sweep/spl2", "sweep/spl4",
    "sweep/chunked", "res_mass/spl1", "res_mass/spl2", "res_mass/spl4", "res_mass/chunked",
    "gtr/fused", "gtr/chunked", "gt/two-pass", "node_scan/multichunk", "node_scan/carry-in",
    "march/residual", "march/sweep", "restrict/space", "prolong/space", "stencil/residual",
    "stencil/sweep", "stencil/res_mass", "coupling/prev", "stencil/node_scan", "coupling/side-output"};
constexpr int kNumVariants = (int)(sizeof(kVariantNames) / sizeof(kVariantNames[0]));
static std::atomic<unsigned long long> g_variants{0};
static inline void note(int bit) { g_variants.fetch_or(1ull << bit, std::memory_order_relaxed); }
enum VariantBit {
    V_RES_DICT, V_RES_PLAIN, V_RES_FOLD, V_RES_SPL1, V_RES_SPL2, V_RES_CHUNKED, V_SWEEP_DICT, V_SWEEP_PLAIN,
    V_SWEEP_SPL1, V_SWEEP_SPL2, V_SWEEP_SPL4, V_SWEEP_CHUNKED, V_RM_SPL1, V_RM_SPL2, V_RM_SPL4, V_RM_CHUNKED,
    V_GTR_FUSED, V_GTR_CHUNKED, V_GT_TWOPASS, V_SCAN_MULTI, V_SCAN_CARRY, V_MARCH_RES, V_MARCH_SWEEP,
    V_RESTRICT_SPACE, V_PROLONG_SPACE, V_STENCIL_RES, V_STENCIL_SWEEP, V_STENCIL_RM, V_COUPLING_PREV,
    V_SN_SCAN, V_BSLAB_SIDE
};
unsigned long long variants(bool reset) {
    return reset ? g_variants.exchange(0) : g_variants.load();
}
const char *variant_name(int bit) { return bit >= 0 && bit < kNumVariants ? kVariantNames[bit] : nullptr; }

KT make_kt(const TimeMats &tm) {
    KT k{};
    for (int i = 0; i < kMaxQ * kMaxQ; ++i) { k.Ct[i] = tm.Ct[i]; k.Mt[i] = tm.Mt[i]; k.Ctinv[i] = tm.Ctinv[i]; }
    for (int i = 0; i < kMaxQ; ++i) k.g[i] = tm.g[i];
    return k;
}

constexpr int kBlock = 256;

// ---------------------------------------------------------------- helpers
// y = D^{-1} v for the (Q x Q) Jacobi block D = Ct*dm + t*Mt*dk (cofactor inverse)
template <int Q>
__device__ __forceinline__ void block_solve(const KT &kt, double dm, double dk, double t, const double *v, double *y) {
    double D[Q * Q];
#pragma unroll
    for (int i = 0; i < Q * Q; ++i) D[i] = kt.Ct[i] * dm + t * kt.Mt[i] * dk;
    if constexpr (Q == 1) {
        y[0] = v[0] / D[0];
    } else if constexpr (Q == 2) {
        const double inv = 1.0 / (D[0] * D[3] - D[1] * D[2]);
        y[0] = (D[3] * v[0] - D[1] * v[1]) * inv;
        y[1] = (D[0] * v[1] - D[2] * v[0]) * inv;
    } else {
        const double c00 = D[4] * D[8] - D[5] * D[7], c01 = D[5] * D[6] - D[3] * D[8], c02 = D[3] * D[7] - D[4] * D[6];
        const double inv = 1.0 / (D[0] * c00 + D[1] * c01 + D[2] * c02);
        const double B[9] = {c00, D[2] * D[7] - D[1] * D[8], D[1] * D[5] - D[2] * D[4],
                             c01, D[0] * D[8] - D[2] * D[6], D[2] * D[3] - D[0] * D[5],
                             c02, D[1] * D[6] - D[0] * D[7], D[0] * D[4] - D[1] * D[3]};
#pragma unroll
        for (int i = 0; i < 3; ++i) y[i] = (B[3 * i] * v[0] + B[3 * i + 1] * v[1] + B[3 * i + 2] * v[2]) * inv;
    }
}

template <int Q>
__device__ __forceinline__ void block_mul(const KT &kt, double dm, double dk, double t, const double *v, double *y) {
#pragma unroll
    for (int b = 0; b < Q; ++b) {
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < Q; ++a) acc += (kt.Ct[b * Q + a] * dm + t * kt.Mt[b * Q + a] * dk) * v[a];
        y[b] = acc;
    }
}

__device__ __forceinline__ double block_reduce_sum(double v, double *sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    v = 0.0;
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        v = lane < nw ? sh[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    }
    return v;
}

// Thread mapping of the row kernels: LPR lanes cover one row,
// each lane SPL (= 2 when S is even) consecutive slabs via 16-byte loads; a warp
// covers 32/LPR rows, a CTA 8 warps.  Blocks are ordered slab-chunk-major so
// the CTAs resident at any moment work on the same chunk of LPR*SPL slabs of
// neighbouring rows: the x rows they gather stay in L2 (working set ~ 3 planes
// of rows x one chunk instead of 3 planes x all slabs).
struct Map {
    int rows, S, spl, lpr_log2, rpw, rows_per_cta, n_rowblocks, chunk, n_chunks;
};

__device__ __forceinline__ bool map_thread(const Map &m, int &row, int &k0) {
    const int chunk = blockIdx.x / m.n_rowblocks;
    const int rb = blockIdx.x - chunk * m.n_rowblocks;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    row = rb * m.rows_per_cta + warp * m.rpw + (lane >> m.lpr_log2);
    k0 = chunk * m.chunk + (lane & ((1 << m.lpr_log2) - 1)) * m.spl;
    return row < m.rows && k0 < m.S;
}

// Box-scheduled mapping: CTA = (slab chunk, node box); its warps
// loop over the box's rows (sched[bptr[b] .. bptr[b+1])), LPR lanes per row,
// SPL slabs per lane.  Rows of one box share most of their ELL columns, so a
// column's x chunk is fetched from L2 once per CTA and re-read from L1.
struct BoxMap {
    int S, spl, lpr_log2, rpw, chunk, n_boxes, n_chunks, box_major;
    const int *sched, *bptr;
};

// Warp-uniform loop: every lane runs the same number of iterations (so row-group
// shuffles are safe); lanes without work get valid = false, a clamped in-bounds
// row/slab, and must not store.
template <class F>
__device__ __forceinline__ void box_loop(const BoxMap &m, F &&body) {
    int chunk, b;
    if (m.box_major) { b = blockIdx.x / m.n_chunks; chunk = blockIdx.x - b * m.n_chunks; }
    else { chunk = blockIdx.x / m.n_boxes; b = blockIdx.x - chunk * m.n_boxes; }
    const int beg = __ldg(m.bptr + b), end = __ldg(m.bptr + b + 1);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int k0 = chunk * m.chunk + (lane & ((1 << m.lpr_log2) - 1)) * m.spl;
    const bool kval = k0 < m.S;
    const int step = (blockDim.x >> 5) * m.rpw;
    for (int ib = beg + warp * m.rpw; ib < end; ib += step) {
        const int i = ib + (lane >> m.lpr_log2);
        const bool valid = kval && i < end;
        body(__ldg(m.sched + (i < end ? i : beg)), kval ? k0 : 0, valid);
    }
}

__device__ __forceinline__ void ld_ent(const Ent *p, double &v, int &c) {
    const double2 t = __ldg(reinterpret_cast<const double2 *>(p));
    v = t.x;
    c = (int)(unsigned long long)__double_as_longlong(t.y);
}

template <int SPL>
__device__ __forceinline__ void ldv(const double *__restrict__ p, double *v) {
    if constexpr (SPL == 4) {
        const double2 t0 = __ldg(reinterpret_cast<const double2 *>(p));
        const double2 t1 = __ldg(reinterpret_cast<const double2 *>(p) + 1);
        v[0] = t0.x; v[1] = t0.y; v[2] = t1.x; v[3] = t1.y;
    } else if constexpr (SPL == 2) {
        const double2 t = __ldg(reinterpret_cast<const double2 *>(p));
        v[0] = t.x; v[1] = t.y;
    } else {
        v[0] = __ldg(p);
    }
}

template <int SPL>
__device__ __forceinline__ void ldv_rw(const double *p, double *v) {   // data this kernel also writes
    if constexpr (SPL == 4) {
        const double2 t0 = *reinterpret_cast<const double2 *>(p);
        const double2 t1 = *(reinterpret_cast<const double2 *>(p) + 1);
        v[0] = t0.x; v[1] = t0.y; v[2] = t1.x; v[3] = t1.y;
    } else if constexpr (SPL == 2) {
        const double2 t = *reinterpret_cast<const double2 *>(p);
        v[0] = t.x; v[1] = t.y;
    } else {
        v[0] = *p;
    }
}

template <int SPL>
__device__ __forceinline__ void stv(double *p, const double *v) {
    if constexpr (SPL == 4) {
        reinterpret_cast<double2 *>(p)[0] = make_double2(v[0], v[1]);
        reinterpret_cast<double2 *>(p)[1] = make_double2(v[2], v[3]);
    } else if constexpr (SPL == 2) *reinterpret_cast<double2 *>(p) = make_double2(v[0], v[1]);
    else p[0] = v[0];
}

// Merged M/K ELL: one column list, (M value, K value) pairs; one gather feeds both products.
// Dictionary form (levels whose operator has at most kTabSize distinct (M, K) pairs, e.g.
// uniform meshes with piecewise-constant coefficients): entry = col << 8 | value id, rows padded
// to a multiple of 4 entries and read 4 at a time, values from the constant bank (warp-uniform
// index: served by the constant cache, not the L1 data pipe that bounds these kernels).
struct MKELL {
    const int *col;
    const double2 *val;
    int width;
    const unsigned *pk = nullptr;
    int tab = 0;
};

constexpr int kTabSize = 256, kTabSlots = 14;
#ifndef ST_DICT_UNROLL
#define ST_DICT_UNROLL 9
#endif
constexpr int kDictUnroll = ST_DICT_UNROLL;   // batches of 4 dictionary entries unrolled
#ifndef ST_SWEEP_MINB
#define ST_SWEEP_MINB 3
#endif
__constant__ double2 c_mk_tab[kTabSize * kTabSlots];

template <int Q, int SPL>
__device__ __forceinline__ void mk_fma(const double2 v, const double *__restrict__ xc, int S,
                                       double (&mx)[Q][SPL], double (&kx)[Q][SPL]) {
#pragma unroll
    for (int a = 0; a < Q; ++a) {
        double xv[SPL];
        ldv<SPL>(xc + a * S, xv);
#pragma unroll
        for (int j = 0; j < SPL; ++j) {
            mx[a][j] = fma(v.x, xv[j], mx[a][j]);
            kx[a][j] = fma(v.y, xv[j], kx[a][j]);
        }
    }
}

template <int Q, int SPL, int W, bool DICT = false, bool FOLD = false>
__device__ __forceinline__ void spatial_apply_mk(const MKELL &A, int row, int k0, int S,
                                                 const double *__restrict__ x,
                                                 double (&mx)[Q][SPL], double (&kx)[Q][SPL],
                                                 const double *cp = nullptr, bool cp_prev = false,
                                                 double *mp0 = nullptr) {
    const size_t QS = (size_t)Q * S;
#pragma unroll
    for (int a = 0; a < Q; ++a)
#pragma unroll
        for (int j = 0; j < SPL; ++j) { mx[a][j] = 0.0; kx[a][j] = 0.0; }
    if (DICT) {
        static_assert(!DICT || W > 0, "dictionary ELL needs a compile-time width");
        constexpr int W4 = (W + 3) / 4 * 4;
        const uint4 *pp = reinterpret_cast<const uint4 *>(A.pk + (size_t)row * W4);
#pragma unroll (kDictUnroll)
        for (int s0 = 0; s0 < W; s0 += 4) {
            const uint4 e4 = __ldg(pp + s0 / 4);
            const unsigned es[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (s0 + t < W) {
                    const double2 v = c_mk_tab[A.tab + (es[t] & 255u)];
                    mk_fma<Q, SPL>(v, x + (size_t)(es[t] >> 8) * QS + k0, S, mx, kx);
                }
        }
        return;
    }
    const int w = W > 0 ? W : A.width;
    const int *cc = A.col + (size_t)row * w;
    const double2 *vv = A.val + (size_t)row * w;
#pragma unroll (W > 0 ? W : 3)
    for (int s = 0; s < w; ++s) {
        const int c = __ldg(cc + s);
        const double2 v = __ldg(vv + s);
        mk_fma<Q, SPL>(v, x + (size_t)c * QS + k0, S, mx, kx);
        // FOLD (M and K share one 33-slot pattern, e.g. jittered hexes): the first lane of a row
        // group also gathers x_q of the slab before its chunk for the upwind coupling here, so
        // its 33 loads overlap the merged gathers instead of forming a serial tail
        if (FOLD && cp) *mp0 = fma(v.x, __ldg(cp + (cp_prev ? (size_t)c : (size_t)c * QS)), *mp0);
    }
}

// Upwind coupling (Nt (x) M) x_{k-1} = e_0 (M x)[q][k-1]: the previous slab's M-image
// is the own lane's (j >= 1) or the previous lane's (j = 0) already computed mx[q];
// only the first lane of a row group (k0 at a chunk start) gathers it explicitly.
template <int Q, int SPL, int WM>
__device__ __forceinline__ void coupling(const DevELL &M, int row, int k0, int S, int lpr,
                                         const double *__restrict__ x, const double *__restrict__ prev,
                                         const double (&mx)[Q][SPL], double (&mp)[SPL]) {
#pragma unroll
    for (int j = 1; j < SPL; ++j) mp[j] = mx[Q - 1][j - 1];
    const double up = __shfl_up_sync(0xffffffffu, mx[Q - 1][SPL - 1], 1, lpr);
    const int lane_in_row = (threadIdx.x & 31) & (lpr - 1);
    if (lane_in_row != 0) {
        mp[0] = up;
    } else {
        double acc = 0.0;
        const int wm = WM > 0 ? WM : M.width;
        const Ent *eM = M.e + (size_t)row * wm;
        if (k0 > 0) {
            for (int s = 0; s < wm; ++s) {
                double v; int c;
                ld_ent(eM + s, v, c);
                acc = fma(v, __ldg(x + (size_t)c * Q * S + (Q - 1) * S + k0 - 1), acc);
            }
        } else if (prev) {
            for (int s = 0; s < wm; ++s) {
                double v; int c;
                ld_ent(eM + s, v, c);
                acc = fma(v, __ldg(prev + c), acc);
            }
        }
        mp[0] = acc;
    }
}

// ------------------------------------------------------------ residual
// r = f - L x; optionally z = omega_s D^{-1} r (first Jacobi sweep of B from zero)
// and per-block partial sums of |r|^2.
template <int Q, int SPL, int WM, int WK, bool R_OUT, bool Z_OUT, bool NORM, bool COUPLE = true, bool DICT = false>
__global__ void __launch_bounds__(kBlock, DICT ? 4 : 0) k_residual(BoxMap m, DevELL M, MKELL MK, const double *__restrict__ tau,
                                                     const double *__restrict__ x, const double *__restrict__ f,
                                                     const double *__restrict__ prev, double *__restrict__ r,
                                                     double *__restrict__ z, const double *__restrict__ dM,
                                                     const double *__restrict__ dK, double omega_s, KT kt,
                                                     double *__restrict__ partial) {
    double nrm = 0.0;
    box_loop(m, [&](int row, int k0, bool valid) {
        const int S = m.S;
        double mx[Q][SPL], kx[Q][SPL], mp[SPL];
        constexpr bool FOLD = !DICT && COUPLE && WM == 33 && WK == 33;
        if (FOLD) {
            const int lpr = 1 << m.lpr_log2;
            const bool first = ((threadIdx.x & 31) & (lpr - 1)) == 0;
            const double *cp = !first ? nullptr : k0 > 0 ? x + (size_t)(Q - 1) * S + k0 - 1 : prev;
            double mp0 = 0.0;
            spatial_apply_mk<Q, SPL, WK, false, true>(MK, row, k0, S, x, mx, kx, cp, k0 == 0, &mp0);
#pragma unroll
            for (int j = 1; j < SPL; ++j) mp[j] = mx[Q - 1][j - 1];
            const double up = __shfl_up_sync(0xffffffffu, mx[Q - 1][SPL - 1], 1, lpr);
            mp[0] = first ? mp0 : up;
        } else {
            spatial_apply_mk<Q, SPL, WK, DICT>(MK, row, k0, S, x, mx, kx);
            if (COUPLE) coupling<Q, SPL, WM>(M, row, k0, S, 1 << m.lpr_log2, x, prev, mx, mp);
            else
#pragma unroll
                for (int j = 0; j < SPL; ++j) mp[j] = 0.0;
        }
        if (!valid) return;
        double t[SPL];
        ldv<SPL>(tau + k0, t);
        const size_t base = (size_t)row * Q * S + k0;
        double rr[Q][SPL];
#pragma unroll
        for (int b = 0; b < Q; ++b) {
            double fv[SPL];
            ldv<SPL>(f + base + b * S, fv);
#pragma unroll
            for (int j = 0; j < SPL; ++j) {
                double acc = 0.0;
#pragma unroll
                for (int a = 0; a < Q; ++a) acc += kt.Ct[b * Q + a] * mx[a][j] + t[j] * kt.Mt[b * Q + a] * kx[a][j];
                rr[b][j] = fv[j] - acc + (b == 0 ? mp[j] : 0.0);
            }
        }
        if (R_OUT)
#pragma unroll
            for (int b = 0; b < Q; ++b) stv<SPL>(r + base + b * S, rr[b]);
        if (Z_OUT) {
            const double dm = __ldg(dM + row), dk = __ldg(dK + row);
            double zz[Q][SPL];
#pragma unroll
            for (int j = 0; j < SPL; ++j) {
                double v[Q], y[Q];
#pragma unroll
                for (int b = 0; b < Q; ++b) v[b] = rr[b][j];
                block_solve<Q>(kt, dm, dk, t[j], v, y);
#pragma unroll
                for (int b = 0; b < Q; ++b) zz[b][j] = omega_s * y[b];
            }
#pragma unroll
            for (int b = 0; b < Q; ++b) stv<SPL>(z + base + b * S, zz[b]);
        }
        if (NORM)
#pragma unroll
            for (int b = 0; b < Q; ++b)
#pragma unroll
                for (int j = 0; j < SPL; ++j) nrm += rr[b][j] * rr[b][j];
    });
    if (NORM) {
        __shared__ double sh[kBlock / 32];
        const double s = block_reduce_sum(nrm, sh);
        if (threadIdx.x == 0) partial[blockIdx.x] = s;
    }
}

// ------------------------------------------------------ Jacobi sweep on A_k
// znew = z + omega_s D^{-1} (r - A_k z); r read from memory or, for the sweep
// right after the fused first one, reconstructed pointwise as r = D z / omega_s.
// LAST: x += omega * znew (the smoother update of Eq. 2), in place (x is only
// read at its own row).
template <int Q, int SPL, int WM, int WK, bool LAST, bool RECON, bool DICT = false>
__global__ void __launch_bounds__(kBlock, DICT ? ST_SWEEP_MINB : 0) k_sweep(BoxMap m, DevELL M, MKELL MK, const double *__restrict__ tau,
                                                  const double *__restrict__ dM, const double *__restrict__ dK,
                                                  const double *__restrict__ z, const double *__restrict__ r,
                                                  double *out, double omega_s, double omega, KT kt) {
    box_loop(m, [&](int row, int k0, bool valid) {
    const int S = m.S;
    double mz[Q][SPL], kz[Q][SPL];
    spatial_apply_mk<Q, SPL, WK, DICT>(MK, row, k0, S, z, mz, kz);
    if (!valid) return;
    double t[SPL];
    ldv<SPL>(tau + k0, t);
    const double dm = __ldg(dM + row), dk = __ldg(dK + row);
    const size_t base = (size_t)row * Q * S + k0;
    double zr[Q][SPL], rr[Q][SPL], res[Q][SPL];
#pragma unroll
    for (int a = 0; a < Q; ++a) ldv<SPL>(z + base + a * S, zr[a]);
    if (!RECON)
#pragma unroll
        for (int a = 0; a < Q; ++a) ldv<SPL>(r + base + a * S, rr[a]);
#pragma unroll
    for (int j = 0; j < SPL; ++j) {
        double v[Q], rv[Q], d[Q], y[Q];
#pragma unroll
        for (int a = 0; a < Q; ++a) v[a] = zr[a][j];
        if (RECON) {
            block_mul<Q>(kt, dm, dk, t[j], v, rv);
#pragma unroll
            for (int a = 0; a < Q; ++a) rv[a] /= omega_s;
        } else {
#pragma unroll
            for (int a = 0; a < Q; ++a) rv[a] = rr[a][j];
        }
#pragma unroll
        for (int b = 0; b < Q; ++b) {
            double acc = 0.0;
#pragma unroll
            for (int a = 0; a < Q; ++a) acc += kt.Ct[b * Q + a] * mz[a][j] + t[j] * kt.Mt[b * Q + a] * kz[a][j];
            d[b] = rv[b] - acc;
        }
        block_solve<Q>(kt, dm, dk, t[j], d, y);
#pragma unroll
        for (int a = 0; a < Q; ++a) res[a][j] = zr[a][j] + omega_s * y[a];
    }
    if (LAST) {
#pragma unroll
        for (int a = 0; a < Q; ++a) {
            double xv[SPL];
            ldv_rw<SPL>(out + base + a * S, xv);
#pragma unroll
            for (int j = 0; j < SPL; ++j) xv[j] += omega * res[a][j];
            stv<SPL>(out + base + a * S, xv);
        }
    } else {
#pragma unroll
        for (int a = 0; a < Q; ++a) stv<SPL>(out + base + a * S, res[a]);
    }
});
}

template <int Q>
__global__ void __launch_bounds__(kBlock) k_axpy(size_t n, double alpha, const double *__restrict__ z, double *__restrict__ x) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) x[i] += alpha * z[i];
}

// ------------------------------------------------- two-pass nodal residual
// Pass 1 (edge rows): u = f - (Ct (x) M) x + (Nt (x) M) x_prev, the residual without K
// (G^T K = 0, so G^T u = G^T (f - L x): the G^T (f - L x) of Eq. (5)).  Pays off where M is narrow (9 slots on uniform
// hexes against 54 for the node-row G^T M of k_gtr): fewer L1 gathers for one more vector pass.
template <int Q, int SPL, int WM>
__global__ void __launch_bounds__(kBlock, 4) k_res_mass(BoxMap m, DevELL M, const double *__restrict__ x,
                                                     const double *__restrict__ f, const double *__restrict__ prev,
                                                     double *__restrict__ u, KT kt) {
    box_loop(m, [&](int row, int k0, bool valid) {
        const int S = m.S;
        const size_t QS = (size_t)Q * S;
        double mx[Q][SPL], mp[SPL];
#pragma unroll
        for (int a = 0; a < Q; ++a)
#pragma unroll
            for (int j = 0; j < SPL; ++j) mx[a][j] = 0.0;
        const int wm = WM > 0 ? WM : M.width;
        const Ent *eM = M.e + (size_t)row * wm;
#pragma unroll (WM > 0 ? WM : 3)
        for (int s = 0; s < wm; ++s) {
            double v; int c;
            ld_ent(eM + s, v, c);
            const double *xc = x + (size_t)c * QS + k0;
#pragma unroll
            for (int a = 0; a < Q; ++a) {
                double xv[SPL];
                ldv<SPL>(xc + a * S, xv);
#pragma unroll
                for (int j = 0; j < SPL; ++j) mx[a][j] = fma(v, xv[j], mx[a][j]);
            }
        }
        coupling<Q, SPL, WM>(M, row, k0, S, 1 << m.lpr_log2, x, prev, mx, mp);
        if (!valid) return;
        const size_t base = (size_t)row * QS + k0;
#pragma unroll
        for (int b = 0; b < Q; ++b) {
            double fv[SPL], uv[SPL];
            ldv<SPL>(f + base + b * S, fv);
#pragma unroll
            for (int j = 0; j < SPL; ++j) {
                double acc = 0.0;
#pragma unroll
                for (int a = 0; a < Q; ++a) acc += kt.Ct[b * Q + a] * mx[a][j];
                uv[j] = fv[j] - acc + (b == 0 ? mp[j] : 0.0);
            }
            stv<SPL>(u + base + b * S, uv);
        }
    });
}

// Pass 2 (node rows): w = G^T u, zn = omega_n w / d_n (w stored for nu_n > 2)
template <int Q, int SPL, bool W_OUT>
__global__ void __launch_bounds__(kBlock) k_gt(BoxMap m, DevELL GT, const double *__restrict__ u,
                                               const double *__restrict__ dN, double omega_n,
                                               double *__restrict__ zn, double *__restrict__ w) {
    box_loop(m, [&](int node, int k0, bool valid) {
        if (!valid) return;
        const int S = m.S;
        const size_t QS = (size_t)Q * S;
        double g[Q][SPL];
#pragma unroll
        for (int a = 0; a < Q; ++a)
#pragma unroll
            for (int j = 0; j < SPL; ++j) g[a][j] = 0.0;
        const int *gc = GT.col + (size_t)node * GT.width;
        for (int s = 0; s < GT.width; ++s) {
            const int code = __ldg(gc + s);
            if (code < 0) break;
            const double sg = (code & 1) ? -1.0 : 1.0;
            const double *ue = u + (size_t)(code >> 1) * QS + k0;
#pragma unroll
            for (int a = 0; a < Q; ++a) {
                double uv[SPL];
                ldv<SPL>(ue + a * S, uv);
#pragma unroll
                for (int j = 0; j < SPL; ++j) g[a][j] = fma(sg, uv[j], g[a][j]);
            }
        }
        const double inv = omega_n / __ldg(dN + node);
        const size_t base = (size_t)node * QS + k0;
#pragma unroll
        for (int a = 0; a < Q; ++a) {
            double zv[SPL];
#pragma unroll
            for (int j = 0; j < SPL; ++j) zv[j] = g[a][j] * inv;
            stv<SPL>(zn + base + a * S, zv);
            if (W_OUT) stv<SPL>(w + base + a * S, g[a]);
        }
    });
}

// ------------------------------------------------------- nodal correction
// Fused nodal residual (first half of Eq. 5): w = G^T (f - L x) computed per node without the
// edge residual: G^T K = 0, so w = G^T f - sum_a Ct[b][a] (G^T M x_a) + e_0 (G^T M x_q)(k-1);
// zn = omega_n w / d_n is the first Jacobi sweep on K_n (w stored for nu_n > 2).
template <int Q, int SPL, bool W_OUT, bool COUPLE = true, bool CTINV = false>
__global__ void __launch_bounds__(kBlock) k_gtr(BoxMap m, DevELL GT, DevELL GtM, const double *__restrict__ x,
                                                const double *__restrict__ f, const double *__restrict__ prev,
                                                const double *__restrict__ dN, double omega_n, KT kt,
                                                double *__restrict__ zn, double *__restrict__ w) {
    box_loop(m, [&](int node, int k0, bool valid) {
        const int S = m.S;
        const size_t QS = (size_t)Q * S;
        double gm[Q][SPL];
#pragma unroll
        for (int a = 0; a < Q; ++a)
#pragma unroll
            for (int j = 0; j < SPL; ++j) gm[a][j] = 0.0;
        // coupling: (G^T M x_q) at slab k-1 comes from the previous lane of the row group; the
        // first lane gathers it inside the G^T M loop (its loads overlap the main gathers)
        const int lpr = 1 << m.lpr_log2;
        const bool first = ((threadIdx.x & 31) & (lpr - 1)) == 0;
        const double *cp = !(COUPLE && first) ? nullptr : k0 > 0 ? x + (size_t)(Q - 1) * S + k0 - 1 : prev;
        double acc0 = 0.0;
        const Ent *e = GtM.e + (size_t)node * GtM.width;
#pragma unroll 6
        for (int s = 0; s < GtM.width; ++s) {
            double v; int c;
            ld_ent(e + s, v, c);
            const double *xc = x + (size_t)c * QS + k0;
#pragma unroll
            for (int a = 0; a < Q; ++a) {
                double xv[SPL];
                ldv<SPL>(xc + a * S, xv);
#pragma unroll
                for (int j = 0; j < SPL; ++j) gm[a][j] = fma(v, xv[j], gm[a][j]);
            }
            if (cp) acc0 = fma(v, __ldg(cp + (k0 > 0 ? (size_t)c * QS : (size_t)c)), acc0);
        }
        double mp[SPL];
#pragma unroll
        for (int j = 1; j < SPL; ++j) mp[j] = COUPLE ? gm[Q - 1][j - 1] : 0.0;
        const double up = __shfl_up_sync(0xffffffffu, gm[Q - 1][SPL - 1], 1, lpr);
        mp[0] = !COUPLE ? 0.0 : first ? acc0 : up;
        if (!valid) return;
        double gf[Q][SPL];
#pragma unroll
        for (int a = 0; a < Q; ++a)
#pragma unroll
            for (int j = 0; j < SPL; ++j) gf[a][j] = 0.0;
        const int *gc = GT.col + (size_t)node * GT.width;
        for (int s = 0; s < GT.width; ++s) {
            const int code = __ldg(gc + s);
            if (code < 0) break;
            const double sg = (code & 1) ? -1.0 : 1.0;
            const double *fe = f + (size_t)(code >> 1) * QS + k0;
#pragma unroll
            for (int a = 0; a < Q; ++a) {
                double fv[SPL];
                ldv<SPL>(fe + a * S, fv);
#pragma unroll
                for (int j = 0; j < SPL; ++j) gf[a][j] = fma(sg, fv[j], gf[a][j]);
            }
        }
        const double inv = omega_n / __ldg(dN + node);
        const size_t base = (size_t)node * QS + k0;
        double wv[Q][SPL];
#pragma unroll
        for (int b = 0; b < Q; ++b)
#pragma unroll
            for (int j = 0; j < SPL; ++j) {
                double acc = 0.0;
#pragma unroll
                for (int a = 0; a < Q; ++a) acc += kt.Ct[b * Q + a] * gm[a][j];
                wv[b][j] = gf[b][j] - acc + (b == 0 ? mp[j] : 0.0);
            }
#pragma unroll
        for (int b = 0; b < Q; ++b) {
            double zv[SPL];
#pragma unroll
            for (int j = 0; j < SPL; ++j) {
                double v = wv[b][j];
                if (CTINV) {   // inner hybrid smoother: y = omega_n Ct^{-1} w / d_n (R13)
                    v = 0.0;
#pragma unroll
                    for (int a = 0; a < Q; ++a) v += kt.Ctinv[b * Q + a] * wv[a][j];
                }
                zv[j] = v * inv;
            }
            stv<SPL>(zn + base + b * S, zv);
            if (W_OUT) stv<SPL>(w + base + b * S, wv[b]);
        }
    });
}

// middle nodal sweep: zout = z + omega_n (w - K_n z)/dN
template <int Q, int SPL>
__global__ void __launch_bounds__(kBlock) k_node_sweep(BoxMap m, DevELL Kn, const double *__restrict__ dN,
                                                       const double *__restrict__ z, const double *__restrict__ w,
                                                       double omega_n, double *__restrict__ zout) {
    box_loop(m, [&](int node, int k0, bool valid) {
    if (!valid) return;
    const int S = m.S;
    double kz[Q][SPL];
#pragma unroll
    for (int a = 0; a < Q; ++a)
#pragma unroll
        for (int j = 0; j < SPL; ++j) kz[a][j] = 0.0;
    const Ent *en = Kn.e + (size_t)node * Kn.width;
    for (int s = 0; s < Kn.width; ++s) {
        double v; int c;
        ld_ent(en + s, v, c);
        const double *zc = z + (size_t)c * Q * S + k0;
#pragma unroll
        for (int a = 0; a < Q; ++a) {
            double zv[SPL];
            ldv<SPL>(zc + a * S, zv);
#pragma unroll
            for (int j = 0; j < SPL; ++j) kz[a][j] = fma(v, zv[j], kz[a][j]);
        }
    }
    const double d = __ldg(dN + node);
    const size_t base = (size_t)node * Q * S + k0;
#pragma unroll
    for (int a = 0; a < Q; ++a) {
        double zv[SPL], wv[SPL];
        ldv<SPL>(z + base + a * S, zv);
        ldv<SPL>(w + base + a * S, wv);
#pragma unroll
        for (int j = 0; j < SPL; ++j) zv[j] = zv[j] + omega_n * (wv[j] - kz[a][j]) / d;
        stv<SPL>(zout + base + a * S, zv);
    }
});
}

// Last nodal step fused with the time integration Sigma_t (R2): one warp per
// node row walks the slabs in chunks of 32*SPL; per slab
//   z2 = z + omega_n (w - K_n z)/dN          (MODE 1: w = dN z/omega_n; MODE 2: w read; MODE 0: z2 = z)
//   s_k = (Ct^{-1} z2)_q,  e_k = carry + sum_{j<=k} s_j   (lane-local pair + warp inclusive scan)
//   y_k = Ct^{-1} z2 + g e_{k-1},  g = Ct^{-1} e_0
// tot (optional) receives the row's e_{S-1} (rank carry for multi-GPU slabs).
template <int Q, int SPL, int MODE, int KW = 0>
__global__ void __launch_bounds__(kBlock) k_node_scan(int nodes, int S, DevELL Kn, const double *__restrict__ dN,
                                                      const double *__restrict__ z, const double *__restrict__ w,
                                                      double omega_n, KT kt, const double *__restrict__ carry_in,
                                                      double *__restrict__ y, double *__restrict__ tot) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= nodes) return;
    const int node = warp;
    const double d = __ldg(dN + node);
    const size_t base = (size_t)node * Q * S;
    double carry = carry_in ? __ldg(carry_in + node) : 0.0;
    const Ent *en = Kn.e + (size_t)node * Kn.width;
    for (int kc = 0; kc < S; kc += 32 * SPL) {
        const int k0 = kc + lane * SPL;
        const bool valid = k0 < S;
        double z2[Q][SPL];
#pragma unroll
        for (int a = 0; a < Q; ++a)
#pragma unroll
            for (int j = 0; j < SPL; ++j) z2[a][j] = 0.0;
        if (valid) {
            double zr[Q][SPL];
#pragma unroll
            for (int a = 0; a < Q; ++a) ldv<SPL>(z + base + a * S + k0, zr[a]);
            if (MODE == 0) {
#pragma unroll
                for (int a = 0; a < Q; ++a)
#pragma unroll
                    for (int j = 0; j < SPL; ++j) z2[a][j] = zr[a][j];
            } else {
                double kz[Q][SPL];
#pragma unroll
                for (int a = 0; a < Q; ++a)
#pragma unroll
                    for (int j = 0; j < SPL; ++j) kz[a][j] = 0.0;
                const int kw = KW > 0 ? KW : Kn.width;
#pragma unroll (KW > 0 ? KW : 1)
                for (int s = 0; s < kw; ++s) {
                    double v; int c;
                    ld_ent(en + s, v, c);
                    const double *zc = z + (size_t)c * Q * S + k0;
#pragma unroll
                    for (int a = 0; a < Q; ++a) {
                        double zv[SPL];
                        ldv<SPL>(zc + a * S, zv);
#pragma unroll
                        for (int j = 0; j < SPL; ++j) kz[a][j] = fma(v, zv[j], kz[a][j]);
                    }
                }
#pragma unroll
                for (int a = 0; a < Q; ++a) {
                    double wv[SPL];
                    if (MODE == 2) ldv<SPL>(w + base + a * S + k0, wv);
#pragma unroll
                    for (int j = 0; j < SPL; ++j) {
                        const double wa = MODE == 1 ? d * zr[a][j] / omega_n : wv[j];
                        z2[a][j] = zr[a][j] + omega_n * (wa - kz[a][j]) / d;
                    }
                }
            }
        }
        double u[Q][SPL], sl[SPL];
#pragma unroll
        for (int j = 0; j < SPL; ++j) {
#pragma unroll
            for (int a = 0; a < Q; ++a) {
                double acc = 0.0;
#pragma unroll
                for (int b = 0; b < Q; ++b) acc += kt.Ctinv[a * Q + b] * z2[b][j];
                u[a][j] = acc;
            }
            sl[j] = u[Q - 1][j];
        }
        double lsum = 0.0;
#pragma unroll
        for (int j = 0; j < SPL; ++j) lsum += sl[j];
        double incl = lsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double tt = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += tt;
        }
        double e = carry + incl - lsum;     // end value before this lane's first slab
        if (valid) {
            double out[Q][SPL];
#pragma unroll
            for (int j = 0; j < SPL; ++j) {
#pragma unroll
                for (int a = 0; a < Q; ++a) out[a][j] = u[a][j] + kt.g[a] * e;
                e += sl[j];
            }
#pragma unroll
            for (int a = 0; a < Q; ++a) stv<SPL>(y + base + a * S + k0, out[a]);
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (tot && lane == 0) tot[node] = carry;
}

// x += G (y + g carry) : x[e][a][k] += y[end][a][k] - y[start][a][k] + g_a (carry[end] - carry[start])
// (carry: integrated end value before this slab block, R2; null = 0)
template <int Q, int SPL>
__global__ void __launch_bounds__(kBlock) k_g_update(BoxMap m, const int *__restrict__ en, const double *__restrict__ y,
                                                     const double *__restrict__ carry, const double *__restrict__ cc,
                                                     int n_nodes, KT kt, double *__restrict__ x, double *__restrict__ bslab,
                                                     int n_edges) {
    box_loop(m, [&](int e, int k0, bool valid) {
    if (!valid) return;
    const int S = m.S;
    const int n0 = __ldg(en + 2 * e), n1 = __ldg(en + 2 * e + 1);
    const size_t QS = (size_t)Q * S;
    double dc = carry ? __ldg(carry + n1) - __ldg(carry + n0) : 0.0;
    if (cc) {       // chunk carries of the structured node scan (32-slab chunks; a lane's slabs share one)
        const double *c = cc + (size_t)(k0 / 32) * n_nodes;        // kStSPW = 32 (stencil.cuh)
        dc += __ldg(c + n1) - __ldg(c + n0);
    }
#pragma unroll
    for (int a = 0; a < Q; ++a) {
        double y0[SPL], y1[SPL], xv[SPL];
        ldv<SPL>(y + n0 * QS + a * S + k0, y0);
        ldv<SPL>(y + n1 * QS + a * S + k0, y1);
        ldv_rw<SPL>(x + e * QS + a * S + k0, xv);
#pragma unroll
        for (int j = 0; j < SPL; ++j) xv[j] += y1[j] - y0[j] + kt.g[a] * dc;
        stv<SPL>(x + e * QS + a * S + k0, xv);
        // side output: x_q of the last slab of a 32-slab chunk, for the next chunk's coupling
        if (bslab && a == Q - 1 && (k0 + SPL) % 32 == 0 && k0 + SPL < S)
            bslab[(size_t)((k0 + SPL) / 32) * n_edges + e] = xv[SPL - 1];
    }
});
}

// strided slab copy between space-time vectors with the same rows and Q:
// dst[row][a][dk0 + s] (+)= src[row][a][sk0 + s], s < ns
__global__ void __launch_bounds__(kBlock) k_copy_slabs(int rows, int Q, int ns, double *__restrict__ dst, int dS, int dk0,
                                                       const double *__restrict__ src, int sS, int sk0, int add) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= (long long)rows * Q * ns) return;
    const int s = (int)(i % ns);
    const long long ra = i / ns;
    const int a = (int)(ra % Q), row = (int)(ra / Q);
    const double v = src[((long long)row * Q + a) * sS + sk0 + s];
    double *d = dst + ((long long)row * Q + a) * dS + dk0 + s;
    *d = add ? *d + v : v;
}

// out[row] = x[row][q][S-1] (the trace handed to the next rank)
__global__ void __launch_bounds__(kBlock) k_end_values(int rows, int Q, int S, const double *__restrict__ x,
                                                       double *__restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < rows) out[i] = x[((long long)i * Q + Q - 1) * S + S - 1];
}

// ------------------------------------------------ pencil march (uniform hex levels)
// Grid: blocks ordered slab-chunk-major; block = 4 warps = 4 consecutive pencils (j, k)
// of one slab chunk.  Lane = (slab, time node a) with a fastest (Q = 1 or 2 lanes per
// slab), so every thread carries the march window of ONE time node; the time-matrix
// combination exchanges the partner lane's images with shfl_xor.  HALO (residual): the
// first slab of the warp is the slab before the chunk, whose mass image of time node q
// feeds the next slab's upwind coupling by a shuffle; chunk stride = 32/Q - 1 slabs.
struct MarchMap {
    int S, n_pencils, n_pblocks, stride;
};
constexpr int kMarchWarps = 4;

template <int Q, bool HALO>
__device__ __forceinline__ void march_coords(const MarchMap &mm, const Grid3 &g, int &j, int &k, int &ks, int &a,
                                             bool &out_ok, bool &pencil_ok) {
    const int chunk = blockIdx.x / mm.n_pblocks;
    const int pb = blockIdx.x - chunk * mm.n_pblocks;
    const int p = pb * kMarchWarps + (threadIdx.x >> 5);
    pencil_ok = p < mm.n_pencils;
    const int pp = pencil_ok ? p : 0;
    j = pp % (g.ny + 1);
    k = pp / (g.ny + 1);
    const int lane = threadIdx.x & 31;
    a = lane % Q;
    const int sl = lane / Q;
    ks = chunk * mm.stride + sl - (HALO ? 1 : 0);
    out_ok = (HALO ? sl >= 1 : true) && ks < mm.S;
    if (ks >= mm.S) ks = mm.S - 1;
}

// the (Q x Q) time combination for the lane's own test index b = a:
//   (A x)_b = sum_a' Ct[b][a'] M_a' + t Mt[b][a'] K_a'   with M_a', K_a' of the partner lanes
template <int Q>
__device__ __forceinline__ double time_combine(const KT &kt, int b, double t, double mimg, double kimg) {
    double acc = 0.0;
#pragma unroll
    for (int ap = 0; ap < Q; ++ap) {
        const double mo = Q == 1 ? mimg : __shfl_sync(0xffffffffu, mimg, ((threadIdx.x & 31) & ~(Q - 1)) + ap);
        const double ko = Q == 1 ? kimg : __shfl_sync(0xffffffffu, kimg, ((threadIdx.x & 31) & ~(Q - 1)) + ap);
        acc += kt.Ct[b * Q + ap] * mo + t * kt.Mt[b * Q + ap] * ko;
    }
    return acc;
}

// y_b = (D^{-1} v)_b for the lane's own b, D = Ct dm + t Mt dk, v spread over the Q lanes of a slab
template <int Q>
__device__ __forceinline__ double block_solve_lanes(const KT &kt, int b, double dm, double dk, double t, double vb) {
    double v[Q], y[Q];
#pragma unroll
    for (int ap = 0; ap < Q; ++ap)
        v[ap] = Q == 1 ? vb : __shfl_sync(0xffffffffu, vb, ((threadIdx.x & 31) & ~(Q - 1)) + ap);
    block_solve<Q>(kt, dm, dk, t, v, y);
    double out = y[0];
#pragma unroll
    for (int ap = 1; ap < Q; ++ap)
        if (b == ap) out = y[ap];
    return out;
}

template <int Q>
__device__ __forceinline__ double block_mul_lanes(const KT &kt, int b, double dm, double dk, double t, double vb) {
    double v[Q], y[Q];
#pragma unroll
    for (int ap = 0; ap < Q; ++ap)
        v[ap] = Q == 1 ? vb : __shfl_sync(0xffffffffu, vb, ((threadIdx.x & 31) & ~(Q - 1)) + ap);
    block_mul<Q>(kt, dm, dk, t, v, y);
    double out = y[0];
#pragma unroll
    for (int ap = 1; ap < Q; ++ap)
        if (b == ap) out = y[ap];
    return out;
}

template <int Q, bool R_OUT, bool Z_OUT, bool NORM>
__global__ void __launch_bounds__(32 * kMarchWarps, 3) k_res_march(MarchMap mm, Grid3 g, const double *__restrict__ tau,
                                                                const double *__restrict__ x,
                                                                const double *__restrict__ f,
                                                                const double *__restrict__ prev, double *__restrict__ r,
                                                                double *__restrict__ z, const double *__restrict__ dM,
                                                                const double *__restrict__ dK, double omega_s, KT kt,
                                                                double *__restrict__ partial) {
    int j, k, ks, a;
    bool out_ok, pencil_ok;
    march_coords<Q, true>(mm, g, j, k, ks, a, out_ok, pencil_ok);
    double nrm = 0.0;
    if (pencil_ok) {
        const int S = mm.S, QS = Q * S;
        const Lane ln{x, prev, S, QS, ks, Q - 1};
        const double t = ks >= 0 ? __ldg(tau + ks) : 0.0;
        Win w;
        win_init(g, ln, a, j, k, w);
        StepLoads cur, nxt;
        load_step(g, ln, a, 0, j, k, cur);
        for (int i = 0; i <= g.nx; ++i) {
            if (i < g.nx) load_step(g, ln, a, i + 1, j, k, nxt);   // software pipeline: next step's gathers in flight
            Cells c;
            load_cells2(g, i, j, k, c);
            double o[6];
            step(g, c, cur, w, o);
            cur = nxt;
#pragma unroll
            for (int e = 0; e < 3; ++e) {
                const bool exists = e == 0 ? i < g.nx : (e == 1 ? j < g.ny : k < g.nz);   // warp-uniform
                if (!exists) continue;
                // upwind coupling: time node 0 of slab ks takes the mass image of node q of slab ks-1
                const double mp = __shfl_up_sync(0xffffffffu, o[e], 1);
                const double ax = time_combine<Q>(kt, a, t, o[e], o[3 + e]);
                const int row = e == 0 ? xid(g, i, j, k) : (e == 1 ? yid(g, i, j, k) : zid(g, i, j, k));
                const size_t idx = (size_t)row * QS + a * S + ks;
                // (the halo lane of chunk 0 has ks = -1: never touch f there)
                const double rr = (out_ok ? __ldg(f + idx) : 0.0) - ax + (a == 0 ? mp : 0.0);
                if (R_OUT && out_ok) r[idx] = rr;
                if (Z_OUT) {
                    const double y = block_solve_lanes<Q>(kt, a, __ldg(dM + row), __ldg(dK + row), t, rr);
                    if (out_ok) z[idx] = omega_s * y;
                }
                if (NORM && out_ok) nrm += rr * rr;
            }
        }
    }
    if (NORM) {
        __shared__ double sh[kMarchWarps];
        const double s = block_reduce_sum(nrm, sh);
        if (threadIdx.x == 0) partial[blockIdx.x] = s;
    }
}

// Jacobi sweep on A_k with the march: znew = z + omega_s D^{-1}(r - A_k z), r = D z / omega_s
// (RECON) or read; LAST: x += omega znew, else out = znew.
template <int Q, bool LAST, bool RECON>
__global__ void __launch_bounds__(32 * kMarchWarps, 3) k_sweep_march(MarchMap mm, Grid3 g, const double *__restrict__ tau,
                                                                  const double *__restrict__ dM,
                                                                  const double *__restrict__ dK,
                                                                  const double *__restrict__ z,
                                                                  const double *__restrict__ r, double *out,
                                                                  double omega_s, double omega, KT kt) {
    int j, k, ks, a;
    bool out_ok, pencil_ok;
    march_coords<Q, false>(mm, g, j, k, ks, a, out_ok, pencil_ok);
    if (!pencil_ok) return;
    const int S = mm.S, QS = Q * S;
    const Lane ln{z, nullptr, S, QS, ks, Q - 1};
    const double t = __ldg(tau + ks);
    Win w;
    win_init(g, ln, a, j, k, w);
    StepLoads cur, nxt;
    load_step(g, ln, a, 0, j, k, cur);
    for (int i = 0; i <= g.nx; ++i) {
        if (i < g.nx) load_step(g, ln, a, i + 1, j, k, nxt);
        Cells c;
        load_cells2(g, i, j, k, c);
        double o[6];
        step(g, c, cur, w, o);
        cur = nxt;
#pragma unroll
        for (int e = 0; e < 3; ++e) {
            const bool exists = e == 0 ? i < g.nx : (e == 1 ? j < g.ny : k < g.nz);
            if (!exists) continue;
            const int row = e == 0 ? xid(g, i, j, k) : (e == 1 ? yid(g, i, j, k) : zid(g, i, j, k));
            const size_t idx = (size_t)row * QS + a * S + ks;
            const double dm = __ldg(dM + row), dk = __ldg(dK + row);
            const double zr = z[idx];
            const double rv = RECON ? block_mul_lanes<Q>(kt, a, dm, dk, t, zr) / omega_s : __ldg(r + idx);
            const double d = rv - time_combine<Q>(kt, a, t, o[e], o[3 + e]);
            const double y = block_solve_lanes<Q>(kt, a, dm, dk, t, d);
            if (!out_ok) continue;
            if (LAST) out[idx] += omega * (zr + omega_s * y);
            else out[idx] = zr + omega_s * y;
        }
    }
}

// ------------------------------------------------------------- transfers
// Restriction: fc[rc][a][K] = sum_{(rf,w) in R_s row rc} w * sum_{j,b} Pt_K[(j Q + b)][a] r[rf][b][2K+j]
// one thread per (coarse row, coarse slab K); the fine slab pair (2K, 2K+1) is one 16-byte load.
// space-only restriction / prolongation of the inner spatial V-cycle (R13, the
// approximation of A_k^{-1} in Eq. (2)): same slabs
template <int Q, bool PROLONG>
__global__ void __launch_bounds__(kBlock) k_space_transfer(Map m, DevELL T, const double *__restrict__ in,
                                                           double *__restrict__ out) {
    int row, k;
    if (!map_thread(m, row, k)) return;
    const int S = m.S;
    double acc[Q];
#pragma unroll
    for (int a = 0; a < Q; ++a) acc[a] = 0.0;
    for (int s = 0; s < T.width; ++s) {
        double wgt; int c;
        ld_ent(T.e + (size_t)row * T.width + s, wgt, c);
        const double *src = in + (size_t)c * Q * S + k;
#pragma unroll
        for (int a = 0; a < Q; ++a) acc[a] = fma(wgt, __ldg(src + a * S), acc[a]);
    }
    const size_t base = (size_t)row * Q * S + k;
#pragma unroll
    for (int a = 0; a < Q; ++a) {
        if (PROLONG) out[base + a * S] += acc[a];
        else out[base + a * S] = acc[a];
    }
}

// z = omega D^{-1} r (the first block-Jacobi sweep from zero), pointwise
template <int Q>
__global__ void __launch_bounds__(kBlock) k_jacobi_point(Map m, const double *__restrict__ tau,
                                                         const double *__restrict__ dM, const double *__restrict__ dK,
                                                         const double *__restrict__ r, double *__restrict__ z,
                                                         double omega, KT kt) {
    int row, k;
    if (!map_thread(m, row, k)) return;
    const int S = m.S;
    const size_t base = (size_t)row * Q * S + k;
    double v[Q], y[Q];
#pragma unroll
    for (int a = 0; a < Q; ++a) v[a] = __ldg(r + base + a * S);
    block_solve<Q>(kt, __ldg(dM + row), __ldg(dK + row), __ldg(tau + k), v, y);
#pragma unroll
    for (int a = 0; a < Q; ++a) z[base + a * S] = omega * y[a];
}

// The (2Q x Q) time matrices of the CTA's coarse slabs (one slab chunk, <= 32 slabs) staged in shared
// memory as Ps[entry][slab]: every lane reads its own slab's entries conflict-free, instead of 2Q^2
// loads per thread that each span 32 x 64 bytes (the L1 wavefronts of those loads bounded k_prolong)
template <int Q>
__device__ __forceinline__ void stage_pt(const Map &m, const double *__restrict__ Pt, double (*Ps)[32]) {
    constexpr int N = 2 * Q * Q;
    const int K0 = (blockIdx.x / m.n_rowblocks) * m.chunk;
    for (int t = threadIdx.x; t < N * m.chunk; t += blockDim.x) {
        const int kk = t / N, idx = t - kk * N;
        if (K0 + kk < m.S) Ps[idx][kk] = __ldg(Pt + (size_t)(K0 + kk) * N + idx);
    }
    __syncthreads();
}

template <int Q, bool SPACE>
__global__ void __launch_bounds__(kBlock) k_restrict(Map m, DevELL Rg, const double *__restrict__ r,
                                                     const double *__restrict__ Pt, double *__restrict__ fc) {
    __shared__ double Ps[2 * Q * Q][32];
    stage_pt<Q>(m, Pt, Ps);
    int rc, K;
    if (!map_thread(m, rc, K)) return;
    const int Sc = m.S, S = 2 * Sc;
    const int kk = K - (blockIdx.x / m.n_rowblocks) * m.chunk;
    double P[2 * Q * Q];
#pragma unroll
    for (int i = 0; i < 2 * Q * Q; ++i) P[i] = Ps[i][kk];
    double acc[Q];
#pragma unroll
    for (int a = 0; a < Q; ++a) acc[a] = 0.0;
    const int width = SPACE ? Rg.width : 1;
    for (int s = 0; s < width; ++s) {
        double wgt = 1.0;
        int rf = rc;
        if (SPACE) ld_ent(Rg.e + (size_t)rc * Rg.width + s, wgt, rf);
        const double *rr = r + (size_t)rf * Q * S + 2 * K;
        double fv[2 * Q];
#pragma unroll
        for (int b = 0; b < Q; ++b) {
            const double2 t = __ldg(reinterpret_cast<const double2 *>(rr + b * S));
            fv[b] = t.x; fv[Q + b] = t.y;
        }
#pragma unroll
        for (int a = 0; a < Q; ++a) {
            double t = 0.0;
#pragma unroll
            for (int jb = 0; jb < 2 * Q; ++jb) t += P[jb * Q + a] * fv[jb];
            acc[a] = fma(wgt, t, acc[a]);
        }
    }
    const size_t base = (size_t)rc * Q * Sc + K;
#pragma unroll
    for (int a = 0; a < Q; ++a) fc[base + a * Sc] = acc[a];
}

// Prolongation: x[rf][b][2K+j] += sum_a Pt_K[(j Q + b)][a] * sum_{(rc,w) in P_s row rf} w xc[rc][a][K]
// one thread per (fine row, coarse slab K) writing the fine slab pair as one 16-byte store.
template <int Q, bool SPACE>
__global__ void __launch_bounds__(kBlock) k_prolong(Map m, DevELL Pg, const double *__restrict__ xc,
                                                    const double *__restrict__ Pt, double *__restrict__ x,
                                                    double *__restrict__ bslab, int n_edges) {
    __shared__ double Ps[2 * Q * Q][32];
    stage_pt<Q>(m, Pt, Ps);
    int rf, K;
    if (!map_thread(m, rf, K)) return;
    const int kk = K - (blockIdx.x / m.n_rowblocks) * m.chunk;
    const int Sc = m.S, S = 2 * Sc;
    double v[Q];
#pragma unroll
    for (int a = 0; a < Q; ++a) v[a] = 0.0;
    const int width = SPACE ? Pg.width : 1;
    for (int s = 0; s < width; ++s) {
        double wgt = 1.0;
        int rc = rf;
        if (SPACE) ld_ent(Pg.e + (size_t)rf * Pg.width + s, wgt, rc);
        const double *xr = xc + (size_t)rc * Q * Sc + K;
#pragma unroll
        for (int a = 0; a < Q; ++a) v[a] = fma(wgt, __ldg(xr + a * Sc), v[a]);
    }
    const size_t base = (size_t)rf * Q * S + 2 * K;
#pragma unroll
    for (int b = 0; b < Q; ++b) {
        double t0 = 0.0, t1 = 0.0;
#pragma unroll
        for (int a = 0; a < Q; ++a) {
            t0 += Ps[b * Q + a][kk] * v[a];
            t1 += Ps[(Q + b) * Q + a][kk] * v[a];
        }
        double2 *px = reinterpret_cast<double2 *>(x + base + b * S);
        double2 xv = *px;
        xv.x += t0; xv.y += t1;
        *px = xv;
        // side output: x_q of a chunk's last slab (fine slab 2K + 1 = 32c - 1) for the coupling
        if (bslab && b == Q - 1 && (2 * K + 2) % 32 == 0 && 2 * K + 2 < S)
            bslab[(size_t)((2 * K + 2) / 32) * n_edges + rf] = xv.y;
    }
}

// ------------------------------------------------------- coarsest solve
// slab k of the forward substitution x_k = A_k^{-1} (f_k + Nt (x) M x_{k-1}) with
// the dense inverse (index a*n + e); every block rebuilds the right-hand side in
// shared memory, then one warp per output row does the dense row product.
template <int Q>
__global__ void __launch_bounds__(kBlock) k_coarsest(int n, int S, int k, DevELL M, const double *__restrict__ Ainv,
                                                     const double *__restrict__ f, double *__restrict__ x) {
    extern __shared__ double rhs[];
    const int N = Q * n;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int a = i / n, e = i - a * n;
        double v = f[(size_t)e * Q * S + a * S + k];
        if (a == 0 && k > 0) {
            double mp = 0.0;
            for (int s = 0; s < M.width; ++s) {
                const Ent en = M.e[(size_t)e * M.width + s];
                mp = fma(en.v, x[(size_t)en.c * Q * S + (Q - 1) * S + k - 1], mp);
            }
            v += mp;
        }
        rhs[i] = v;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const double *A = Ainv + (size_t)k * N * N;
    for (int i = gw; i < N; i += nw) {
        double acc = 0.0;
        for (int j = lane; j < N; j += 32) acc = fma(__ldg(A + (size_t)i * N + j), rhs[j], acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
        if (lane == 0) {
            const int a = i / n, e = i - a * n;
            x[(size_t)e * Q * S + a * S + k] = acc;
        }
    }
}

__global__ void __launch_bounds__(kBlock) k_norm2(size_t n, const double *__restrict__ v, double *__restrict__ partial) {
    __shared__ double sh[kBlock / 32];
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const double a = i < n ? v[i] : 0.0;
    const double s = block_reduce_sum(a * a, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void __launch_bounds__(1024) k_reduce(int n, const double *__restrict__ partial, double *__restrict__ out) {
    __shared__ double sh[32];
    double v = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) v += partial[i];
    v = block_reduce_sum(v, sh);
    if (threadIdx.x == 0) *out = v;
}

#include "stencil.cuh"
#include "nstencil.cuh"

// --------------------------------------------------------------- launchers
static inline int nblocks(long long work) { return (int)((work + kBlock - 1) / kBlock); }

// launches issued by a launcher beyond the one its caller counts (the stencil coupling pre-pass)
static thread_local int g_extra_launches = 0;
int take_extra_launches() { const int n = g_extra_launches; g_extra_launches = 0; return n; }

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link-time libcuda dependency)
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !ptr)
            throw std::runtime_error("cuTensorMapEncodeTiled not available");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }();
    return fn;
}

// 5-D tiled view (slab, b, i, j, z-level) of one edge block of a space-time vector with S slabs and
// Q time nodes per row; box (bs, bq, bi, bj, 1)
static void encode_block(CUtensorMap *m, const double *base, int S, int Q, int ni, int nj, int nl, int bs, int bq,
                         int bi, int bj) {
    const cuuint64_t rs = (cuuint64_t)Q * S * 8;
    const cuuint64_t dims[5] = {(cuuint64_t)S, (cuuint64_t)Q, (cuuint64_t)ni, (cuuint64_t)nj, (cuuint64_t)nl};
    const cuuint64_t str[4] = {(cuuint64_t)S * 8, rs, rs * ni, rs * ni * nj};
    const cuuint32_t box[5] = {(cuuint32_t)bs, (cuuint32_t)bq, (cuuint32_t)bi, (cuuint32_t)bj, 1};
    const cuuint32_t es[5] = {1, 1, 1, 1, 1};
    const CUresult r = tmap_encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double *>(base), dims, str, box,
                                      es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed");
}

// the three edge blocks of vector v (x-, y-, z-edges) with boxes (bs, bq, tile extents + halo)
template <class Tl>
static void encode_vector(CUtensorMap *mx, CUtensorMap *my, CUtensorMap *mz, const DevLevel &L, const double *v, int S,
                          int Q, int bs, int bq) {
    const Grid3 &G = L.grid;
    const size_t QS = (size_t)Q * S;
    encode_block(mx, v, S, Q, G.nx, G.ny + 1, G.nz + 1, bs, bq, Tl::TI + 1, Tl::TJ + 2);
    encode_block(my, v + (size_t)G.Ex * QS, S, Q, G.nx + 1, G.ny, G.nz + 1, bs, bq, Tl::TI + 2, Tl::TJ + 1);
    encode_block(mz, v + (size_t)(G.Ex + G.Ey) * QS, S, Q, G.nx + 1, G.ny + 1, G.nz, bs, bq, Tl::TI + 2, Tl::TJ + 2);
}

template <int Q, class Tl>
static void stencil_maps(const DevLevel &L, const double *v, StMaps &m) {
    encode_vector<Tl>(&m.x, &m.y, &m.z, L, v, L.S, Q, kStSPW, Q);
}

// opt the stencil kernels into their dynamic shared memory (once per kernel and process)
template <class K>
static void stencil_smem_attr(K kernel, int bytes) {
    static std::mutex mu;
    static std::vector<const void *> done;
    std::lock_guard<std::mutex> lk(mu);
    const void *key = reinterpret_cast<const void *>(kernel);
    for (const void *d : done)
        if (d == key) return;
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess)
        throw std::runtime_error(std::string("stencil smem attribute: ") + cudaGetErrorString(e));
    done.push_back(key);
}

template <class Tl>
static StGeo stencil_geo(const DevLevel &L) {
    StGeo g{};
    g.nx = L.grid.nx; g.ny = L.grid.ny; g.nz = L.grid.nz; g.Ex = L.grid.Ex; g.Ey = L.grid.Ey;
    g.S = L.S;
    g.tiles_i = (g.nx + 1 + Tl::TI - 1) / Tl::TI;
    const int tiles_j = (g.ny + 1 + Tl::TJ - 1) / Tl::TJ;
    g.n_tiles = g.tiles_i * tiles_j;
    g.n_chunks = L.S / kStSPW;
    return g;
}
static inline int grid(const StGeo &g) { return g.n_tiles * g.n_chunks; }

bool stencil_applies(const DevLevel &L, int Q) {
    return L.use_stencil && L.st_tab && (Q == 1 || Q == 2) && L.S % kStSPW == 0;
}

bool bslab_producer(const DevLevel &L, int Q) { return stencil_applies(L, Q) && L.st_bslab; }


static Map make_map(int rows, int S, bool allow_pairs = true) {
    Map m{};
    m.rows = rows;
    m.S = S;
    m.spl = (allow_pairs && S % 2 == 0) ? 2 : 1;
    const int lanes = (S + m.spl - 1) / m.spl;
    int l2 = 0;
    while ((1 << l2) < lanes && l2 < 5) ++l2;
    m.lpr_log2 = l2;
    m.rpw = 32 >> l2;
    m.rows_per_cta = m.rpw * (kBlock / 32);
    m.n_rowblocks = (rows + m.rows_per_cta - 1) / m.rows_per_cta;
    m.chunk = (1 << l2) * m.spl;
    m.n_chunks = (S + m.chunk - 1) / m.chunk;
    return m;
}
static inline int grid(const Map &m) { return m.n_rowblocks * m.n_chunks; }

static BoxMap make_boxmap(int S, const int *sched, const int *bptr, int n_boxes, int max_lpr_log2 = 4, int spl_max = 2) {
    BoxMap m{};
    m.S = S;
    m.spl = (spl_max >= 4 && S % 4 == 0 && S >= 128) ? 4 : (S % 2 == 0 ? 2 : 1);
    const int lanes = (S + m.spl - 1) / m.spl;
    int l2 = 0;
    while ((1 << l2) < lanes && l2 < max_lpr_log2) ++l2;
    m.lpr_log2 = l2;
    m.rpw = 32 >> l2;
    m.chunk = (1 << l2) * m.spl;
    m.n_boxes = n_boxes;
    m.n_chunks = (S + m.chunk - 1) / m.chunk;
    // CTA order: all slab chunks of a box back to back (measured 2% faster than chunk-major);
    // tuning knob ST_BOX_MAJOR=0 restores chunk-major
    static const int order = [] { const char *e = std::getenv("ST_BOX_MAJOR"); return e ? std::atoi(e) : 1; }();
    m.box_major = order;
    m.sched = sched;
    m.bptr = bptr;
    return m;
}
static inline int grid(const BoxMap &m) { return m.n_boxes * ((m.S + m.chunk - 1) / m.chunk); }
static inline BoxMap edge_map(const DevLevel &L, int spl_max = 2) {
    return make_boxmap(L.S, L.sched_e, L.bptr_e, L.nbox_e, L.lpr_log2, spl_max);
}
static inline BoxMap node_map(const DevLevel &L) { return make_boxmap(L.S, L.sched_n, L.bptr_n, L.nbox_n); }

#define ST_DISPATCH_Q(Q, ...)                                   \
    switch (Q) {                                                \
        case 1: { constexpr int QQ = 1; __VA_ARGS__; } break;   \
        case 2: { constexpr int QQ = 2; __VA_ARGS__; } break;   \
        case 3: { constexpr int QQ = 3; __VA_ARGS__; } break;   \
        default: throw std::invalid_argument("Q out of range"); \
    }
#define ST_DISPATCH_Q12(Q, ...)                                 \
    switch (Q) {                                                \
        case 1: { constexpr int QQ = 1; __VA_ARGS__; } break;   \
        case 2: { constexpr int QQ = 2; __VA_ARGS__; } break;   \
        default: throw std::invalid_argument("march: Q <= 2");  \
    }
#define ST_DISPATCH_SPL(spl, ...)                               \
    if (spl == 2) { constexpr int SP = 2; __VA_ARGS__; }        \
    else if (spl == 1) { constexpr int SP = 1; __VA_ARGS__; }   \
    else throw std::logic_error("slabs per lane not instantiated for this kernel");
#define ST_DISPATCH_SPL4(spl, ...)                              \
    if (spl == 4) { constexpr int SP = 4; __VA_ARGS__; }        \
    else if (spl == 2) { constexpr int SP = 2; __VA_ARGS__; }   \
    else if (spl == 1) { constexpr int SP = 1; __VA_ARGS__; }   \
    else throw std::logic_error("slabs per lane not instantiated for this kernel");
// compile-time ELL widths of the common stencils: uniform hexes (9, 33), general hexes
// (33, 33), uniform quads (3, 7), general quads (7, 7); anything else runtime
#define ST_DISPATCH_W(wm, wk, ...)                                                        \
    if (wm == 9 && wk == 33 && MK.pk) { constexpr int WM_ = 9, WK_ = 33; constexpr bool DI_ = true; __VA_ARGS__; } \
    else if (wm == 3 && wk == 7 && MK.pk) { constexpr int WM_ = 3, WK_ = 7; constexpr bool DI_ = true; __VA_ARGS__; } \
    else if (wm == 9 && wk == 33) { constexpr int WM_ = 9, WK_ = 33; constexpr bool DI_ = false; __VA_ARGS__; } \
    else if (wm == 33 && wk == 33) { constexpr int WM_ = 33, WK_ = 33; constexpr bool DI_ = false; __VA_ARGS__; } \
    else if (wm == 3 && wk == 7) { constexpr int WM_ = 3, WK_ = 7; constexpr bool DI_ = false; __VA_ARGS__; } \
    else if (wm == 7 && wk == 7) { constexpr int WM_ = 7, WK_ = 7; constexpr bool DI_ = false; __VA_ARGS__; } \
    else { constexpr int WM_ = 0, WK_ = 0; constexpr bool DI_ = false; __VA_ARGS__; }

static MarchMap march_map(const DevLevel &L, bool halo) {
    MarchMap mm{};
    mm.S = L.S;
    mm.n_pencils = (L.grid.ny + 1) * (L.grid.nz + 1);
    mm.n_pblocks = (mm.n_pencils + kMarchWarps - 1) / kMarchWarps;
    mm.stride = 32 / L.Q - (halo ? 1 : 0);
    return mm;
}
static inline int grid(const MarchMap &mm) { return mm.n_pblocks * ((mm.S + mm.stride - 1) / mm.stride); }

// the upwind coupling of every chunk's first slab (k_st_coupling: 9 mass entries per row and chunk),
// or null: nothing when x = 0 and there is no previous rank; the slab before each chunk from the
// side output of the kernel that last wrote x when api.cpp vouches for it (L.xs), else from k_st_bslab
template <int Q>
static const double *stencil_coupling(Stream st, const DevLevel &L, const StGeo &g, const double *x,
                                      const double *prev) {
    const bool zero = L.xs == XS_ZERO && L.xs_ptr == x;
    if (!((g.n_chunks > 1 && !zero) || prev)) return nullptr;
    const bool have_b = zero || (L.xs == XS_BSLAB && L.xs_ptr == x);
    if (!have_b) {
        const long long nb1 = (long long)L.n_edges * (g.n_chunks - 1);
        if (nb1 > 0) {
            k_st_bslab<Q><<<nblocks(nb1), kBlock, 0, st>>>(L.n_edges, L.S, g.n_chunks, x, L.st_bslab);
            ++g_extra_launches;
        }
    } else {
        note(V_BSLAB_SIDE);
    }
    if (L.M.width > 9) throw std::logic_error("stencil coupling: mass ELL wider than 9");
    k_st_coupling<<<nblocks(L.n_edges), kBlock, 0, st>>>(L.n_edges, g.n_chunks, L.M, zero ? nullptr : L.st_bslab,
                                                         prev, L.st_cpl);
    ++g_extra_launches;
    return L.st_cpl;
}

int launch_residual(Stream st, const DevLevel &L, const KT &kt, int Q, const double *x, const double *f,
                    const double *prev, double *r, double *z, double omega_s, double *partial) {
    if (stencil_applies(L, Q)) {
        note(V_STENCIL_RES);
        if (prev) note(V_COUPLING_PREV);
        using Tl = StTileRes;
        const StGeo g = stencil_geo<Tl>(L);
        const int nb = grid(g), nt = 32 * Tl::Warps;
        const size_t sm = Q == 1 ? sizeof(StSmem<1, Tl>) + 128 : sizeof(StSmem<2, Tl>) + 128;
        ST_DISPATCH_Q12(Q, {
            const double *cpl = stencil_coupling<QQ>(st, L, g, x, prev);
            StMaps maps;
            stencil_maps<QQ, Tl>(L, x, maps);
            auto launch = [&](auto kern) {
                stencil_smem_attr(kern, (int)sm);
                kern<<<nb, nt, sm, st>>>(g, *L.st_tab, maps, cpl, L.tau, f, r, z, omega_s, kt, partial);
            };
            if (partial) {
                if (r) launch(k_st_residual<QQ, true, false, true>);
                else launch(k_st_residual<QQ, false, false, true>);
            } else if (r && z) {
                launch(k_st_residual<QQ, true, true, false>);
            } else if (z) {
                launch(k_st_residual<QQ, false, true, false>);
            } else {
                launch(k_st_residual<QQ, true, false, false>);
            }
        });
        return nb;
    }
    if (L.use_march && Q <= 2) {
        note(V_MARCH_RES);
        const MarchMap mm = march_map(L, true);
        const int g = grid(mm);
        const int nt = 32 * kMarchWarps;
        ST_DISPATCH_Q12(Q, {
            if (partial) {
                if (r) k_res_march<QQ, true, false, true><<<g, nt, 0, st>>>(mm, L.grid, L.tau, x, f, prev, r, z, L.dM, L.dK, omega_s, kt, partial);
                else k_res_march<QQ, false, false, true><<<g, nt, 0, st>>>(mm, L.grid, L.tau, x, f, prev, r, z, L.dM, L.dK, omega_s, kt, partial);
            } else if (r && z) {
                k_res_march<QQ, true, true, false><<<g, nt, 0, st>>>(mm, L.grid, L.tau, x, f, prev, r, z, L.dM, L.dK, omega_s, kt, partial);
            } else if (z) {
                k_res_march<QQ, false, true, false><<<g, nt, 0, st>>>(mm, L.grid, L.tau, x, f, prev, r, z, L.dM, L.dK, omega_s, kt, partial);
            } else {
                k_res_march<QQ, true, false, false><<<g, nt, 0, st>>>(mm, L.grid, L.tau, x, f, prev, r, z, L.dM, L.dK, omega_s, kt, partial);
            }
        });
        return g;
    }
    const BoxMap m = edge_map(L);
    const int g = grid(m);
    const MKELL MK{L.mk_col, L.mk_val, L.mk_width, L.mk_pk, L.mk_tab};
    note(MK.pk && (L.M.width == 9 || L.M.width == 3) ? V_RES_DICT : V_RES_PLAIN);
    if (!MK.pk && L.M.width == 33 && L.mk_width == 33) note(V_RES_FOLD);
    note(m.spl == 2 ? V_RES_SPL2 : V_RES_SPL1);
    if (m.n_chunks > 1) note(V_RES_CHUNKED);
    if (prev) note(V_COUPLING_PREV);
    ST_DISPATCH_Q(Q, ST_DISPATCH_SPL(m.spl, ST_DISPATCH_W(L.M.width, L.mk_width, {
        if (partial) {
            if (r) k_residual<QQ, SP, WM_, WK_, true, false, true, true, DI_><<<g, kBlock, 0, st>>>(m, L.M, MK, L.tau, x, f, prev, r, z, L.dM, L.dK, omega_s, kt, partial);
            else k_residual<QQ, SP, WM_, WK_, false, false, true, true, DI_><<<g, kBlock, 0, st>>>(m, L.M, MK, L.tau, x, f, prev, r, z, L.dM, L.dK, omega_s, kt, partial);
        } else if (r && z) {
            k_residual<QQ, SP, WM_, WK_, true, true, false, true, DI_><<<g, kBlock, 0, st>>>(m, L.M, MK, L.tau, x, f, prev, r, z, L.dM, L.dK, omega_s, kt, partial);
        } else if (z) {
            k_residual<QQ, SP, WM_, WK_, false, true, false, true, DI_><<<g, kBlock, 0, st>>>(m, L.M, MK, L.tau, x, f, prev, r, z, L.dM, L.dK, omega_s, kt, partial);
        } else {
            k_residual<QQ, SP, WM_, WK_, true, false, false, true, DI_><<<g, kBlock, 0, st>>>(m, L.M, MK, L.tau, x, f, prev, r, z, L.dM, L.dK, omega_s, kt, partial);
        }
    })));
    return g;
}

int residual_partials(const DevLevel &L) {
    if (stencil_applies(L, L.Q)) return grid(stencil_geo<StTileRes>(L));
    return (L.use_march && L.Q <= 2) ? grid(march_map(L, true)) : grid(edge_map(L));
}

void launch_sweep(Stream st, const DevLevel &L, const KT &kt, int Q, bool last, bool recon, const double *z,
                  const double *r, double *out, double omega_s, double omega) {
    if (stencil_applies(L, Q)) {
        note(V_STENCIL_SWEEP);
        using Tl = StTileSweep;
        const StGeo g = stencil_geo<Tl>(L);
        const int nb = grid(g), nt = 32 * Tl::Warps;
        const size_t sm = Q == 1 ? sizeof(StSmem<1, Tl>) + 128 : sizeof(StSmem<2, Tl>) + 128;
        ST_DISPATCH_Q12(Q, {
            StMaps maps;
            stencil_maps<QQ, Tl>(L, z, maps);
            auto launch = [&](auto kern) {
                stencil_smem_attr(kern, (int)sm);
                kern<<<nb, nt, sm, st>>>(g, *L.st_tab, maps, L.tau, r, out, omega_s, omega, kt,
                                         last ? L.st_bslab : nullptr);
            };
            if (last && recon) launch(k_st_sweep<QQ, true, true>);
            else if (last) launch(k_st_sweep<QQ, true, false>);
            else if (recon) launch(k_st_sweep<QQ, false, true>);
            else launch(k_st_sweep<QQ, false, false>);
        });
        return;
    }
    if (L.use_march && Q <= 2) {
        note(V_MARCH_SWEEP);
        const MarchMap mm = march_map(L, false);
        const int g = grid(mm), nt = 32 * kMarchWarps;
        ST_DISPATCH_Q12(Q, {
            if (last && recon) k_sweep_march<QQ, true, true><<<g, nt, 0, st>>>(mm, L.grid, L.tau, L.dM, L.dK, z, r, out, omega_s, omega, kt);
            else if (last) k_sweep_march<QQ, true, false><<<g, nt, 0, st>>>(mm, L.grid, L.tau, L.dM, L.dK, z, r, out, omega_s, omega, kt);
            else if (recon) k_sweep_march<QQ, false, true><<<g, nt, 0, st>>>(mm, L.grid, L.tau, L.dM, L.dK, z, r, out, omega_s, omega, kt);
            else k_sweep_march<QQ, false, false><<<g, nt, 0, st>>>(mm, L.grid, L.tau, L.dM, L.dK, z, r, out, omega_s, omega, kt);
        });
        return;
    }
    // Plain ELL: 4 slabs per lane (measured faster than 2 for the sweep, not for the residual).
    // Dictionary ELL (stencil levels): 2 slabs per lane, measured 305 vs 354 ms per 5 V-cycles
    // on c4 (the dictionary at 4 slabs per lane, 128 registers, was 13 % slower).
    // Env ST_SWEEP_DICT=0 forces the plain form (measurements).
    static const bool no_dict = std::getenv("ST_SWEEP_DICT") && std::getenv("ST_SWEEP_DICT")[0] == '0';
    const bool dict = L.mk_pk && !no_dict;
    static const int plain_spl = std::getenv("ST_SWEEP_PLAIN_SPL") ? std::atoi(std::getenv("ST_SWEEP_PLAIN_SPL")) : 4;
    const BoxMap m = edge_map(L, dict ? 2 : plain_spl);
    const int g = grid(m);
    const MKELL MK{L.mk_col, L.mk_val, L.mk_width, dict ? L.mk_pk : nullptr, L.mk_tab};
    note(MK.pk && (L.M.width == 9 || L.M.width == 3) ? V_SWEEP_DICT : V_SWEEP_PLAIN);
    note(m.spl == 4 ? V_SWEEP_SPL4 : m.spl == 2 ? V_SWEEP_SPL2 : V_SWEEP_SPL1);
    if (m.n_chunks > 1) note(V_SWEEP_CHUNKED);
    ST_DISPATCH_Q(Q, ST_DISPATCH_SPL4(m.spl, ST_DISPATCH_W(L.M.width, L.mk_width, {
        if (last && recon) k_sweep<QQ, SP, WM_, WK_, true, true, DI_><<<g, kBlock, 0, st>>>(m, L.M, MK, L.tau, L.dM, L.dK, z, r, out, omega_s, omega, kt);
        else if (last) k_sweep<QQ, SP, WM_, WK_, true, false, DI_><<<g, kBlock, 0, st>>>(m, L.M, MK, L.tau, L.dM, L.dK, z, r, out, omega_s, omega, kt);
        else if (recon) k_sweep<QQ, SP, WM_, WK_, false, true, DI_><<<g, kBlock, 0, st>>>(m, L.M, MK, L.tau, L.dM, L.dK, z, r, out, omega_s, omega, kt);
        else k_sweep<QQ, SP, WM_, WK_, false, false, DI_><<<g, kBlock, 0, st>>>(m, L.M, MK, L.tau, L.dM, L.dK, z, r, out, omega_s, omega, kt);
    })));
}

// out[i] = sum_{b < nb} in[b n + i], blocks added in rank order (the Sigma_t carry of R2)
__global__ void __launch_bounds__(kBlock) k_sum_blocks(size_t n, int nb, const double *__restrict__ in,
                                                       double *__restrict__ out) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double acc = 0.0;
    for (int b = 0; b < nb; ++b) acc += in[(size_t)b * n + i];
    out[i] = acc;
}

void launch_sum_blocks(Stream st, size_t n, int nb, const double *in, double *out) {
    if (n) k_sum_blocks<<<nblocks((long long)n), kBlock, 0, st>>>(n, nb, in, out);
}

void launch_axpy(Stream st, size_t n, double alpha, const double *z, double *x) {
    k_axpy<1><<<nblocks((long long)n), kBlock, 0, st>>>(n, alpha, z, x);
}


void launch_gtr(Stream st, const DevLevel &L, const KT &kt, int Q, const double *x, const double *f, const double *prev,
                double omega_n, double *zn, double *w) {
    const BoxMap m = make_boxmap(L.S, L.sched_n, L.bptr_n, L.nbox_n, L.lpr_log2);
    note(V_GTR_FUSED);
    if (m.n_chunks > 1) note(V_GTR_CHUNKED);
    if (prev) note(V_COUPLING_PREV);
    ST_DISPATCH_Q(Q, ST_DISPATCH_SPL(m.spl, {
        if (w) k_gtr<QQ, SP, true><<<grid(m), kBlock, 0, st>>>(m, L.GT, L.GtM, x, f, prev, L.dN, omega_n, kt, zn, w);
        else k_gtr<QQ, SP, false><<<grid(m), kBlock, 0, st>>>(m, L.GT, L.GtM, x, f, prev, L.dN, omega_n, kt, zn, w);
    }));
}

void launch_res_mass(Stream st, const DevLevel &L, const KT &kt, int Q, const double *x, const double *f,
                     const double *prev, double *u) {
    if (stencil_applies(L, Q)) {
        note(V_STENCIL_RM);
        if (prev) note(V_COUPLING_PREV);
        using Tl = StTileMass;
        const StGeo g = stencil_geo<Tl>(L);
        const size_t sm = Q == 1 ? sizeof(StSmem<1, Tl>) + 128 : sizeof(StSmem<2, Tl>) + 128;
        ST_DISPATCH_Q12(Q, {
            const double *cpl = stencil_coupling<QQ>(st, L, g, x, prev);
            StMaps maps;
            stencil_maps<QQ, Tl>(L, x, maps);
            stencil_smem_attr(k_st_res_mass<QQ>, (int)sm);
            k_st_res_mass<QQ><<<grid(g), 32 * Tl::Warps, sm, st>>>(g, *L.st_tab, maps, cpl, f, u, kt);
        });
        return;
    }
    // 4 slabs per lane: measured 68 vs 75 ms per 5 c4 V-cycles at 2 (env ST_RESMASS_SPL)
    static const int spl = std::getenv("ST_RESMASS_SPL") ? std::atoi(std::getenv("ST_RESMASS_SPL")) : 4;
    const BoxMap m = edge_map(L, spl);
    note(m.spl == 4 ? V_RM_SPL4 : m.spl == 2 ? V_RM_SPL2 : V_RM_SPL1);
    if (m.n_chunks > 1) note(V_RM_CHUNKED);
    if (prev) note(V_COUPLING_PREV);
    ST_DISPATCH_Q(Q, ST_DISPATCH_SPL4(m.spl, {
        if (L.M.width == 9) k_res_mass<QQ, SP, 9><<<grid(m), kBlock, 0, st>>>(m, L.M, x, f, prev, u, kt);
        else if (L.M.width == 3) k_res_mass<QQ, SP, 3><<<grid(m), kBlock, 0, st>>>(m, L.M, x, f, prev, u, kt);
        else k_res_mass<QQ, SP, 0><<<grid(m), kBlock, 0, st>>>(m, L.M, x, f, prev, u, kt);
    }));
}

void launch_gt(Stream st, const DevLevel &L, int Q, const double *u, double omega_n, double *zn, double *w) {
    const BoxMap m = make_boxmap(L.S, L.sched_n, L.bptr_n, L.nbox_n, L.lpr_log2);
    note(V_GT_TWOPASS);
    ST_DISPATCH_Q(Q, ST_DISPATCH_SPL(m.spl, {
        if (w) k_gt<QQ, SP, true><<<grid(m), kBlock, 0, st>>>(m, L.GT, u, L.dN, omega_n, zn, w);
        else k_gt<QQ, SP, false><<<grid(m), kBlock, 0, st>>>(m, L.GT, u, L.dN, omega_n, zn, w);
    }));
}

void launch_node_sweep(Stream st, const DevLevel &L, int Q, const double *z, const double *w, double omega_n,
                       double *zout) {
    const BoxMap m = node_map(L);
    ST_DISPATCH_Q(Q, ST_DISPATCH_SPL(m.spl, k_node_sweep<QQ, SP><<<grid(m), kBlock, 0, st>>>(m, L.Kn, L.dN, z, w, omega_n, zout)));
}

static SnGeo sn_geo(const DevLevel &L) {
    SnGeo g{};
    g.nx = L.grid.nx; g.ny = L.grid.ny; g.nz = L.grid.nz;
    g.S = L.S;
    g.tiles_i = (g.nx + 1 + SnTileT::TI - 1) / SnTileT::TI;
    g.n_tiles = g.tiles_i * ((g.ny + 1 + SnTileT::TJ - 1) / SnTileT::TJ);
    g.n_chunks = L.S / kStSPW;
    g.n_nodes = L.n_nodes;
    return g;
}

bool launch_node_scan(Stream st, const DevLevel &L, const KT &kt, int Q, int mode, const double *z,
                      const double *w, double omega_n, const double *carry, double *y, double *tot) {
    if (L.sn_tab && !carry && (mode == 1 || mode == 2) && (Q == 1 || Q == 2) && L.S % kStSPW == 0) {
        // structured node march (nstencil.cuh) + chunk carries
        note(V_SN_SCAN);
        const SnGeo g = sn_geo(L);
        CUtensorMap mz;
        encode_block(&mz, z, L.S, Q, g.nx + 1, g.ny + 1, g.nz + 1, kStSPW, Q, SnTileT::TI + 2, SnTileT::TJ + 2);
        const int nb = g.n_tiles * g.n_chunks, nt = 32 * SnTileT::Warps;
        ST_DISPATCH_Q12(Q, {
            const size_t sm = sizeof(SnSmem<QQ, SnTileT>) + 128;
            auto launch = [&](auto kern) {
                stencil_smem_attr(kern, (int)sm);
                kern<<<nb, nt, sm, st>>>(g, *L.sn_tab, mz, w, omega_n, kt, y, L.sn_ctot);
            };
            if (mode == 1) launch(k_sn_scan<QQ, 1>);
            else launch(k_sn_scan<QQ, 2>);
        });
        k_sn_carry<<<nblocks(L.n_nodes), kBlock, 0, st>>>(L.n_nodes, g.n_chunks, L.sn_ctot, L.sn_cc, tot);
        ++g_extra_launches;
        return true;
    }
    const int g = nblocks((long long)L.n_nodes * 32);
    const int spl = L.S % 2 == 0 ? 2 : 1;
    if (L.S > 32 * spl) note(V_SCAN_MULTI);
    if (carry) note(V_SCAN_CARRY);
    // compile-time K_n widths of the hex (27) and quad (9) node stencils: the gathers of one slab
    // chunk are all in flight at once (measured 1.1 TB/s with the runtime-width loop)
    ST_DISPATCH_Q(Q, ST_DISPATCH_SPL(spl, {
        if (mode == 0) k_node_scan<QQ, SP, 0><<<g, kBlock, 0, st>>>(L.n_nodes, L.S, L.Kn, L.dN, z, w, omega_n, kt, carry, y, tot);
        else if (L.Kn.width == 27) {
            if (mode == 1) k_node_scan<QQ, SP, 1, 27><<<g, kBlock, 0, st>>>(L.n_nodes, L.S, L.Kn, L.dN, z, w, omega_n, kt, carry, y, tot);
            else k_node_scan<QQ, SP, 2, 27><<<g, kBlock, 0, st>>>(L.n_nodes, L.S, L.Kn, L.dN, z, w, omega_n, kt, carry, y, tot);
        } else if (L.Kn.width == 9) {
            if (mode == 1) k_node_scan<QQ, SP, 1, 9><<<g, kBlock, 0, st>>>(L.n_nodes, L.S, L.Kn, L.dN, z, w, omega_n, kt, carry, y, tot);
            else k_node_scan<QQ, SP, 2, 9><<<g, kBlock, 0, st>>>(L.n_nodes, L.S, L.Kn, L.dN, z, w, omega_n, kt, carry, y, tot);
        } else if (mode == 1) k_node_scan<QQ, SP, 1><<<g, kBlock, 0, st>>>(L.n_nodes, L.S, L.Kn, L.dN, z, w, omega_n, kt, carry, y, tot);
        else k_node_scan<QQ, SP, 2><<<g, kBlock, 0, st>>>(L.n_nodes, L.S, L.Kn, L.dN, z, w, omega_n, kt, carry, y, tot);
    }));
    return false;
}

void launch_g_update(Stream st, const DevLevel &L, const KT &kt, int Q, const double *y, const double *carry,
                     const double *cc, double *x) {
    const BoxMap m = edge_map(L);
    if (cc && (m.chunk % kStSPW != 0 && m.S > m.chunk)) throw std::logic_error("g_update: lane slabs straddle a chunk");
    double *bs = bslab_producer(L, Q) ? L.st_bslab : nullptr;
    ST_DISPATCH_Q(Q, ST_DISPATCH_SPL(m.spl, k_g_update<QQ, SP><<<grid(m), kBlock, 0, st>>>(m, L.edge_nodes, y, carry, cc,
                                                                                            L.n_nodes, kt, x, bs, L.n_edges)));
}

void launch_copy_slabs(Stream st, int rows, int Q, int ns, double *dst, int dS, int dk0, const double *src, int sS,
                       int sk0, bool add) {
    const long long n = (long long)rows * Q * ns;
    if (n > 0) k_copy_slabs<<<nblocks(n), kBlock, 0, st>>>(rows, Q, ns, dst, dS, dk0, src, sS, sk0, add ? 1 : 0);
}

void launch_end_values(Stream st, int rows, int Q, int S, const double *x, double *out) {
    k_end_values<<<nblocks(rows), kBlock, 0, st>>>(rows, Q, S, x, out);
}

void launch_restrict(Stream st, const DevLevel &F, const DevLevel &C, int Q, const double *r, double *fc) {
    const Map m = make_map(C.n_edges, C.S, false);
    if (F.space_coarsened) note(V_RESTRICT_SPACE);
    ST_DISPATCH_Q(Q, {
        if (F.space_coarsened) k_restrict<QQ, true><<<grid(m), kBlock, 0, st>>>(m, F.Rg, r, F.Pt, fc);
        else k_restrict<QQ, false><<<grid(m), kBlock, 0, st>>>(m, F.Rg, r, F.Pt, fc);
    });
}

void launch_prolong(Stream st, const DevLevel &F, int Q, const double *xc, double *x) {
    const Map m = make_map(F.n_edges, F.S / 2, false);
    if (F.space_coarsened) note(V_PROLONG_SPACE);
    ST_DISPATCH_Q(Q, {
        double *bs = bslab_producer(F, Q) ? F.st_bslab : nullptr;
        if (F.space_coarsened) k_prolong<QQ, true><<<grid(m), kBlock, 0, st>>>(m, F.Pg, xc, F.Pt, x, bs, F.n_edges);
        else k_prolong<QQ, false><<<grid(m), kBlock, 0, st>>>(m, F.Pg, xc, F.Pt, x, bs, F.n_edges);
    });
}

// constant-bank slots for dictionary ELL tables (shared by all handles of the process)
static std::mutex g_tab_mu;
static bool g_tab_used[kTabSlots];

int acquire_mk_table(const double2 *vals, int n) {
    if (n > kTabSize) return -1;
    std::lock_guard<std::mutex> lk(g_tab_mu);
    for (int s = 0; s < kTabSlots; ++s)
        if (!g_tab_used[s]) {
            if (cudaMemcpyToSymbol(c_mk_tab, vals, sizeof(double2) * n, sizeof(double2) * s * kTabSize) != cudaSuccess)
                return -1;
            g_tab_used[s] = true;
            return s * kTabSize;
        }
    return -1;
}

void release_mk_table(int offset) {
    std::lock_guard<std::mutex> lk(g_tab_mu);
    if (offset >= 0 && offset / kTabSize < kTabSlots) g_tab_used[offset / kTabSize] = false;
}

// inner spatial V-cycle pieces (R13)
void launch_residual_local(Stream st, const DevLevel &L, const KT &kt, int Q, const double *z, const double *r,
                           double *d) {
    const BoxMap m = edge_map(L);
    const MKELL MK{L.mk_col, L.mk_val, L.mk_width, L.mk_pk, L.mk_tab};
    ST_DISPATCH_Q(Q, ST_DISPATCH_SPL(m.spl, ST_DISPATCH_W(L.M.width, L.mk_width, {
        k_residual<QQ, SP, WM_, WK_, true, false, false, false, DI_><<<grid(m), kBlock, 0, st>>>(m, L.M, MK, L.tau, z, r, nullptr, d, nullptr, L.dM, L.dK, 0.0, kt, nullptr);
    })));
}

void launch_nodal_step(Stream st, const DevLevel &L, const KT &kt, int Q, const double *r, const double *z,
                       double omega_n, double *y) {
    const BoxMap m = make_boxmap(L.S, L.sched_n, L.bptr_n, L.nbox_n, L.lpr_log2);
    ST_DISPATCH_Q(Q, ST_DISPATCH_SPL(m.spl, {
        k_gtr<QQ, SP, false, false, true><<<grid(m), kBlock, 0, st>>>(m, L.GT, L.GtM, z, r, nullptr, L.dN, omega_n, kt, y, nullptr);
    }));
}

void launch_jacobi_point(Stream st, const DevLevel &L, const KT &kt, int Q, const double *r, double *z, double omega) {
    const Map m = make_map(L.n_edges, L.S, false);
    ST_DISPATCH_Q(Q, k_jacobi_point<QQ><<<grid(m), kBlock, 0, st>>>(m, L.tau, L.dM, L.dK, r, z, omega, kt));
}

void launch_space_transfer(Stream st, const DevLevel &F, const DevLevel &C, int Q, bool prolong, const double *in,
                           double *out) {
    const Map m = make_map(prolong ? F.n_edges : C.n_edges, F.S, false);
    ST_DISPATCH_Q(Q, {
        if (prolong) k_space_transfer<QQ, true><<<grid(m), kBlock, 0, st>>>(m, F.Pg, in, out);
        else k_space_transfer<QQ, false><<<grid(m), kBlock, 0, st>>>(m, F.Rg, in, out);
    });
}

int launch_coarsest(Stream st, const DevLevel &L, int Q, const double *f, double *x) {
    const int N = Q * L.n_edges;
    const int blocks = std::min(148, (N + 7) / 8);
    const size_t smem = sizeof(double) * N;
    for (int k = 0; k < L.S; ++k) {
        ST_DISPATCH_Q(Q, k_coarsest<QQ><<<blocks, kBlock, smem, st>>>(L.n_edges, L.S, k, L.M, L.Ainv, f, x));
    }
    return L.S;
}

int launch_norm2(Stream st, size_t n, const double *v, double *partial) {
    const int g = nblocks((long long)n);
    k_norm2<<<g, kBlock, 0, st>>>(n, v, partial);
    return g;
}

void launch_reduce(Stream st, int n, const double *partial, double *out) {
    k_reduce<<<1, 1024, 0, st>>>(n, partial, out);
}

}  // namespace st
