// internal.h — host/device data structures of libst (not part of the C-ABI).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/st.h"

namespace st {

constexpr int kMaxQ = 3;

// dG(q) time matrices, row-major [test b][trial a], plus derived quantities
// used by the kernels (R1/R2).
struct TimeMats {
    int Q;
    double Ct[kMaxQ * kMaxQ], Mt[kMaxQ * kMaxQ], Nt[kMaxQ * kMaxQ];
    double Ctinv[kMaxQ * kMaxQ];
    double g[kMaxQ];        // Ct^{-1} e_0
};

// ELL matrix on the host: width slots per row, row-major [row][slot].
struct HostELL {
    int rows = 0, width = 0;
    std::vector<int> col;
    std::vector<double> val;
};

// packed ELL entry: one 16-byte (warp-broadcast) load per nonzero
struct __attribute__((aligned(16))) Ent {
    double v;
    int c;
    int pad;
};

struct DevELL {
    int rows = 0, width = 0;
    Ent *e = nullptr;       // [row][slot]
    int *col = nullptr;     // only for index-only operators (G^T incidence)
};

struct HostMesh {
    int dim = 3;
    int n[3] = {1, 1, 1};
    int n_nodes = 0, n_edges = 0, n_cells = 0, Ex = 0, Ey = 0;
    std::vector<double> coords;               // n_nodes x dim
    std::vector<int> edge_nodes;              // 2 per edge (start, end)
    std::vector<int> cell_edges;              // 12 (3D) / 4 (2D) per cell, reference order
    std::vector<int> cell_nodes;              // 8 / 4 per cell, a + 2b + 4c
};

struct HostLevel {
    HostMesh mesh;
    std::vector<double> sigma, nu, ratio_min;   // per cell
    std::vector<double> tau;                    // per slab
    HostELL M, K, Kn;
    std::vector<double> dM, dK, dN;             // diagonals
    HostELL GT;                                 // node -> signed incident edges: col = 2*e + (sign<0), -1 pad
    HostELL GtM;                                // G^T M_sigma (nodes x edges): the nodal residual operator
    HostELL MK;                                 // merged pattern of M and K: col, val = M entry, valK = K entry
    std::vector<double> MKk;
    double lambda = 0;                          // Eq. (3) value of this level
    bool space_coarsened = false;               // this -> next
    HostELL Pg;                                 // fine edge -> coarse edges (prolongation rows)
    HostELL Rg;                                 // coarse edge -> fine edges (restriction rows)
    std::vector<double> Pt;                     // per coarse slab: (2Q x Q) time prolongation, row-major
    std::vector<double> Ainv;                   // coarsest only: per slab dense (QN x QN)
    // box schedules: rows ordered by small node boxes (box b = rows sched[bptr[b] .. bptr[b+1]))
    std::vector<int> sched_e, bptr_e, sched_n, bptr_n;
    bool uniform = false;                       // all cells the same axis-aligned box
    double hbox[3] = {0, 0, 0};
};

// Structured stencil table (stencil.cuh): (M, K) coefficients per edge direction T, boundary class
// (3 x 3: the two transverse coordinates at 0 / inside / at n) and structural slot (33).  Passed to
// the kernels by value (kernel parameter space, 14256 bytes).
constexpr int kStClasses = 9, kStSlots = 33;
struct StencilTab {
    double2 c[3][kStClasses][kStSlots];
};
bool build_stencil_tab(const HostLevel &L, StencilTab &tab);   // false: the level is not class-uniform

// Structured node stencil table (nstencil.cuh): the 27 K_n coefficients of a node per boundary class
// (each coordinate at 0 / inside / at n: class 9 ci + 3 cj + cl), slot 9 (di + 1) + 3 (dj + 1) + (dl + 1);
// kernel parameter space (5832 bytes).
constexpr int kSnClasses = 27, kSnSlots = 27, kSnInterior = 13;
struct NodeTab {
    double c[kSnClasses][kSnSlots];
    double dinv[kSnClasses];        // 1 / the class's diagonal (the Jacobi divisor d_n)
};
bool build_node_tab(const HostLevel &L, NodeTab &tab);         // false: K_n is not class-uniform

// Slot numbering of the stencil table: for a row of direction T at node p, neighbour edge of
// direction T2 at node p + (o0, o1, o2); block of T2 == T: o_T = 0, the other two offsets in
// {-1,0,1} (9 slots); T2 != T: o_T in {0,1}, o_T2 in {-1,0}, the third in {-1,0,1} (12 slots);
// blocks ordered T2 = 0, 1, 2.
__host__ __device__ constexpr int st_slot(int T, int T2, int o0, int o1, int o2) {
    // block start (blocks of the directions before T2), then the position inside the block
    return ((T2 > 0 ? (T == 0 ? 9 : 12) : 0) + (T2 > 1 ? (T == 1 ? 9 : 12) : 0)) +
           (T2 == T
                ? (T == 0 ? (o1 + 1) * 3 + (o2 + 1) : T == 1 ? (o0 + 1) * 3 + (o2 + 1) : (o0 + 1) * 3 + (o1 + 1))
                : ((T == 0 ? o0 : T == 1 ? o1 : o2) * 6 + ((T2 == 0 ? o0 : T2 == 1 ? o1 : o2) + 1) * 3 +
                   ((3 - T - T2 == 0 ? o0 : 3 - T - T2 == 1 ? o1 : o2) + 1)));
}

// boundary class of a coordinate v in [0, n]: 0 at 0, 2 at n, 1 inside
__host__ __device__ __forceinline__ int st_cls(int v, int n) { return v <= 0 ? 0 : (v >= n ? 2 : 1); }


// uniform axis-aligned hex level for the matrix-free pencil march (march.cuh)
struct Grid3 {
    int nx, ny, nz, Ex, Ey;
    double mx, my, mz;
    double wx, wy, wz;
    const double *sigma, *nu;
};

enum XState { XS_UNKNOWN = 0, XS_ZERO = 1, XS_BSLAB = 2 };

struct DevLevel {
    int n_edges = 0, n_nodes = 0, S = 0, Q = 1;
    DevELL M, K, Kn, GT, Pg, Rg, GtM;
    int mk_width = 0;
    int *mk_col = nullptr;          // [row][slot] union columns of M and K
    double2 *mk_val = nullptr;      // [row][slot] (M value, K value)
    unsigned *mk_pk = nullptr;      // dictionary form: [row][slot (width padded to 4)] col << 8 | value id, or null
    int mk_tab = 0;                 // offset of this level's value table in the constant bank
    double *dM = nullptr, *dK = nullptr, *dN = nullptr;
    int *edge_nodes = nullptr;
    int *sched_e = nullptr, *bptr_e = nullptr, *sched_n = nullptr, *bptr_n = nullptr;
    int nbox_e = 0, nbox_n = 0;
    bool use_march = false;
    bool use_stencil = false;       // structured stencil march (stencil.cuh) for residual and sweep
    StencilTab *st_tab = nullptr;   // host copy of the level's stencil table (owned by the handle)
    double *st_cpl = nullptr;       // [row][chunk] upwind coupling of each 32-slab chunk's first slab
    double *st_bslab = nullptr;     // [row][chunk] x_q of the slab before each chunk (k_st_bslab)
    NodeTab *sn_tab = nullptr;      // host copy of the level's node stencil table (structured node scan), or null
    double *sn_ctot = nullptr;      // [chunk][node] Sigma_t chunk totals (k_sn_scan)
    double *sn_cc = nullptr;        // [chunk][node] chunk carries (k_sn_carry), added by the G update
    bool sn_pending = false;        // the last node scan left its chunk carries for the G update
    // what the V-cycle driver (api.cpp) knows about x = xs_ptr on this level: nothing, x = 0, or
    // st_bslab holds x_q of every chunk's last slab (side output of the sweep / G update /
    // prolongation that last wrote x); the residual's chunk coupling then skips k_st_bslab
    int xs = 0;
    const double *xs_ptr = nullptr;
    int lpr_log2 = 5;       // edge kernels: log2(lanes per row); slab chunk = 2 << lpr_log2 (32: measured best)
    Grid3 grid{};
    double *tau = nullptr;
    double *Pt = nullptr;
    double *Ainv = nullptr;
    bool space_coarsened = false;
    int inner_id = -1;      // index of this level's inner spatial V-cycle levels (st_handle::inner), -1: none
    // work vectors (ST layout)
    double *x = nullptr, *f = nullptr;          // coarse levels only (level 0 uses caller's)
    double *r = nullptr, *z = nullptr, *z2 = nullptr;    // edge temporaries
    double *zn = nullptr, *y = nullptr, *wn = nullptr, *zn2 = nullptr;   // node temporaries
};

struct Options {
    std::string spec = "SAS";
    double omega = 0.5;
    int nu_s = 2;
    double omega_s = 0.6;
    int nu_n = 2;
    double omega_n = 0.6;
    double lambda_crit = 0.1;
    int mode = 0;
    int min_slabs = 1;
    int inner = 0;          // 0: nu_s block-Jacobi sweeps for A_k^{-1}; 1: inner spatial V-cycle (R13)
    int nu_in = 2;
    double omega_in = 0.4;
    int kernel_path = 0;    // 0: assembled ELL operators (default); 1: matrix-free pencil march on uniform hex levels
};

// kernel-side time constants (passed by value to kernels)
struct KT {
    double Ct[kMaxQ * kMaxQ], Mt[kMaxQ * kMaxQ], Ctinv[kMaxQ * kMaxQ], g[kMaxQ];
};
KT make_kt(const TimeMats &tm);

// kernels.cu launchers (all asynchronous on `st`)
typedef struct CUstream_st *Stream;
int launch_residual(Stream st, const DevLevel &L, const KT &kt, int Q, const double *x, const double *f,
                    const double *prev, double *r, double *z, double omega_s, double *partial);
void launch_sweep(Stream st, const DevLevel &L, const KT &kt, int Q, bool last, bool recon, const double *z,
                  const double *r, double *out, double omega_s, double omega);
void launch_axpy(Stream st, size_t n, double alpha, const double *z, double *x);
void launch_sum_blocks(Stream st, size_t n, int nb, const double *in, double *out);
void launch_gtr(Stream st, const DevLevel &L, const KT &kt, int Q, const double *x, const double *f, const double *prev,
                double omega_n, double *zn, double *w);
void launch_node_sweep(Stream st, const DevLevel &L, int Q, const double *z, const double *w, double omega_n,
                       double *zout);
// true when the sweep (last), the G update and the prolongation of this level write the chunk
// boundary slabs of x into L.st_bslab as a side output
bool bslab_producer(const DevLevel &L, int Q);
// returns true when it left chunk carries (L.sn_cc) that the G update of this level must add
bool launch_node_scan(Stream st, const DevLevel &L, const KT &kt, int Q, int mode, const double *z,
                      const double *w, double omega_n, const double *carry, double *y, double *tot);
// cc: chunk carries [S/32][node] of the structured node scan, or null
void launch_g_update(Stream st, const DevLevel &L, const KT &kt, int Q, const double *y, const double *carry,
                     const double *cc, double *x);
void launch_copy_slabs(Stream st, int rows, int Q, int ns, double *dst, int dS, int dk0, const double *src, int sS,
                       int sk0, bool add);
void launch_end_values(Stream st, int rows, int Q, int S, const double *x, double *out);
void launch_restrict(Stream st, const DevLevel &F, const DevLevel &C, int Q, const double *r, double *fc);
void launch_prolong(Stream st, const DevLevel &F, int Q, const double *xc, double *x);
int launch_coarsest(Stream st, const DevLevel &L, int Q, const double *f, double *x);
int acquire_mk_table(const double2 *vals, int n);   // -1: no free constant-bank slot
void release_mk_table(int offset);
void launch_res_mass(Stream st, const DevLevel &L, const KT &kt, int Q, const double *x, const double *f,
                     const double *prev, double *u);
void launch_gt(Stream st, const DevLevel &L, int Q, const double *u, double omega_n, double *zn, double *w);
void launch_residual_local(Stream st, const DevLevel &L, const KT &kt, int Q, const double *z, const double *r,
                           double *d);
void launch_nodal_step(Stream st, const DevLevel &L, const KT &kt, int Q, const double *r, const double *z,
                       double omega_n, double *y);
void launch_jacobi_point(Stream st, const DevLevel &L, const KT &kt, int Q, const double *r, double *z, double omega);
void launch_space_transfer(Stream st, const DevLevel &F, const DevLevel &C, int Q, bool prolong, const double *in,
                           double *out);
void launch_reduce(Stream st, int n, const double *partial, double *out);
int launch_norm2(Stream st, size_t n, const double *v, double *partial);
int residual_partials(const DevLevel &L);
bool stencil_applies(const DevLevel &L, int Q);
int take_extra_launches();   // launches issued beyond the count the caller passes to run()
unsigned long long variants(bool reset);   // bit i set: variant_name(i) has run in this process
const char *variant_name(int bit);

// setup.cpp
TimeMats time_matrices(int q);
HostMesh make_mesh(int dim, const int n[3], const double *coords);
void assemble(HostLevel &L);
void build_chain(const HostLevel &L0, std::vector<HostLevel> &chain);
void build_hierarchy(const st_params &p, const Options &o, const TimeMats &tm,
                     std::vector<HostLevel> &levels);

}  // namespace st
