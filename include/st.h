/*
 * st.h — C-ABI of the B200 space-time multigrid for the eddy-current equation
 *        sigma du/dt + curl(nu curl u) = f      (arXiv:1911.09548, §2-§4)
 *
 * Discretisation: lowest-order Nedelec edge elements on a structured hex (3D)
 * or quad (2D) mesh of the unit cube/square, upwind dG(q) in time on slabs
 * (q = 0 is the paper's implicit Euler, Eq. (1)).  The
 * space-time system L x = f is solved by the V-cycle of
 * l.84 with the hybrid smoother SAS (l.207-226): S = damped block Jacobi in
 * time, Eq. (2) (l.79-82); A = nodal auxiliary space correction, Eq. (5)
 * (l.180-189); spatial coarsening decided per level by the rule Eq. (3)
 * (l.105-109).  Readings of the paper: DESIGN.md §0(c).
 *
 * Numbering (shared by specification with oracle/mesh.py):
 *   node (i,j,k)   id = i + (nx+1)*(j + (ny+1)*k)
 *   x-edges first  id = i + nx*(j + (ny+1)*k)                 (i<nx)
 *   then y-edges   id = Ex + i + (nx+1)*(j + ny*k)             (j<ny)
 *   then z-edges   id = Ex + Ey + i + (nx+1)*(j + (ny+1)*k)    (k<nz)
 *   cell (i,j,k)   id = i + nx*(j + ny*k)
 *   every edge points from its lower to its higher node id.
 * Space-time vector layout ("ST layout"): v[edge][a][slab], slab fastest,
 *   a = 0..q the dG time node (Lagrange basis at s = a/q of the reference slab).
 *   Element (e, a, k) is at e*(q+1)*S + a*S + k.  f is the space-time load
 *   vector (right-hand side of L x = f); the initial state is zero.
 *
 * Memory: every pointer argument documented "device" must be a CUDA device
 * pointer on the device that was current at st_setup, and space-time vectors
 * (x, f, r, fc, xc) must be 16-byte aligned (the kernels move slab pairs as
 * 16-byte vectors; a misaligned vector is refused with code 1); "host" pointers are
 * ordinary (pageable or pinned) host memory.  The library never takes
 * ownership of caller memory; it owns everything it allocates in st_setup and
 * frees it in st_free.  All device work is enqueued on the handle's stream
 * (st_set_stream); functions returning results to the host synchronise it.
 *
 * Errors: every function returns 0 on success and a nonzero code otherwise
 * (1 invalid argument, 2 CUDA error, 3 unsupported configuration, 4 out of
 * memory); st_last_error() gives a human-readable message (thread-local).
 * No function falls back to a CPU implementation.
 */
#ifndef ST_H
#define ST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct st_handle st_handle;

typedef struct st_params {
    /* mesh: dim = 2 or 3; n = cells per direction (nz ignored when dim = 2) */
    int dim, nx, ny, nz;
    /* host, (n_nodes x dim) node coordinates in node-id order, or NULL for the
     * uniform mesh of the unit cube/square.  Cells must not be inverted. */
    const double *coords;
    /* host, per cell: conductivity sigma (alpha in Eq. 3) and reluctivity
     * nu = mu^{-1} (beta in Eq. 3); both > 0 */
    const double *sigma, *nu;
    /* host, n_slabs slab lengths tau_k > 0 of the finest time grid */
    const double *tau;
    int n_slabs;
    int q;                 /* dG degree in time: 0, 1 or 2 */
    /* method parameters (R3, R4, R9); pass <= 0 / NULL for defaults */
    const char *spec;      /* smoother string over {S,A}, default "SAS" (l.226) */
    double omega;          /* Eq. (2) damping, default 0.5 (l.79) */
    int nu_s;              /* block-Jacobi sweeps approximating A_k^{-1}, default 2 */
    double omega_s;        /* their damping, default 0.6 (3D) / 0.5 (2D) */
    int nu_n;              /* Jacobi sweeps approximating K_n^{-1}, default 2 */
    double omega_n;        /* their damping, default 0.6 */
    double lambda_crit;    /* Eq. (3) threshold, default 0.1 (l.292) */
    int mode;              /* 0 auto (Eq. 3 per level), 1 semi-time only, 2 full at the top level only (Table 1) */
    int min_slabs;         /* stop time coarsening at this many slabs, default 1 */
    int kernel_path;       /* 0: assembled ELL operators on every level (default, fastest
                              measured); 1: matrix-free pencil march on uniform hex levels */
    int rank, nranks;      /* multi-GPU (one process per GPU): nranks <= 1 means single GPU.
                              With nranks > 1, tau is the GLOBAL slab array; this rank owns the
                              contiguous block [rank*n_slabs/nranks, (rank+1)*n_slabs/nranks)
                              and its vectors hold only that block (ST layout with S = block). */
    /* approximation of A_k^{-1} inside S (Eq. 2; R13): inner = 0 (default) uses nu_s
       damped block-Jacobi sweeps; inner = 1 one inner SPATIAL V-cycle per slab over the spatial
       coarsening chain of the level's mesh, nu_in (default 2) hybrid sweeps per side: a damped
       edge block-Jacobi sweep (omega_in, default 0.4) and a nodal step on range(G) (omega_n).
       Pass 0 for the defaults. */
    int inner;
    int nu_in;
    double omega_in;
} st_params;

typedef struct st_info_t {
    int n_levels;
    int q;
    int64_t n_dofs;                 /* finest level: n_edges * (q+1) * n_slabs */
    int level_n_edges[32], level_n_nodes[32], level_n_slabs[32];
    int level_space_coarsened[32];  /* 1 if level l -> l+1 coarsened space too */
    double level_lambda[32];        /* Eq. (3) lambda of level l (min over cells) */
    int64_t kernel_launches;        /* kernels launched by this handle so far */
    int64_t device_bytes;           /* bytes of device memory the handle owns */
    int level_matrix_free[32];      /* 1 if level l runs the matrix-free pencil march */
} st_info_t;

/* Build the level hierarchy (mesh coarsening by Eq. 3, operators, transfers,
 * dense coarsest inverse) on the current CUDA device.  *out receives the handle. */
int st_setup(const st_params *p, st_handle **out);
int st_free(st_handle *h);

/* Enqueue all further work on `stream` (a cudaStream_t; NULL = legacy default). */
int st_set_stream(st_handle *h, void *stream);

/* r = f - L x on the finest level (device pointers, ST layout; r may be NULL).
 * If norms != NULL (host, 2 doubles) it receives ||f - L x||_2 and ||f||_2
 * (synchronises). */
int st_residual(st_handle *h, const double *x, const double *f, double *r, double *norms);

/* One V-cycle in place: x <- V(x, f).  Device pointers, ST layout.
 * Asynchronous on the handle's stream. */
int st_vcycle(st_handle *h, double *x, const double *f);

/* enable = 1: st_vcycle and st_solve replay the V-cycle's launch sequence as a CUDA graph,
 * captured on first use for each (x, f) pointer pair (the graph bakes the pointers in; at most
 * 8 pairs are kept, oldest evicted).  Removes the host launch cost of the ~10^2-10^3 kernels of
 * a cycle (small problems are launch-bound).  Ignored while st_profile is recording.
 * enable = 0 (default) launches kernels directly and frees the graphs. */
int st_set_graphs(st_handle *h, int enable);

/* V-cycles from the given x until ||f - L x|| <= tol ||f|| or maxit cycles.
 * Device pointers.  *iters (host) = cycles run; hist (host, maxit+1 doubles,
 * may be NULL) = relative residual before each cycle and after the last.
 * tol <= 0 with hist == NULL runs exactly maxit cycles and computes no norm. */
int st_solve(st_handle *h, double *x, const double *f, double tol, int maxit,
             int *iters, double *hist);

/* Same as st_solve with HOST buffers x (in/out) and f (in): copies f and x to
 * the device, solves, copies x back (all inside the call). */
int st_solve_host(st_handle *h, double *x_host, const double *f_host, double tol,
                  int maxit, int *iters, double *hist);

/* Streaming solve of n independent problems L x_i = f_i held in HOST memory (page-locked
 * memory lets the copies overlap): each from x_i = 0, or from x_host[i] when init_from_x != 0,
 * with st_solve's stopping rule.  Two device buffer pairs and two copy streams: the H2D copy of
 * problem i+1 and the D2H copy of problem i-1 run while problem i is solved.  x_host[i] (out)
 * is complete when the call returns.  iters (n ints) and hist (n * (maxit+1) doubles, problem
 * i at hist + i*(maxit+1)) may be NULL.  Single-process handles only. */
int st_solve_many_host(st_handle *h, int n, double *const *x_host, const double *const *f_host,
                       int init_from_x, double tol, int maxit, int *iters, double *hist);

int st_info(const st_handle *h, st_info_t *info);

/* Per-kernel timing with CUDA events recorded on the handle's stream around
 * every launch (enable = 1 starts a fresh record, 0 stops recording). */
int st_profile(st_handle *h, int enable);

typedef struct st_kstat {
    char name[32];          /* kernel family, e.g. "residual", "sweep", "node_scan" */
    int64_t launches;
    double ms;              /* summed CUDA-event durations */
    double bytes;           /* summed algorithmic bytes */
} st_kstat;

/* Synchronises the stream and returns up to `max` per-family aggregates of
 * the launches recorded since st_profile(h, 1); *n = number of families. */
int st_profile_read(st_handle *h, st_kstat *out, int max, int *n);

/* ---- level operations: a driver (multi-GPU: paper_1911_09548_b200/distributed.py)
 * sequences the V-cycle itself around its collectives.  set = 0: this rank's distributed
 * levels 0..g0 over its slab block; set = 1 (rank 0 of a multi-rank handle only): the
 * gathered global levels g0..L-1 (index 0 of set 1 is global level g0).  All vector
 * arguments are device pointers in ST layout for that level's slab count; `prev` is the
 * time-node-q trace of the slab before the block (n_edges values) or NULL (zero initial
 * state); `tot` / `carry` hold one value per node (the integrated end value of the nodal
 * correction's time scan, R2).  Asynchronous unless stated. */
typedef struct st_level_t {
    int set, level, global_level;
    int n_slabs, slab0;          /* slab count of this level in this set, first global slab */
    int n_edges, n_nodes, q;
    int coarsest, space_coarsened;
    double *x, *f;               /* the level's own work vectors (NULL for set 0, level 0) */
    double *r;                   /* the level's residual scratch (overwritten by every level op) */
} st_level_t;

int st_lv_count(const st_handle *h, int set, int *n);
int st_lv_get(const st_handle *h, int set, int level, st_level_t *out);
/* r = f - L x (r may be NULL); norm2 (host, may be NULL) receives ||r||^2 (synchronises) */
int st_lv_residual(st_handle *h, int set, int level, const double *x, const double *f, const double *prev,
                   double *r, double *norm2);
int st_lv_smooth_S(st_handle *h, int set, int level, double *x, const double *f, const double *prev);  /* Eq. (2) */
int st_lv_correct_local(st_handle *h, int set, int level, double *x, const double *f, const double *prev,
                        double *tot);                                                          /* Eq. (5), 1st half */
int st_lv_correct_apply(st_handle *h, int set, int level, double *x, const double *carry);     /* Eq. (5), 2nd half */
int st_lv_restrict(st_handle *h, int set, int level, const double *r, double *fc);             /* level -> level+1 */
int st_lv_prolong(st_handle *h, int set, int level, const double *xc, double *x);              /* x += P xc */
int st_lv_vcycle(st_handle *h, int set, int level, double *x, const double *f);                /* within the set */
int st_lv_end_values(st_handle *h, int set, int level, const double *x, double *out);
/* dst[row][a][dk0+s] (+)= src[row][a][sk0+s] for s < ns, rows x (q+1) rows of slabs */
int st_copy_slabs(st_handle *h, int rows, int q, int ns, double *dst, int dS, int dk0, const double *src, int sS,
                  int sk0, int add);
int st_zero(st_handle *h, double *ptr, int64_t n);
/* Vector operations of the multi-GPU driver (device pointers, n elements, on the handle's stream):
 * y += alpha x; out = sum over b < nb of the blocks in[b*n .. (b+1)*n) (the Sigma_t carry of the
 * ranks before this one, R2; nb = 0 gives zeros); *out (host) = ||v||_2^2 (synchronises). */
int st_vec_axpy(st_handle *h, int64_t n, double alpha, const double *x, double *y);
int st_vec_sum_blocks(st_handle *h, int64_t n, int nb, const double *in, double *out);
int st_vec_norm2(st_handle *h, int64_t n, const double *v, double *out);
int st_sync(st_handle *h);

/* Host-only (no CUDA device needed): build the level hierarchy of p on the
 * host and report it in *info (kernel_launches = device_bytes = 0). */
int st_plan(const st_params *p, st_info_t *info);

/* Host-only: the assembled operator `which` (0 = M_sigma, 1 = K_nu, 2 = K_n,
 * 3 = prolongation P_edge of level -> level+1) of hierarchy level `level`, as
 * ELL with `*width` slots per row (padding slots carry value 0).  Call with
 * col = val = NULL to get *rows and *width, then with host arrays of
 * rows*width entries.  For checking the setup against an independent
 * assembly. */
int st_host_matrix(const st_params *p, int level, int which, int *rows, int *width, int *col, double *val);

/* Diagnostics: bit i of *mask (host) is set when the kernel variant st_variant_name(i) (e.g.
 * "sweep/spl4": the block-Jacobi sweep at 4 slabs per lane; "node_scan/multichunk": the Sigma_t
 * scan carrying over several slab chunks; "stencil/residual", "stencil/sweep",
 * "stencil/node_scan": the TMA-staged structured marches of uniform hex levels) has been
 * launched by this process since the last
 * reset; reset != 0 clears the log after reading.  Lets tests prove which code paths ran.
 * st_variant_name returns NULL past the last variant. */
int st_kernel_variants(uint64_t *mask, int reset);
const char *st_variant_name(int bit);
const char *st_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* ST_H */
