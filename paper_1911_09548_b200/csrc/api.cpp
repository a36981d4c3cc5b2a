// api.cpp — the C-ABI of include/st.h: device hierarchy, V-cycle driver, solve loop.
//
// The V-cycle is driven from the host: per level the hybrid
// smoother (spec read right to left, l.208; reversed for post-smoothing),
// residual + restriction, recursion, prolongation.  Every arithmetic step is
// a kernel of kernels.cu launched on the handle's stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <initializer_list>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "internal.h"

namespace {

thread_local std::string g_err;

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct Unsupported : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char *what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

struct st_handle {
    st::Options o;
    st::TimeMats tm{};
    st::KT kt{};
    int Q = 1;
    std::vector<st::HostLevel> hl;
    std::vector<st::DevLevel> dl;   // this rank's levels 0..(g0 or L-1), local slab blocks
    std::vector<st::DevLevel> dg;   // rank 0 of a multi-rank run: global levels g0..L-1 ("gathered")
    std::vector<std::vector<st::DevLevel>> inner;   // inner spatial V-cycle levels per smoothing level (R13)
    int rank = 0, nranks = 1, g0 = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    double *partial = nullptr;
    int partial_cap = 0;
    double *dscal = nullptr;
    double *hx = nullptr, *hf = nullptr;   // device buffers for st_solve_host
    // st_solve_many_host: double-buffered device problems, copy streams and their events
    double *mx[2] = {nullptr, nullptr}, *mf[2] = {nullptr, nullptr};
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
    int64_t launches = 0;
    int64_t bytes = 0;
    std::vector<void *> allocs;
    int64_t n_dofs = 0;
    // CUDA-graph replay of the single-process V-cycle (st_set_graphs)
    bool use_graphs = false;
    int nodal_res = 3;          // env ST_NODAL_RES: 0 G^T (f - L x) literally, 1 two-pass with
                                // G^T K = 0 (u = f - Ct M x), 2 fused node-row G^T M (K G = 0),
                                // 3 (default) the two-pass mass form on stencil levels, 0 elsewhere
    bool mk_dict = true;        // env ST_MK_DICT=0: never use the dictionary ELL
    bool stencil = true;        // env ST_STENCIL=0: never use the structured stencil march
    std::vector<std::unique_ptr<st::StencilTab>> st_tabs;
    std::vector<std::unique_ptr<st::NodeTab>> sn_tabs;
    std::vector<int> tab_slots;   // constant-bank dictionary slots this handle holds
    cudaStream_t cap_stream = nullptr;
    struct Graph { const double *x, *f; cudaGraphExec_t exec; int64_t launches; };
    std::vector<Graph> graphs;
    void clear_graphs() {
        for (auto &g : graphs) cudaGraphExecDestroy(g.exec);
        graphs.clear();
    }
    // profiling: (family, bytes, start, stop) per recorded launch
    bool prof = false;
    struct Rec { int fam; double bytes; cudaEvent_t a, b; };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    std::vector<std::string> fams;
    int fam_id(const char *name) {
        for (size_t i = 0; i < fams.size(); ++i)
            if (fams[i] == name) return (int)i;
        fams.push_back(name);
        return (int)fams.size() - 1;
    }
    cudaEvent_t ev() {
        if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
        cudaEvent_t e;
        ck(cudaEventCreate(&e), "event");
        return e;
    }
    // run `launch` (which issues exactly `count` kernels) and, when profiling, time it
    bool debug_sync = false;   // env ST_DEBUG_SYNC=1: synchronise and check after every launch
    template <class F>
    void run(const char *fam, double bytes, int count, F &&launch) {
        if (debug_sync) {
            launch();
            launches += count + st::take_extra_launches();
            cudaError_t e = cudaStreamSynchronize(stream);
            if (e == cudaSuccess) e = cudaGetLastError();
            if (e != cudaSuccess) throw CudaError(std::string("kernel ") + fam + ": " + cudaGetErrorString(e));
            return;
        }
        if (!prof) { launch(); launches += count + st::take_extra_launches(); return; }
        Rec r{fam_id(fam), bytes, ev(), ev()};
        ck(cudaEventRecord(r.a, stream), "event record");
        launch();
        ck(cudaEventRecord(r.b, stream), "event record");
        recs.push_back(r);
        launches += count + st::take_extra_launches();
    }

    template <class T>
    T *dalloc(size_t n) {
        void *p = nullptr;
        if (n == 0) n = 1;
        cudaError_t e = cudaMalloc(&p, n * sizeof(T));
        if (e == cudaErrorMemoryAllocation) throw std::bad_alloc();
        ck(e, "cudaMalloc");
        allocs.push_back(p);
        bytes += (int64_t)(n * sizeof(T));
        return (T *)p;
    }
    template <class T>
    T *upload(const std::vector<T> &v) {
        T *p = dalloc<T>(v.size());
        if (!v.empty()) ck(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
        return p;
    }
    st::DevELL upload(const st::HostELL &E) {
        st::DevELL d;
        d.rows = E.rows; d.width = E.width;
        if (E.val.empty()) {
            d.col = upload(E.col);
        } else {
            std::vector<st::Ent> ent(E.col.size());
            for (size_t i = 0; i < ent.size(); ++i) ent[i] = st::Ent{E.val[i], E.col[i], 0};
            d.e = upload(ent);
        }
        return d;
    }
    // merged M/K operator of a level: (col, (M, K)) ELL, plus the dictionary form when the level
    // has a uniform stencil width (33 in 3D, 7 in 2D) and at most 256 distinct (M, K) pairs
    void upload_mk(const st::HostELL &MK, const std::vector<double> &MKk, int m_width, st::DevLevel &D) {
        std::vector<double2> mkv(MK.val.size());
        for (size_t i = 0; i < mkv.size(); ++i) mkv[i] = make_double2(MK.val[i], MKk[i]);
        D.mk_width = MK.width;
        D.mk_col = upload(MK.col);
        D.mk_val = upload(mkv);
        const bool stencil = (m_width == 9 && MK.width == 33) || (m_width == 3 && MK.width == 7);
        if (!mk_dict || !stencil || MK.rows >= (1 << 24)) return;
        std::map<std::pair<uint64_t, uint64_t>, unsigned> ids;
        std::vector<double2> tab;
        const int W = MK.width, W4 = (W + 3) / 4 * 4;
        std::vector<unsigned> pk((size_t)MK.rows * W4, 0u);
        for (int r = 0; r < MK.rows; ++r)
            for (int s = 0; s < W; ++s) {
                const size_t i = (size_t)r * W + s;
                uint64_t a, b;
                std::memcpy(&a, &MK.val[i], 8);
                std::memcpy(&b, &MKk[i], 8);
                auto it = ids.find({a, b});
                if (it == ids.end()) {
                    if (tab.size() == 256) return;        // too many distinct values: plain ELL
                    it = ids.emplace(std::make_pair(a, b), (unsigned)tab.size()).first;
                    tab.push_back(mkv[i]);
                }
                if (MK.col[i] < 0) return;
                pk[(size_t)r * W4 + s] = ((unsigned)MK.col[i] << 8) | it->second;
            }
        const int off = st::acquire_mk_table(tab.data(), (int)tab.size());
        if (off < 0) return;
        tab_slots.push_back(off);
        D.mk_pk = upload(pk);
        D.mk_tab = off;
    }
    ~st_handle() {
        // drain every stream that may still run this handle's kernels or copies before the
        // constant-bank dictionary slots and device buffers are released for reuse
        if (stream) cudaStreamSynchronize(stream);
        if (h2d) cudaStreamSynchronize(h2d);
        if (d2h) cudaStreamSynchronize(d2h);
        clear_graphs();
        for (int b = 0; b < 2; ++b)
            for (cudaEvent_t e : {ev_in[b], ev_done[b], ev_out[b]})
                if (e) cudaEventDestroy(e);
        if (h2d) cudaStreamDestroy(h2d);
        if (d2h) cudaStreamDestroy(d2h);
        for (int t : tab_slots) st::release_mk_table(t);
        if (cap_stream) cudaStreamDestroy(cap_stream);
        for (auto &r : recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
        for (auto e : pool) cudaEventDestroy(e);
        for (void *p : allocs) cudaFree(p);
    }
};

namespace {

using st::DevLevel;

size_t vec_len(const DevLevel &L, int Q, bool nodes = false) {
    return (size_t)(nodes ? L.n_nodes : L.n_edges) * Q * L.S;
}

// Algorithmic bytes: every vector touched once, operators read once.
double ell_bytes(const st::DevELL &E) { return (double)E.rows * E.width * 16.0; }
// (stencil levels read no operator: their coefficients are kernel parameters)
double op_bytes(const DevLevel &L) {
    if (st::stencil_applies(L, L.Q)) return 0.0;
    return ell_bytes(L.M) + ell_bytes(L.K) + 16.0 * L.n_edges;
}
double evec(const DevLevel &L, int Q) { return 8.0 * L.n_edges * Q * L.S; }
double nvec(const DevLevel &L, int Q) { return 8.0 * L.n_nodes * Q * L.S; }

// prev: end values (time node q) of the slab before this level's first slab (the previous
// rank's last slab), or null for the zero initial state (PAPER.md l.47-48 homogeneous u^0)
// One inner spatial V-cycle (R13: the "A_k^{-1} sufficiently well approximated" of
// Eq. (2)) for A_k z = r on all slabs at once (the slabs are
// independent: no time coupling below the outer residual).  V[j] shares the chain operators
// and its own vectors; returns the buffer holding z.  j = 0 enters with the first edge sweep
// from zero already done (fused into the outer residual) and, with xout set, its last edge
// sweep adds omega * z into xout instead of storing z.
double *inner_vcycle(st_handle *h, std::vector<DevLevel> &V, int j, const double *r, double *xout) {
    const auto &o = h->o;
    auto s = (st::Stream)h->stream;
    const int Q = h->Q;
    DevLevel &I = V[j];
    const double ev = evec(I, Q), nv = nvec(I, Q), ob = op_bytes(I);
    const bool coarsest = j + 1 == (int)V.size();
    double *cur = I.z, *oth = I.z2;
    auto nodal = [&] {
        h->run("in_nodal", 2 * ev + nv + ell_bytes(I.GtM) + 8.0 * I.n_nodes, 1,
               [&] { st::launch_nodal_step(s, I, h->kt, Q, r, cur, o.omega_n, I.y); });
        h->run("in_gupdate", 2 * ev + nv + 8.0 * I.n_edges, 1, [&] { st::launch_g_update(s, I, h->kt, Q, I.y, nullptr, nullptr, cur); });
    };
    for (int i = 0; i < o.nu_in; ++i) {
        if (i == 0) {
            if (j > 0) h->run("in_jacobi", 2 * ev, 1, [&] { st::launch_jacobi_point(s, I, h->kt, Q, r, cur, o.omega_in); });
        } else {
            h->run("in_sweep", 3 * ev + ob, 1, [&] { st::launch_sweep(s, I, h->kt, Q, false, false, cur, r, oth, o.omega_in, 0.0); });
            std::swap(cur, oth);
        }
        nodal();
    }
    if (coarsest) {
        if (xout) h->run("axpy", 3 * ev, 1, [&] { st::launch_axpy(s, vec_len(I, Q), o.omega, cur, xout); });
        return cur;
    }
    DevLevel &C = V[j + 1];
    h->run("in_residual", 3 * ev + ob, 1, [&] { st::launch_residual_local(s, I, h->kt, Q, cur, r, oth); });
    h->run("in_restrict", ev + evec(C, Q) + ell_bytes(I.Rg), 1, [&] { st::launch_space_transfer(s, I, C, Q, false, oth, C.r); });
    double *zc = inner_vcycle(h, V, j + 1, C.r, nullptr);
    h->run("in_prolong", 2 * ev + evec(C, Q) + ell_bytes(I.Pg), 1, [&] { st::launch_space_transfer(s, I, C, Q, true, zc, cur); });
    for (int i = 0; i < o.nu_in; ++i) {
        nodal();
        if (xout && i + 1 == o.nu_in) {
            h->run("in_sweep_update", 4 * ev + ob, 1, [&] { st::launch_sweep(s, I, h->kt, Q, true, false, cur, r, xout, o.omega_in, o.omega); });
        } else {
            h->run("in_sweep", 3 * ev + ob, 1, [&] { st::launch_sweep(s, I, h->kt, Q, false, false, cur, r, oth, o.omega_in, 0.0); });
            std::swap(cur, oth);
        }
    }
    return cur;
}

// what the driver knows about the level's x after a kernel wrote it (DevLevel::xs): the stencil
// sweep / G update / prolongation leave the chunk boundary slabs of x in L.st_bslab
static void x_written(st_handle *h, DevLevel &L, const double *x, bool producer) {
    L.xs = producer && st::bslab_producer(L, h->Q) ? st::XS_BSLAB : st::XS_UNKNOWN;
    L.xs_ptr = x;
}
static void x_unknown(DevLevel &L) {
    L.xs = st::XS_UNKNOWN;
    L.xs_ptr = nullptr;
}

void smooth_S(st_handle *h, DevLevel &L, double *x, const double *f, const double *prev) {
    const auto &o = h->o;
    if (o.inner == 1 && L.inner_id >= 0) {
        // Eq. (2) with the inner V-cycle: r = f - L x and its first edge sweep z = omega_in D^{-1} r
        // in one pass, then the rest of the inner cycle, whose last sweep performs x += omega z
        auto &V = h->inner[L.inner_id];
        h->run("residual", 4 * evec(L, h->Q) + op_bytes(L), 1, [&] {
            st::launch_residual((st::Stream)h->stream, L, h->kt, h->Q, x, f, prev, V[0].r, V[0].z, o.omega_in, nullptr);
        });
        inner_vcycle(h, V, 0, V[0].r, x);
        x_written(h, L, x, false);
        return;
    }
    auto s = (st::Stream)h->stream;
    const int Q = h->Q;
    const double ev = evec(L, Q), ob = op_bytes(L);
    if (o.nu_s == 1) {
        h->run("residual", 3 * ev + ob, 1, [&] { st::launch_residual(s, L, h->kt, Q, x, f, prev, nullptr, L.z, o.omega_s, nullptr); });
        h->run("axpy", 3 * ev, 1, [&] { st::launch_axpy(s, vec_len(L, Q), o.omega, L.z, x); });
        x_written(h, L, x, false);
        return;
    }
    if (o.nu_s == 2 && !prev && L.xs == st::XS_ZERO && L.xs_ptr == x) {
        // x = 0 (a coarse level's first smoothing step): r = f, so the first sweep from zero is the
        // pointwise z = omega_s D^{-1} f -- no operator pass (the second sweep rebuilds r from z)
        h->run("residual", 2 * ev, 1, [&] { st::launch_jacobi_point(s, L, h->kt, Q, f, L.z, o.omega_s); });
    } else {
        h->run("residual", (o.nu_s > 2 ? 4 : 3) * ev + ob, 1, [&] {
            st::launch_residual(s, L, h->kt, Q, x, f, prev, o.nu_s > 2 ? L.r : nullptr, L.z, o.omega_s, nullptr);
        });
    }
    double *cur = L.z, *other = L.z2;
    for (int i = 2; i < o.nu_s; ++i) {
        h->run("sweep", 3 * ev + ob, 1, [&] { st::launch_sweep(s, L, h->kt, Q, false, false, cur, L.r, other, o.omega_s, o.omega); });
        std::swap(cur, other);
    }
    h->run("sweep_update", (o.nu_s == 2 ? 3 : 4) * ev + ob, 1, [&] {
        st::launch_sweep(s, L, h->kt, Q, true, o.nu_s == 2, cur, L.r, x, o.omega_s, o.omega);
    });
    x_written(h, L, x, true);
}

// first half of the nodal correction: r, G^T r, nodal sweeps and the local time scan into L.y;
// tot (optional, n_nodes) receives each node's integrated end value (rank carry)
void correct_A_local(st_handle *h, DevLevel &L, double *x, const double *f, const double *prev, double *tot) {
    const auto &o = h->o;
    auto s = (st::Stream)h->stream;
    const int Q = h->Q;
    const double ev = evec(L, Q), nv = nvec(L, Q), kb = ell_bytes(L.Kn) + 8.0 * L.n_nodes;
    if (h->nodal_res == 3 && st::stencil_applies(L, Q)) {
        // uniform hex levels (default): the mass form of the same residual, u = f - (Ct (x) M) x +
        // coupling by the stencil march without its curl-curl part (K G = 0, R17), then
        // w = G^T u; other levels keep the literal form below
        h->run("gtr_mass", 3 * ev + op_bytes(L), 1, [&] { st::launch_res_mass(s, L, h->kt, Q, x, f, prev, L.r); });
        h->run("gt", ev + (o.nu_n > 2 ? 2 : 1) * nv + 8.0 * L.n_nodes, 1,
               [&] { st::launch_gt(s, L, Q, L.r, o.omega_n, L.zn, o.nu_n > 2 ? L.wn : nullptr); });
    } else if (h->nodal_res == 0 || h->nodal_res == 3) {
        // Eq. (5) as written: r = f - L x with the full operator, then w = G^T r
        // on node rows (6 gathers).  The K G = 0 shortcuts below are the same map in exact
        // arithmetic but drop G^T K x, which in fp64 is rounding of size eps |tau K x|: measured
        // against an extended-precision V-cycle they are 7-13x less accurate than this form on the
        // c5 / c3 recipes (R12, tests/test_gpu_bench_paths.py)
        h->run("residual", 3 * ev + op_bytes(L), 1,
               [&] { st::launch_residual(s, L, h->kt, Q, x, f, prev, L.r, nullptr, o.omega_s, nullptr); });
        h->run("gt", ev + (o.nu_n > 2 ? 2 : 1) * nv + 8.0 * L.n_nodes, 1,
               [&] { st::launch_gt(s, L, Q, L.r, o.omega_n, L.zn, o.nu_n > 2 ? L.wn : nullptr); });
    } else if (h->nodal_res == 1 && L.M.width <= 12) {
        // narrow M (uniform meshes): u = f - (Ct (x) M) x + coupling on edge rows, then w = G^T u
        // on node rows (6 gathers) -- one more vector pass, far fewer L1 gathers than G^T M
        h->run("gtr_mass", 3 * ev + ell_bytes(L.M), 1, [&] { st::launch_res_mass(s, L, h->kt, Q, x, f, prev, L.r); });
        h->run("gt", ev + (o.nu_n > 2 ? 2 : 1) * nv + 8.0 * L.n_nodes, 1,
               [&] { st::launch_gt(s, L, Q, L.r, o.omega_n, L.zn, o.nu_n > 2 ? L.wn : nullptr); });
    } else {
        // fused nodal residual: w = G^T (f - L x) by a node-row SpMV with G^T M (K G = 0), zn = omega_n w / d_n
        h->run("gtr", 2 * ev + (o.nu_n > 2 ? 2 : 1) * nv + ell_bytes(L.GtM) + 8.0 * L.n_nodes, 1,
               [&] { st::launch_gtr(s, L, h->kt, Q, x, f, prev, o.omega_n, L.zn, o.nu_n > 2 ? L.wn : nullptr); });
    }
    double *cur = L.zn, *other = L.zn2;
    int mode = o.nu_n == 1 ? 0 : (o.nu_n == 2 ? 1 : 2);
    for (int i = 2; i < o.nu_n; ++i) {
        h->run("node_sweep", 3 * nv + kb, 1, [&] { st::launch_node_sweep(s, L, Q, cur, L.wn, o.omega_n, other); });
        std::swap(cur, other);
    }
    h->run("node_scan", (mode == 2 ? 3 : 2) * nv + kb, 1, [&] { L.sn_pending = st::launch_node_scan(s, L, h->kt, Q, mode, cur, L.wn, o.omega_n, nullptr, L.y, tot); });
}

// second half: x += G (y + g carry), carry (optional, n_nodes) = end value before this block
void correct_A_apply(st_handle *h, DevLevel &L, double *x, const double *carry) {
    auto s = (st::Stream)h->stream;
    const int Q = h->Q;
    h->run("g_update", 2 * evec(L, Q) + nvec(L, Q) + 8.0 * L.n_edges, 1,
           [&] { st::launch_g_update(s, L, h->kt, Q, L.y, carry, L.sn_pending ? L.sn_cc : nullptr, x); });
    x_written(h, L, x, true);
}

void correct_A(st_handle *h, DevLevel &L, double *x, const double *f, const double *prev) {
    correct_A_local(h, L, x, f, prev, nullptr);
    correct_A_apply(h, L, x, nullptr);
}

void hybrid(st_handle *h, DevLevel &L, double *x, const double *f, bool pre) {
    std::string seq = h->o.spec;
    if (!pre) std::reverse(seq.begin(), seq.end());
    for (int i = (int)seq.size() - 1; i >= 0; --i) {   // right to left (l.208)
        if (seq[i] == 'S') smooth_S(h, L, x, f, nullptr);
        else correct_A(h, L, x, f, nullptr);
    }
}

void restrict_to(st_handle *h, DevLevel &L, DevLevel &C, const double *r, double *fc) {
    auto s = (st::Stream)h->stream;
    const int Q = h->Q;
    h->run("restrict", evec(L, Q) + evec(C, Q) + (L.space_coarsened ? ell_bytes(L.Rg) : 0.0), 1,
           [&] { st::launch_restrict(s, L, C, Q, r, fc); });
}

void prolong_from(st_handle *h, DevLevel &L, DevLevel &C, const double *xc, double *x) {
    auto s = (st::Stream)h->stream;
    const int Q = h->Q;
    h->run("prolong", 2 * evec(L, Q) + evec(C, Q) + (L.space_coarsened ? ell_bytes(L.Pg) : 0.0), 1,
           [&] { st::launch_prolong(s, L, Q, xc, x); });
    x_written(h, L, x, true);
}

// single-process V-cycle over the level vector V from level l (the last entry is the coarsest)
void vcycle(st_handle *h, std::vector<DevLevel> &V, int l, double *x, const double *f) {
    DevLevel &L = V[l];
    auto s = (st::Stream)h->stream;
    const int Q = h->Q;
    if (l == (int)V.size() - 1) {
        const double N = (double)Q * L.n_edges;
        h->run("coarsest", L.S * (N * N * 8.0 + 2 * evec(L, Q) / L.S), L.S, [&] { st::launch_coarsest(s, L, Q, f, x); });
        x_written(h, L, x, false);
        return;
    }
    hybrid(h, L, x, f, true);
    DevLevel &C = V[l + 1];
    h->run("residual", 3 * evec(L, Q) + op_bytes(L), 1, [&] { st::launch_residual(s, L, h->kt, Q, x, f, nullptr, L.r, nullptr, h->o.omega_s, nullptr); });
    restrict_to(h, L, C, L.r, C.f);
    if (l + 1 < (int)V.size() - 1) {
        ck(cudaMemsetAsync(C.x, 0, sizeof(double) * vec_len(C, Q), h->stream), "memset");
        C.xs = st::XS_ZERO;         // the first residual of the coarse level needs no chunk coupling
        C.xs_ptr = C.x;
    }
    vcycle(h, V, l + 1, C.x, C.f);
    prolong_from(h, L, C, C.x, x);
    hybrid(h, L, x, f, false);
}

// the single-process V-cycle on the finest level, through a captured CUDA graph when enabled
void run_vcycle(st_handle *h, double *x, const double *f) {
    x_unknown(h->dl[0]);            // the caller may have changed x since the last V-cycle
    if (!h->use_graphs || h->prof || h->debug_sync) { vcycle(h, h->dl, 0, x, f); return; }
    for (auto &g : h->graphs)
        if (g.x == x && g.f == f) {
            ck(cudaGraphLaunch(g.exec, h->stream), "graph launch");
            h->launches += g.launches;
            return;
        }
    if (h->graphs.size() >= 8) {
        cudaGraphExecDestroy(h->graphs.front().exec);
        h->graphs.erase(h->graphs.begin());
    }
    // capture on a private stream (the user's may be the legacy default stream, which cannot
    // capture); nothing executes during capture, the graph is launched on the user's stream
    if (!h->cap_stream) ck(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking), "capture stream");
    const int64_t l0 = h->launches;
    cudaGraph_t graph = nullptr;
    cudaStream_t user = h->stream;
    h->stream = h->cap_stream;
    ck(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal), "begin capture");
    try {
        vcycle(h, h->dl, 0, x, f);
    } catch (...) {
        cudaStreamEndCapture(h->stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        h->stream = user;
        h->launches = l0;
        throw;
    }
    cudaError_t ce = cudaStreamEndCapture(h->stream, &graph);
    h->stream = user;
    ck(ce, "end capture");
    st_handle::Graph g{x, f, nullptr, h->launches - l0};
    h->launches = l0;
    cudaError_t e = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    ck(e, "graph instantiate");
    h->graphs.push_back(g);
    ck(cudaGraphLaunch(g.exec, h->stream), "graph launch");
    h->launches += g.launches;
}

// ||f - L x||^2 (f != null) on level 0 without storing r
double residual_norm2(st_handle *h, const double *x, const double *f) {
    DevLevel &L = h->dl[0];
    auto s = (st::Stream)h->stream;
    int g = 0;
    h->run("residual_norm", 2 * evec(L, h->Q) + op_bytes(L), 1,
           [&] { g = st::launch_residual(s, L, h->kt, h->Q, x, f, nullptr, nullptr, nullptr, h->o.omega_s, h->partial); });
    h->run("reduce", 8.0 * g, 1, [&] { st::launch_reduce(s, g, h->partial, h->dscal); });
    double v = 0;
    ck(cudaMemcpyAsync(&v, h->dscal, sizeof(double), cudaMemcpyDeviceToHost, h->stream), "norm d2h");
    ck(cudaStreamSynchronize(h->stream), "sync");
    return v;
}

double norm2_plain(st_handle *h, const double *v, size_t n) {
    // ||v||^2 via the residual kernel would need x = 0; use a dedicated pass instead
    auto s = (st::Stream)h->stream;
    int g = 0;
    h->run("norm2", 8.0 * n, 1, [&] { g = st::launch_norm2(s, n, v, h->partial); });
    h->run("reduce", 8.0 * g, 1, [&] { st::launch_reduce(s, g, h->partial, h->dscal); });
    double out = 0;
    ck(cudaMemcpyAsync(&out, h->dscal, sizeof(double), cudaMemcpyDeviceToHost, h->stream), "norm d2h");
    ck(cudaStreamSynchronize(h->stream), "sync");
    return out;
}

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

// the kernels move slab pairs / quadruples as 16-byte vectors: device vector arguments must be
// 16-byte aligned (a view at an odd element offset would fault and kill the CUDA context)
bool misaligned(std::initializer_list<const void *> ptrs) {
    for (const void *p : ptrs)
        if (p && (reinterpret_cast<uintptr_t>(p) & 15u)) return true;
    return false;
}
#define ST_CHECK_ALIGNED(...) \
    if (misaligned({__VA_ARGS__})) return fail(1, "device vectors must be 16-byte aligned")

#define ST_GUARD(body)                                              \
    try {                                                           \
        body;                                                       \
        ck(cudaGetLastError(), "kernel launch");                    \
        return 0;                                                   \
    } catch (const Unsupported &e) {                                \
        return fail(3, e.what());                                   \
    } catch (const CudaError &e) {                                  \
        return fail(2, e.what());                                   \
    } catch (const std::bad_alloc &) {                              \
        return fail(4, "out of memory");                            \
    } catch (const std::length_error &e) {                          \
        return fail(3, e.what());                                   \
    } catch (const std::invalid_argument &e) {                      \
        return fail(1, e.what());                                   \
    } catch (const std::exception &e) {                             \
        return fail(1, e.what());                                   \
    }

}  // namespace

extern "C" {

static void parse_options(const st_params *p, st::Options &o) {
    if (p->dim != 2 && p->dim != 3) throw std::invalid_argument("dim must be 2 or 3");
    if (p->nx < 1 || p->ny < 1 || (p->dim == 3 && p->nz < 1)) throw std::invalid_argument("bad mesh size");
    if (!p->sigma || !p->nu || !p->tau || p->n_slabs < 1) throw std::invalid_argument("missing sigma/nu/tau");
    const long long ncell = (long long)p->nx * p->ny * (p->dim == 3 ? p->nz : 1);
    for (long long c = 0; c < ncell; ++c)
        if (!(p->sigma[c] > 0) || !(p->nu[c] > 0)) throw std::invalid_argument("sigma and nu must be > 0");
    for (int k = 0; k < p->n_slabs; ++k)
        if (!(p->tau[k] > 0)) throw std::invalid_argument("tau must be > 0");
    if (p->spec && p->spec[0]) o.spec = p->spec;
    for (char c : o.spec)
        if (c != 'S' && c != 'A') throw std::invalid_argument("spec may only contain S and A");
    if (p->omega > 0) o.omega = p->omega;
    if (p->nu_s > 0) o.nu_s = p->nu_s;
    o.omega_s = p->omega_s > 0 ? p->omega_s : (p->dim == 2 ? 0.5 : 0.6);
    if (p->nu_n > 0) o.nu_n = p->nu_n;
    if (p->omega_n > 0) o.omega_n = p->omega_n;
    if (p->lambda_crit > 0) o.lambda_crit = p->lambda_crit;
    if (p->mode < 0 || p->mode > 2) throw std::invalid_argument("mode must be 0, 1 or 2");
    o.mode = p->mode;
    if (p->min_slabs > 0) o.min_slabs = p->min_slabs;
    if (p->kernel_path < 0 || p->kernel_path > 1) throw std::invalid_argument("kernel_path must be 0 or 1");
    if (p->nranks > 1 && (p->rank < 0 || p->rank >= p->nranks)) throw std::invalid_argument("rank out of range");
    if (p->nranks > 1 && p->n_slabs % p->nranks) throw std::invalid_argument("n_slabs must be a multiple of nranks");
    o.kernel_path = p->kernel_path;
    if (p->inner < 0 || p->inner > 1) throw std::invalid_argument("inner must be 0 (block Jacobi) or 1 (spatial V-cycle)");
    o.inner = p->inner;
    if (p->nu_in > 0) o.nu_in = p->nu_in;
    if (p->omega_in > 0) o.omega_in = p->omega_in;
}

const char *st_last_error(void) { return g_err.c_str(); }

int st_kernel_variants(uint64_t *mask, int reset) {
    if (!mask) return fail(1, "null argument");
    *mask = (uint64_t)st::variants(reset != 0);
    return 0;
}

const char *st_variant_name(int bit) { return st::variant_name(bit); }

int st_setup(const st_params *p, st_handle **out) {
    if (!p || !out) return fail(1, "null argument");
    *out = nullptr;
    st_handle *h = new st_handle();
    try {
        st::Options &o = h->o;
        parse_options(p, o);
        h->tm = st::time_matrices(p->q);
        h->kt = st::make_kt(h->tm);
        h->Q = h->tm.Q;
        st::build_hierarchy(*p, o, h->tm, h->hl);
        const int Q = h->Q;
        h->rank = p->nranks > 1 ? p->rank : 0;
        h->nranks = p->nranks > 1 ? p->nranks : 1;
        const int P = h->nranks, L = (int)h->hl.size();
        // distributed levels: S_l divisible by P with at least one slab per rank; the last of
        // them (g0) is where the V-cycle hands over to the gathered global levels (rank 0)
        int nd = 0;
        while (nd < L && (int)h->hl[nd].tau.size() >= P && (int)h->hl[nd].tau.size() % P == 0) ++nd;
        if (nd == 0) throw std::invalid_argument("n_slabs must be a multiple of nranks");
        h->g0 = P > 1 ? nd - 1 : L - 1;
        ck(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking), "stream");
        h->own_stream = true;
        if (const char *dbg = std::getenv("ST_DEBUG_SYNC")) h->debug_sync = dbg[0] == '1';
        if (const char *nr = std::getenv("ST_NODAL_RES")) h->nodal_res = std::atoi(nr);
        if (const char *md = std::getenv("ST_MK_DICT")) h->mk_dict = md[0] != '0';
        if (const char *sv = std::getenv("ST_STENCIL")) h->stencil = sv[0] != '0';
        size_t max_partial = 1;
        auto build = [&](int l, int b, int cnt, bool coarsest, bool alloc_x) {
            st::HostLevel &H = h->hl[l];
            DevLevel D;
            D.n_edges = H.mesh.n_edges; D.n_nodes = H.mesh.n_nodes; D.S = cnt; D.Q = Q;
            if ((long long)D.n_edges * D.S >= (1LL << 31) || (long long)D.n_nodes * 32 >= (1LL << 31))
                throw Unsupported("level too large for 32-bit thread indexing");
            D.M = h->upload(H.M); D.K = h->upload(H.K); D.Kn = h->upload(H.Kn); D.GT = h->upload(H.GT);
            D.GtM = h->upload(H.GtM);
            h->upload_mk(H.MK, H.MKk, H.M.width, D);
            D.dM = h->upload(H.dM); D.dK = h->upload(H.dK); D.dN = h->upload(H.dN);
            D.edge_nodes = h->upload(H.mesh.edge_nodes);
            D.sched_e = h->upload(H.sched_e); D.bptr_e = h->upload(H.bptr_e);
            D.sched_n = h->upload(H.sched_n); D.bptr_n = h->upload(H.bptr_n);
            D.nbox_e = (int)H.bptr_e.size() - 1; D.nbox_n = (int)H.bptr_n.size() - 1;
            D.tau = h->upload(std::vector<double>(H.tau.begin() + b, H.tau.begin() + b + cnt));
            // structured stencil march (stencil.cuh) on class-uniform hex levels whose slab count
            // fills whole warps; env ST_STENCIL=0 keeps the ELL kernels (measurements)
            if (h->stencil && o.kernel_path == 0 && (Q == 1 || Q == 2) && cnt % 32 == 0 && H.uniform &&
                H.mesh.dim == 3) {
                auto tab = std::make_unique<st::StencilTab>();
                if (st::build_stencil_tab(H, *tab)) {
                    D.use_stencil = true;
                    D.st_tab = tab.get();
                    h->st_tabs.push_back(std::move(tab));
                    D.grid.nx = H.mesh.n[0]; D.grid.ny = H.mesh.n[1]; D.grid.nz = H.mesh.n[2];
                    D.grid.Ex = H.mesh.Ex; D.grid.Ey = H.mesh.Ey;
                    D.st_cpl = h->dalloc<double>((size_t)D.n_edges * (cnt / 32));
                    D.st_bslab = h->dalloc<double>((size_t)D.n_edges * (cnt / 32));
                    // structured node scan on the same levels (env ST_NODE_STENCIL=0: ELL k_node_scan)
                    const char *ns = std::getenv("ST_NODE_STENCIL");
                    auto ntab = std::make_unique<st::NodeTab>();
                    if ((!ns || std::atoi(ns) != 0) && st::build_node_tab(H, *ntab)) {
                        D.sn_tab = ntab.get();
                        h->sn_tabs.push_back(std::move(ntab));
                        D.sn_ctot = h->dalloc<double>((size_t)D.n_nodes * (cnt / 32));
                        D.sn_cc = h->dalloc<double>((size_t)D.n_nodes * (cnt / 32));
                    }
                }
            }
            D.space_coarsened = H.space_coarsened;
            if (const char *e = std::getenv("ST_EDGE_LPR")) D.lpr_log2 = std::max(0, std::min(5, std::atoi(e)));
            // the march uses 32-bit element offsets
            if (H.uniform && o.kernel_path == 1 && Q <= 2 && (long long)H.mesh.n_edges * Q * cnt < (1LL << 31)) {
                const double hx = H.hbox[0], hy = H.hbox[1], hz = H.hbox[2];
                D.use_march = true;
                D.grid.nx = H.mesh.n[0]; D.grid.ny = H.mesh.n[1]; D.grid.nz = H.mesh.n[2];
                D.grid.Ex = H.mesh.Ex; D.grid.Ey = H.mesh.Ey;
                D.grid.mx = hy * hz / hx; D.grid.my = hx * hz / hy; D.grid.mz = hx * hy / hz;
                D.grid.wx = hx / (hy * hz); D.grid.wy = hy / (hx * hz); D.grid.wz = hz / (hx * hy);
                D.grid.sigma = h->upload(H.sigma);
                D.grid.nu = h->upload(H.nu);
            }
            if (!coarsest && l + 1 < L && cnt % 2 == 0) {
                const size_t per = (size_t)2 * Q * Q;
                D.Pt = h->upload(std::vector<double>(H.Pt.begin() + (b / 2) * per, H.Pt.begin() + ((b + cnt) / 2) * per));
            }
            if (!coarsest && l + 1 < L && H.space_coarsened) { D.Pg = h->upload(H.Pg); D.Rg = h->upload(H.Rg); }
            if (coarsest) {
                D.Ainv = h->upload(std::vector<double>(H.Ainv.begin() + (size_t)b * Q * D.n_edges * Q * D.n_edges,
                                                       H.Ainv.begin() + (size_t)(b + cnt) * Q * D.n_edges * Q * D.n_edges));
                if ((size_t)Q * D.n_edges * sizeof(double) > 48 * 1024) throw Unsupported("coarsest level too large");
            }
            const size_t ve = vec_len(D, Q), vn = vec_len(D, Q, true);
            if (alloc_x) { D.x = h->dalloc<double>(ve); D.f = h->dalloc<double>(ve); }
            D.r = h->dalloc<double>(ve);
            D.z = o.nu_s > 2 ? h->dalloc<double>(ve) : D.r;   // r and z are never live together for nu_s <= 2
            if (o.nu_s > 2) D.z2 = h->dalloc<double>(ve);
            D.zn = h->dalloc<double>(vn);
            D.y = h->dalloc<double>(vn);
            if (o.nu_n > 2) { D.wn = h->dalloc<double>(vn); D.zn2 = h->dalloc<double>(vn); }
            max_partial = std::max(max_partial, (ve + 255) / 256);
            max_partial = std::max(max_partial, (size_t)st::residual_partials(D));
            return D;
        };
        for (int l = 0; l <= h->g0; ++l) {
            const int cnt = (int)h->hl[l].tau.size() / P;
            h->dl.push_back(build(l, h->rank * cnt, cnt, P == 1 && l == L - 1, l > 0));
        }
        if (P > 1 && h->rank == 0)
            for (int l = h->g0; l < L; ++l) h->dg.push_back(build(l, 0, (int)h->hl[l].tau.size(), l == L - 1, true));
        if (o.inner == 1) {
            // inner spatial V-cycle (R13): the chain operators are uploaded once and shared by
            // every smoothing level; each level gets its own vectors on its chain segment
            std::vector<st::HostLevel> chain;
            st::build_chain(h->hl[0], chain);
            std::vector<DevLevel> ops;
            for (auto &C : chain) {
                DevLevel D;
                D.n_edges = C.mesh.n_edges; D.n_nodes = C.mesh.n_nodes; D.Q = Q;
                D.M = h->upload(C.M); D.K = h->upload(C.K); D.GT = h->upload(C.GT); D.GtM = h->upload(C.GtM);
                h->upload_mk(C.MK, C.MKk, C.M.width, D);
                D.dM = h->upload(C.dM); D.dK = h->upload(C.dK); D.dN = h->upload(C.dN);
                D.edge_nodes = h->upload(C.mesh.edge_nodes);
                D.sched_e = h->upload(C.sched_e); D.bptr_e = h->upload(C.bptr_e);
                D.sched_n = h->upload(C.sched_n); D.bptr_n = h->upload(C.bptr_n);
                D.nbox_e = (int)C.bptr_e.size() - 1; D.nbox_n = (int)C.bptr_n.size() - 1;
                if (C.space_coarsened) { D.Pg = h->upload(C.Pg); D.Rg = h->upload(C.Rg); }
                if (const char *e = std::getenv("ST_EDGE_LPR")) D.lpr_log2 = std::max(0, std::min(5, std::atoi(e)));
                ops.push_back(D);
            }
            auto attach = [&](std::vector<DevLevel> &levels, int l0) {
                for (size_t i = 0; i < levels.size(); ++i) {
                    DevLevel &D = levels[i];
                    const int l = l0 + (int)i;
                    if (D.Ainv) continue;   // the coarsest level solves exactly
                    int ci = 0;
                    for (int k = 0; k < l; ++k) ci += h->hl[k].space_coarsened ? 1 : 0;
                    std::vector<DevLevel> V;
                    for (int c = ci; c < (int)ops.size(); ++c) {
                        DevLevel I = ops[c];
                        I.S = D.S; I.tau = D.tau;
                        const size_t ve = vec_len(I, Q), vn = vec_len(I, Q, true);
                        if (c == ci) {
                            I.r = D.r;
                            I.z = h->dalloc<double>(ve);
                        } else {
                            I.r = h->dalloc<double>(ve);
                            I.z = h->dalloc<double>(ve);
                        }
                        I.z2 = h->dalloc<double>(ve);
                        I.y = h->dalloc<double>(vn);
                        V.push_back(I);
                    }
                    if (ops[ci].n_edges != D.n_edges) throw std::logic_error("spatial chain does not match the level mesh");
                    D.inner_id = (int)h->inner.size();
                    h->inner.push_back(std::move(V));
                }
            };
            attach(h->dl, 0);
            attach(h->dg, h->g0);
        }
        for (st::HostLevel &H : h->hl) {   // the device owns the operators now; keep the metadata
            H.M = H.K = H.Kn = H.GT = H.Pg = H.Rg = H.GtM = H.MK = st::HostELL();
            std::vector<double>().swap(H.MKk);
            std::vector<double>().swap(H.Ainv);
            std::vector<double>().swap(H.Pt);
            std::vector<int>().swap(H.mesh.cell_edges);
            std::vector<int>().swap(H.mesh.cell_nodes);
            std::vector<int>().swap(H.mesh.edge_nodes);
            std::vector<int>().swap(H.sched_e); std::vector<int>().swap(H.sched_n);
        }
        h->partial = h->dalloc<double>(max_partial);
        h->partial_cap = (int)max_partial;
        h->dscal = h->dalloc<double>(2);
        h->n_dofs = (int64_t)h->dl[0].n_edges * Q * h->dl[0].S;
        ck(cudaDeviceSynchronize(), "setup sync");
    } catch (const Unsupported &e) {
        delete h; return fail(3, e.what());
    } catch (const CudaError &e) {
        delete h; return fail(2, e.what());
    } catch (const std::bad_alloc &) {
        delete h; return fail(4, "out of memory");
    } catch (const std::length_error &e) {
        delete h; return fail(3, e.what());
    } catch (const std::exception &e) {
        delete h; return fail(1, e.what());
    }
    *out = h;
    return 0;
}

int st_free(st_handle *h) {
    if (!h) return 0;
    if (h->stream) cudaStreamSynchronize(h->stream);   // the user's stream too
    if (h->stream && h->own_stream) cudaStreamDestroy(h->stream);
    h->stream = nullptr;
    delete h;
    return 0;
}

int st_set_stream(st_handle *h, void *stream) {
    if (!h) return fail(1, "null handle");
    if (h->stream && h->own_stream) cudaStreamDestroy(h->stream);
    h->stream = (cudaStream_t)stream;
    h->own_stream = false;
    return 0;
}

int st_residual(st_handle *h, const double *x, const double *f, double *r, double *norms) {
    if (!h || !x || !f) return fail(1, "null argument");
    ST_CHECK_ALIGNED(x, f, r);
    ST_GUARD({
        DevLevel &L = h->dl[0];
        x_unknown(L);               // the caller may have changed x since the last call
        auto s = (st::Stream)h->stream;
        if (r) {
            st::launch_residual(s, L, h->kt, h->Q, x, f, nullptr, r, nullptr, h->o.omega_s, nullptr);
            h->launches += 1;
        }
        if (norms) {
            norms[0] = std::sqrt(residual_norm2(h, x, f));
            norms[1] = std::sqrt(norm2_plain(h, f, vec_len(L, h->Q)));
        }
    })
}

int st_vcycle(st_handle *h, double *x, const double *f) {
    if (!h || !x || !f) return fail(1, "null argument");
    ST_CHECK_ALIGNED(x, f);
    if (h->nranks > 1) return fail(1, "multi-rank handles run the V-cycle through the st_lv_* level operations");
    ST_GUARD(run_vcycle(h, x, f))
}

int st_set_graphs(st_handle *h, int enable) {
    if (!h) return fail(1, "null handle");
    if (enable && h->nranks > 1) return fail(1, "graphs apply to the single-process V-cycle only");
    ST_GUARD({
        ck(cudaStreamSynchronize(h->stream), "sync");
        h->clear_graphs();
        h->use_graphs = enable != 0;
    })
}

int st_solve(st_handle *h, double *x, const double *f, double tol, int maxit, int *iters, double *hist) {
    if (!h || !x || !f || maxit < 0) return fail(1, "bad argument");
    ST_CHECK_ALIGNED(x, f);
    if (h->nranks > 1) return fail(1, "multi-rank handles solve through paper_1911_09548_b200.distributed");
    ST_GUARD({
        x_unknown(h->dl[0]);
        if (tol <= 0.0 && !hist) {
            // no stopping test and no history requested: exactly maxit V-cycles, no norms
            for (int it = 0; it < maxit; ++it) run_vcycle(h, x, f);
            if (iters) *iters = maxit;
            return 0;
        }
        const double nf = std::sqrt(norm2_plain(h, f, vec_len(h->dl[0], h->Q)));
        int it = 0;
        for (;; ++it) {
            const double rel = std::sqrt(residual_norm2(h, x, f)) / nf;
            if (hist) hist[it] = rel;
            if (rel <= tol || it == maxit) break;
            run_vcycle(h, x, f);
        }
        if (iters) *iters = it;
    })
}

int st_solve_host(st_handle *h, double *x_host, const double *f_host, double tol, int maxit, int *iters,
                  double *hist) {
    if (!h || !x_host || !f_host) return fail(1, "null argument");
    ST_GUARD({
        const size_t n = vec_len(h->dl[0], h->Q);
        if (!h->hx) { h->hx = h->dalloc<double>(n); h->hf = h->dalloc<double>(n); }
        ck(cudaMemcpyAsync(h->hf, f_host, n * sizeof(double), cudaMemcpyHostToDevice, h->stream), "h2d f");
        ck(cudaMemcpyAsync(h->hx, x_host, n * sizeof(double), cudaMemcpyHostToDevice, h->stream), "h2d x");
        int rc = st_solve(h, h->hx, h->hf, tol, maxit, iters, hist);
        if (rc) throw CudaError(g_err);
        ck(cudaMemcpyAsync(x_host, h->hx, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream), "d2h x");
        ck(cudaStreamSynchronize(h->stream), "sync");
    })
}

int st_solve_many_host(st_handle *h, int n, double *const *x_host, const double *const *f_host, int init_from_x,
                       double tol, int maxit, int *iters, double *hist) {
    if (!h || n < 0 || maxit < 0 || (n > 0 && (!x_host || !f_host))) return fail(1, "bad argument");
    if (h->nranks > 1) return fail(1, "multi-rank handles solve through paper_1911_09548_b200.distributed");
    for (int i = 0; i < n; ++i)
        if (!x_host[i] || !f_host[i]) return fail(1, "null problem buffer");
    ST_GUARD({
        const size_t len = vec_len(h->dl[0], h->Q);
        const size_t bytes = len * sizeof(double);
        if (!h->mx[0]) {
            for (int b = 0; b < 2; ++b) {
                h->mx[b] = h->dalloc<double>(len);
                h->mf[b] = h->dalloc<double>(len);
                ck(cudaEventCreateWithFlags(&h->ev_in[b], cudaEventDisableTiming), "event");
                ck(cudaEventCreateWithFlags(&h->ev_done[b], cudaEventDisableTiming), "event");
                ck(cudaEventCreateWithFlags(&h->ev_out[b], cudaEventDisableTiming), "event");
            }
            ck(cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking), "stream");
            ck(cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking), "stream");
        }
        // f buffer b is free for problem i once problem i-2's solve is done; x buffer b once
        // problem i-2's D2H copy is done too (only the x copy / the zeroing waits for that, so
        // the H2D of f never queues behind the previous D2H)
        auto load = [&](int i) {
            const int b = i & 1;
            ck(cudaStreamWaitEvent(h->h2d, h->ev_done[b], 0), "wait");
            ck(cudaMemcpyAsync(h->mf[b], f_host[i], bytes, cudaMemcpyHostToDevice, h->h2d), "h2d f");
            if (init_from_x) {
                ck(cudaStreamWaitEvent(h->h2d, h->ev_out[b], 0), "wait");
                ck(cudaMemcpyAsync(h->mx[b], x_host[i], bytes, cudaMemcpyHostToDevice, h->h2d), "h2d x");
            }
            ck(cudaEventRecord(h->ev_in[b], h->h2d), "record");
        };
        if (n > 0) load(0);
        for (int i = 0; i < n; ++i) {
            const int b = i & 1;
            if (i + 1 < n) load(i + 1);          // enqueued before this solve blocks on its norms
            ck(cudaStreamWaitEvent(h->stream, h->ev_in[b], 0), "wait");
            ck(cudaStreamWaitEvent(h->stream, h->ev_out[b], 0), "wait");
            if (!init_from_x) ck(cudaMemsetAsync(h->mx[b], 0, bytes, h->stream), "memset");
            int rc = st_solve(h, h->mx[b], h->mf[b], tol, maxit, iters ? iters + i : nullptr,
                              hist ? hist + (size_t)i * (maxit + 1) : nullptr);
            if (rc) throw CudaError(g_err);
            ck(cudaEventRecord(h->ev_done[b], h->stream), "record");
            ck(cudaStreamWaitEvent(h->d2h, h->ev_done[b], 0), "wait");
            ck(cudaMemcpyAsync(x_host[i], h->mx[b], bytes, cudaMemcpyDeviceToHost, h->d2h), "d2h x");
            ck(cudaEventRecord(h->ev_out[b], h->d2h), "record");
        }
        ck(cudaStreamSynchronize(h->d2h), "sync");
        ck(cudaStreamSynchronize(h->h2d), "sync");
    })
}

static void parse_options(const st_params *p, st::Options &o);

int st_profile(st_handle *h, int enable) {
    if (!h) return fail(1, "null handle");
    ST_GUARD({
        ck(cudaStreamSynchronize(h->stream), "sync");
        if (enable) {   // a fresh record: recycle the old events (recs and pool stay disjoint)
            for (auto &r : h->recs) { h->pool.push_back(r.a); h->pool.push_back(r.b); }
            h->recs.clear();
        }
        h->prof = enable != 0;
    })
}

int st_profile_read(st_handle *h, st_kstat *out, int max, int *n) {
    if (!h || !n) return fail(1, "null argument");
    ST_GUARD({
        ck(cudaStreamSynchronize(h->stream), "sync");
        std::vector<st_kstat> agg(h->fams.size());
        for (size_t i = 0; i < agg.size(); ++i) {
            std::memset(&agg[i], 0, sizeof(st_kstat));
            std::strncpy(agg[i].name, h->fams[i].c_str(), sizeof(agg[i].name) - 1);
        }
        for (auto &r : h->recs) {
            float ms = 0;
            ck(cudaEventElapsedTime(&ms, r.a, r.b), "elapsed");
            agg[r.fam].launches += 1;
            agg[r.fam].ms += ms;
            agg[r.fam].bytes += r.bytes;
        }
        *n = (int)agg.size();
        for (int i = 0; i < (int)agg.size() && i < max; ++i) out[i] = agg[i];
    })
}

int st_plan(const st_params *p, st_info_t *info) {
    if (!p || !info) return fail(1, "null argument");
    try {
        st::Options o;
        parse_options(p, o);
        st::TimeMats tm = st::time_matrices(p->q);
        std::vector<st::HostLevel> hl;
        st::build_hierarchy(*p, o, tm, hl);
        std::memset(info, 0, sizeof(*info));
        info->n_levels = (int)std::min<size_t>(32, hl.size());
        info->q = p->q;
        info->n_dofs = (int64_t)hl[0].mesh.n_edges * (p->q + 1) * p->n_slabs;
        for (int l = 0; l < info->n_levels; ++l) {
            info->level_n_edges[l] = hl[l].mesh.n_edges;
            info->level_n_nodes[l] = hl[l].mesh.n_nodes;
            info->level_n_slabs[l] = (int)hl[l].tau.size();
            info->level_space_coarsened[l] = hl[l].space_coarsened ? 1 : 0;
            info->level_lambda[l] = hl[l].lambda;
        }
        return 0;
    } catch (const std::exception &e) {
        return fail(1, e.what());
    }
}

int st_host_matrix(const st_params *p, int level, int which, int *rows, int *width, int *col, double *val) {
    if (!p || !rows || !width) return fail(1, "null argument");
    try {
        st::Options o;
        parse_options(p, o);
        st::TimeMats tm = st::time_matrices(p->q);
        std::vector<st::HostLevel> hl;
        st::build_hierarchy(*p, o, tm, hl);
        if (level < 0 || level >= (int)hl.size()) throw std::invalid_argument("level out of range");
        const st::HostLevel &L = hl[level];
        const st::HostELL *E = which == 0 ? &L.M : which == 1 ? &L.K : which == 2 ? &L.Kn : which == 3 ? &L.Pg : nullptr;
        if (!E) throw std::invalid_argument("which must be 0..3");
        if (which == 3 && !L.space_coarsened) throw std::invalid_argument("level does not coarsen space");
        *rows = E->rows; *width = E->width;
        if (col) std::memcpy(col, E->col.data(), sizeof(int) * E->col.size());
        if (val) std::memcpy(val, E->val.data(), sizeof(double) * E->val.size());
        return 0;
    } catch (const std::exception &e) {
        return fail(1, e.what());
    }
}

static std::vector<DevLevel> &level_set(st_handle *h, int set) {
    if (set == 0) return h->dl;
    if (set == 1 && !h->dg.empty()) return h->dg;
    throw std::invalid_argument("no such level set on this rank");
}

static DevLevel &level_of(st_handle *h, int set, int level) {
    auto &V = level_set(h, set);
    if (level < 0 || level >= (int)V.size()) throw std::invalid_argument("level out of range");
    return V[level];
}

int st_lv_count(const st_handle *hc, int set, int *n) {
    st_handle *h = const_cast<st_handle *>(hc);
    if (!h || !n) return fail(1, "null argument");
    *n = set == 0 ? (int)h->dl.size() : (set == 1 ? (int)h->dg.size() : 0);
    return 0;
}

int st_lv_get(const st_handle *hc, int set, int level, st_level_t *out) {
    st_handle *h = const_cast<st_handle *>(hc);
    if (!h || !out) return fail(1, "null argument");
    try {
        DevLevel &L = level_of(h, set, level);
        const int gl = set == 0 ? level : h->g0 + level;
        std::memset(out, 0, sizeof(*out));
        out->set = set; out->level = level; out->global_level = gl;
        out->n_slabs = L.S;
        out->slab0 = set == 0 ? h->rank * L.S : 0;
        out->n_edges = L.n_edges; out->n_nodes = L.n_nodes; out->q = h->Q - 1;
        out->coarsest = L.Ainv != nullptr;
        out->space_coarsened = L.space_coarsened;
        out->x = L.x; out->f = L.f; out->r = L.r;
        return 0;
    } catch (const std::exception &e) {
        return fail(1, e.what());
    }
}

int st_lv_residual(st_handle *h, int set, int level, const double *x, const double *f, const double *prev, double *r,
                   double *norm2) {
    if (!h || !x || !f) return fail(1, "null argument");
    ST_CHECK_ALIGNED(x, f, r);
    ST_GUARD({
        DevLevel &L = level_of(h, set, level);
        x_unknown(L);               // level operations: the driver moves x between calls
        auto s = (st::Stream)h->stream;
        const int Q = h->Q;
        if (r) h->run("residual", 3 * evec(L, Q) + op_bytes(L), 1, [&] { st::launch_residual(s, L, h->kt, Q, x, f, prev, r, nullptr, h->o.omega_s, nullptr); });
        if (norm2) {
            int g = 0;
            h->run("residual_norm", 2 * evec(L, Q) + op_bytes(L), 1,
                   [&] { g = st::launch_residual(s, L, h->kt, Q, x, f, prev, nullptr, nullptr, h->o.omega_s, h->partial); });
            h->run("reduce", 8.0 * g, 1, [&] { st::launch_reduce(s, g, h->partial, h->dscal); });
            ck(cudaMemcpyAsync(norm2, h->dscal, sizeof(double), cudaMemcpyDeviceToHost, h->stream), "norm d2h");
            ck(cudaStreamSynchronize(h->stream), "sync");
        }
    })
}

int st_lv_smooth_S(st_handle *h, int set, int level, double *x, const double *f, const double *prev) {
    if (!h || !x || !f) return fail(1, "null argument");
    ST_CHECK_ALIGNED(x, f);
    ST_GUARD({
        DevLevel &L = level_of(h, set, level);
        x_unknown(L);
        smooth_S(h, L, x, f, prev);
    })
}

int st_lv_correct_local(st_handle *h, int set, int level, double *x, const double *f, const double *prev, double *tot) {
    if (!h || !x || !f) return fail(1, "null argument");
    ST_CHECK_ALIGNED(x, f);
    ST_GUARD({
        DevLevel &L = level_of(h, set, level);
        x_unknown(L);
        correct_A_local(h, L, x, f, prev, tot);
    })
}

int st_lv_correct_apply(st_handle *h, int set, int level, double *x, const double *carry) {
    if (!h || !x) return fail(1, "null argument");
    ST_CHECK_ALIGNED(x);
    ST_GUARD(correct_A_apply(h, level_of(h, set, level), x, carry))
}

int st_lv_restrict(st_handle *h, int set, int level, const double *r, double *fc) {
    if (!h || !r || !fc) return fail(1, "null argument");
    ST_CHECK_ALIGNED(r, fc);
    ST_GUARD({
        auto &V = level_set(h, set);
        if (level < 0 || level + 1 >= (int)V.size()) throw std::invalid_argument("no coarser level in this set");
        restrict_to(h, V[level], V[level + 1], r, fc);
    })
}

int st_lv_prolong(st_handle *h, int set, int level, const double *xc, double *x) {
    if (!h || !xc || !x) return fail(1, "null argument");
    ST_CHECK_ALIGNED(xc, x);
    ST_GUARD({
        auto &V = level_set(h, set);
        if (level < 0 || level + 1 >= (int)V.size()) throw std::invalid_argument("no coarser level in this set");
        prolong_from(h, V[level], V[level + 1], xc, x);
    })
}

int st_lv_vcycle(st_handle *h, int set, int level, double *x, const double *f) {
    if (!h || !x || !f) return fail(1, "null argument");
    ST_CHECK_ALIGNED(x, f);
    ST_GUARD({
        auto &V = level_set(h, set);
        if (V.back().Ainv == nullptr) throw std::invalid_argument("this level set has no coarsest level");
        if (level < 0 || level >= (int)V.size()) throw std::invalid_argument("level out of range");
        x_unknown(V[level]);
        vcycle(h, V, level, x, f);
    })
}

int st_lv_end_values(st_handle *h, int set, int level, const double *x, double *out) {
    if (!h || !x || !out) return fail(1, "null argument");
    ST_GUARD({
        DevLevel &L = level_of(h, set, level);
        h->run("end_values", 16.0 * L.n_edges, 1, [&] { st::launch_end_values((st::Stream)h->stream, L.n_edges, h->Q, L.S, x, out); });
    })
}

int st_copy_slabs(st_handle *h, int rows, int q, int ns, double *dst, int dS, int dk0, const double *src, int sS, int sk0,
                  int add) {
    if (!h || !dst || !src || rows < 0 || ns < 0 || dk0 < 0 || sk0 < 0 || dk0 + ns > dS || sk0 + ns > sS)
        return fail(1, "bad argument");
    ST_GUARD(h->run("copy_slabs", 16.0 * rows * (q + 1) * ns, 1, [&] {
        st::launch_copy_slabs((st::Stream)h->stream, rows, q + 1, ns, dst, dS, dk0, src, sS, sk0, add != 0);
    }))
}

int st_zero(st_handle *h, double *ptr, int64_t n) {
    if (!h || (!ptr && n)) return fail(1, "null argument");
    ST_GUARD(ck(cudaMemsetAsync(ptr, 0, sizeof(double) * (size_t)n, h->stream), "memset"))
}

int st_vec_axpy(st_handle *h, int64_t n, double alpha, const double *x, double *y) {
    if (!h || n < 0 || (n && (!x || !y))) return fail(1, "bad argument");
    ST_GUARD(if (n) h->run("axpy", 24.0 * n, 1, [&] { st::launch_axpy((st::Stream)h->stream, (size_t)n, alpha, x, y); }))
}

int st_vec_sum_blocks(st_handle *h, int64_t n, int nb, const double *in, double *out) {
    if (!h || n < 0 || nb < 0 || (n && (!out || (nb && !in)))) return fail(1, "bad argument");
    ST_GUARD(if (n) h->run("sum_blocks", 8.0 * n * (nb + 1), 1,
                           [&] { st::launch_sum_blocks((st::Stream)h->stream, (size_t)n, nb, in, out); }))
}

int st_vec_norm2(st_handle *h, int64_t n, const double *v, double *out) {
    if (!h || n < 0 || !out || (n && !v)) return fail(1, "bad argument");
    if ((size_t)n > (size_t)h->partial_cap * 256) return fail(1, "vector longer than the handle's level vectors");
    ST_GUARD(*out = n ? norm2_plain(h, v, (size_t)n) : 0.0)
}

int st_sync(st_handle *h) {
    if (!h) return fail(1, "null handle");
    ST_GUARD(ck(cudaStreamSynchronize(h->stream), "sync"))
}

int st_info(const st_handle *h, st_info_t *info) {
    if (!h || !info) return fail(1, "null argument");
    std::memset(info, 0, sizeof(*info));
    info->n_levels = (int)std::min<size_t>(32, h->hl.size());
    info->q = h->Q - 1;
    info->n_dofs = h->n_dofs;
    for (int l = 0; l < info->n_levels; ++l) {
        info->level_n_edges[l] = h->hl[l].mesh.n_edges;
        info->level_n_nodes[l] = h->hl[l].mesh.n_nodes;
        info->level_n_slabs[l] = (int)h->hl[l].tau.size();
        info->level_space_coarsened[l] = h->hl[l].space_coarsened ? 1 : 0;
        info->level_lambda[l] = h->hl[l].lambda;
    }
    for (int l = 0; l < info->n_levels; ++l) {
        const DevLevel *D = l < (int)h->dl.size() ? &h->dl[l]
                          : (l - h->g0 < (int)h->dg.size() ? &h->dg[l - h->g0] : nullptr);
        info->level_matrix_free[l] = D && D->use_march ? 1 : 0;
    }
    info->kernel_launches = h->launches;
    info->device_bytes = h->bytes;
    return 0;
}

}  // extern "C"
