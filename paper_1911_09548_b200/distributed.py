"""Multi-GPU space-time V-cycle: one process per GPU, each owning a contiguous block of slabs.

The hot path stays in libst's kernels (GPU backend `GpuOps`, calling the st_lv_* level
operations of include/st.h); this module only sequences them around the collectives the
method needs (north star; "Only the application of L requires forward
communication for neighboring time nodes"):

  * before every residual (each S and A step, and the one before restriction): the trace of
    the previous rank's last slab (time node q, one value per edge) - a right shift over ranks;
  * the time integration Sigma_t of the nodal correction (Eq. 5): each rank scans its block with
    zero carry, the per-node block totals are all-gathered and rank r adds the sum of ranks < r
    (R2: Sigma_t is a prefix sum of s_k = (Ct^{-1} z_k)_q);
  * residual norms: all-reduce of the squared local norms;
  * the first level with fewer slabs than ranks: the residual is gathered onto rank 0, which
    runs the coarse levels alone (its "gathered" level set) and scatters the correction back.

Communication uses torch.distributed (NCCL on GPUs, gloo on CPU in tests/test_distributed.py,
where the same driver runs with the CPU oracle as backend).  The driver never computes: every
arithmetic step is a backend call (with GpuOps a libst kernel: level operations, the Sigma_t rank
carry st_vec_sum_blocks, the coarse-correction add st_vec_axpy, norms st_vec_norm2); torch only
moves memory (collectives, slab-block copies)."""
import torch
import torch.distributed as dist


class TorchComm:
    """Collectives over torch.distributed (any backend) on backend tensors.  With the gloo
    backend and CUDA tensors (tests running several ranks on one GPU), messages are staged
    through host memory; with NCCL they go device to device over NVLink."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.stage = dist.get_backend(group) == "gloo"

    def _out(self, t):
        return t.cpu() if (self.stage and t.is_cuda) else t

    def _back(self, t, like):
        return t.to(like.device) if t.device != like.device else t

    def shift_right(self, send):
        """Rank r sends `send` to r+1 and returns what r-1 sent (None on rank 0)."""
        s = self._out(send)
        recv = torch.empty_like(s) if self.rank > 0 else None
        ops = []
        if self.rank + 1 < self.size:
            ops.append(dist.P2POp(dist.isend, s, self.rank + 1, self.group))
        if self.rank > 0:
            ops.append(dist.P2POp(dist.irecv, recv, self.rank - 1, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return self._back(recv, send) if recv is not None else None

    def allgather(self, t):
        s = self._out(t)
        out = [torch.empty_like(s) for _ in range(self.size)]
        dist.all_gather(out, s, group=self.group)
        return [self._back(o, t) for o in out]

    def allreduce_sum(self, value, like):
        t = torch.tensor([value], dtype=torch.float64, device="cpu" if self.stage else like.device)
        dist.all_reduce(t, group=self.group)
        return float(t.item())

    def gather_to_root(self, t):
        s = self._out(t)
        if self.rank == 0:
            out = [s] + [torch.empty_like(s) for _ in range(1, self.size)]
            for r in range(1, self.size):
                dist.recv(out[r], r, group=self.group)
            return [self._back(o, t) for o in out]
        dist.send(s, 0, group=self.group)
        return None

    def scatter_from_root(self, parts, like):
        if self.rank == 0:
            for r in range(1, self.size):
                dist.send(self._out(parts[r].contiguous()), r, group=self.group)
            return parts[0]
        out = torch.empty_like(self._out(like))
        dist.recv(out, 0, group=self.group)
        return self._back(out, like)


class LocalComm:
    """Single-process stand-in for TorchComm (no collectives needed)."""
    rank, size = 0, 1


class DistributedVCycle:
    """V-cycle over the slab blocks of all ranks, same arithmetic as the
    single-process V-cycle of the library (levels, smoother order, transfers)."""

    def __init__(self, ops, comm, spec="SAS"):
        self.ops, self.comm, self.spec = ops, comm, spec
        self.g0 = ops.n_levels(0) - 1           # last distributed level

    # -- helpers ------------------------------------------------------------
    def halo(self, l, x):
        if self.comm.size == 1:
            return None
        return self.comm.shift_right(self.ops.end_values(l, x))

    def hybrid(self, l, x, f, pre):
        seq = self.spec if pre else self.spec[::-1]
        for ch in reversed(seq):                       # right to left
            prev = self.halo(l, x)
            if ch == "S":
                self.ops.smooth_S(l, x, f, prev)
            else:
                tot = self.ops.correct_local(l, x, f, prev)
                carry = None
                if self.comm.size > 1:
                    # Sigma_t across ranks (R2): the end values integrated over the ranks before
                    # this one, summed by a kernel in rank order
                    tots = self.comm.allgather(tot)
                    if self.comm.rank > 0:
                        carry = self.ops.carry(tots, self.comm.rank)
                self.ops.correct_apply(l, x, carry)

    def residual_norm2(self, x, f):
        local = self.ops.residual_norm2(0, x, f, self.halo(0, x))
        return self.comm.allreduce_sum(local, f) if self.comm.size > 1 else local

    def norm2(self, f):
        local = self.ops.norm2(f)
        return self.comm.allreduce_sum(local, f) if self.comm.size > 1 else local

    def solve(self, x, f, tol=1e-8, maxit=100):
        """V-cycles until ||f - L x|| <= tol ||f|| over all ranks (same stopping rule as st_solve)."""
        nf = self.norm2(f) ** 0.5
        hist = []
        for it in range(maxit + 1):
            hist.append(self.residual_norm2(x, f) ** 0.5 / nf)
            if hist[-1] <= tol or it == maxit:
                break
            self.vcycle(x, f)
        return len(hist) - 1, hist

    # -- the cycle ------------------------------------------------------------
    def vcycle(self, x, f):
        self.cycle(0, x, f)

    def cycle(self, l, x, f):
        ops = self.ops
        if self.comm.size == 1 and l == self.g0:
            ops.vcycle_set(0, l, x, f)                   # coarsest level of a single process
            return
        if l == self.g0 and ops.gathered_is_coarsest():
            # the coarsest level itself is distributed: gather f, solve on rank 0, scatter x
            fg = self.gather(l, f)
            xg = ops.gathered_vector(0, "x") if self.comm.rank == 0 else None
            if self.comm.rank == 0:
                ops.vcycle_set(1, 0, xg, fg)
            ops.assign(x, self.scatter(l, xg, x))
            return
        self.hybrid(l, x, f, True)
        r = ops.residual(l, x, f, self.halo(l, x))
        if l < self.g0:
            xc, fc = ops.level_vectors(l + 1)
            ops.restrict(0, l, r, fc)
            ops.zero(xc)
            self.cycle(l + 1, xc, fc)
            ops.prolong(0, l, xc, x)
        else:
            # l == g0: restriction pairs slabs of different ranks -> coarse levels on rank 0
            rg = self.gather(l, r)
            cg = None
            if self.comm.rank == 0:
                xc, fc = ops.gathered_vector(1, "x"), ops.gathered_vector(1, "f")
                ops.restrict(1, 0, rg, fc)
                ops.zero(xc)
                ops.vcycle_set(1, 1, xc, fc)
                cg = ops.gathered_vector(0, "r")
                ops.zero(cg)
                ops.prolong(1, 0, xc, cg)
            ops.add(x, self.scatter(l, cg, x))
        self.hybrid(l, x, f, False)

    # -- slab-block gather / scatter between set 0 level g0 and set 1 level 0 ----
    def gather(self, l, v):
        parts = self.comm.gather_to_root(v)
        if self.comm.rank != 0:
            return None
        return self.ops.join_slabs(parts)

    def scatter(self, l, vg, like):
        parts = self.ops.split_slabs(vg, self.comm.size) if self.comm.rank == 0 else None
        return self.comm.scatter_from_root(parts, like)


class _Dev:
    """Zero-copy torch view of a libst device buffer (__cuda_array_interface__)."""

    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": "<f8", "data": (ptr, False), "version": 3}


def device_view(ptr, shape):
    return torch.as_tensor(_Dev(ptr, tuple(shape)), device="cuda")


class GpuOps:
    """Backend over a multi-rank libst handle (paper_1911_09548_b200.Solver with rank/nranks)."""

    def __init__(self, solver):
        self.s = solver
        self.q = solver.q
        self._views = {}

    def n_levels(self, set_):
        return self.s.n_levels(set_)

    def _lv(self, set_, l):
        return self.s.level(set_, l)

    def _vec(self, set_, l, which):
        key = (set_, l, which)
        if key not in self._views:
            L = self._lv(set_, l)
            self._views[key] = device_view(getattr(L, which), (L.n_edges, self.q + 1, L.n_slabs))
        return self._views[key]

    def level_vectors(self, l):
        return self._vec(0, l, "x"), self._vec(0, l, "f")

    def gathered_vector(self, l, which):
        return self._vec(1, l, which)

    def gathered_is_coarsest(self):
        # the last distributed level g0 is the global coarsest level
        return self.s.n_levels(0) == self.s.info()["n_levels"]

    def end_values(self, l, x):
        L = self._lv(0, l)
        out = torch.empty(L.n_edges, dtype=torch.float64, device="cuda")
        self.s.lv("end_values", 0, l, x, out)
        return out

    def smooth_S(self, l, x, f, prev):
        self.s.lv("smooth_S", 0, l, x, f, prev)

    def correct_local(self, l, x, f, prev):
        L = self._lv(0, l)
        tot = torch.empty(L.n_nodes, dtype=torch.float64, device="cuda")
        self.s.lv("correct_local", 0, l, x, f, prev, tot)
        return tot

    def correct_apply(self, l, x, carry):
        self.s.lv("correct_apply", 0, l, x, carry)

    def residual(self, l, x, f, prev):
        r = self._vec(0, l, "r")
        self.s.lv("residual", 0, l, x, f, prev, r, None)
        return r

    def residual_norm2(self, l, x, f, prev):
        return self.s.lv_residual_norm2(0, l, x, f, prev)

    def restrict(self, set_, l, r, fc):
        self.s.lv("restrict", set_, l, r, fc)

    def prolong(self, set_, l, xc, x):
        self.s.lv("prolong", set_, l, xc, x)

    def vcycle_set(self, set_, l, x, f):
        self.s.lv("vcycle", set_, l, x, f)

    def zero(self, t):
        self.s.zero(t)

    def add(self, x, c):
        self.s.axpy(1.0, c, x)

    def assign(self, x, c):
        x.copy_(c)                      # a device copy (no arithmetic)

    def carry(self, tots, rank):
        out = torch.empty_like(tots[0])
        self.s.sum_blocks(torch.stack(tots[:rank]), rank, out)
        return out

    def norm2(self, v):
        return self.s.norm2(v)

    def join_slabs(self, parts):
        L = self._lv(1, 0)
        out = self._vec(1, 0, "f")
        ns = parts[0].shape[2]
        for r, p in enumerate(parts):
            self.s.copy_slabs(L.n_edges, ns, out, L.n_slabs, r * ns, p, ns, 0)
        return out

    def split_slabs(self, vg, P):
        L = self._lv(1, 0)
        ns = L.n_slabs // P
        parts = []
        for r in range(P):
            t = torch.empty((L.n_edges, self.q + 1, ns), dtype=torch.float64, device="cuda")
            self.s.copy_slabs(L.n_edges, ns, t, ns, 0, vg, L.n_slabs, r * ns)
            parts.append(t)
        return parts
