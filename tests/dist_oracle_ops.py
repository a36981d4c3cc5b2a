"""CPU oracle backend of paper_1911_09548_b200.distributed for the gloo tests (test-only).

Each rank holds its slab block of every distributed level as torch CPU tensors in ST layout
(n_edges, q+1, S_block); arithmetic is done by oracle functions on the block (with the
previous rank's trace as initial state), rank 0 additionally runs the global coarse levels
with the single-process oracle.  Used only by tests: the product path never imports oracle."""
import numpy as np
import torch

import workloads
from oracle import mesh, multigrid as mg, spacetime as sto, time_dg


def _np(t):
    return workloads.to_oracle(t.numpy())


def _put(t, X):
    t.copy_(torch.from_numpy(workloads.from_oracle(X)))


class OracleOps:
    def __init__(self, w, rank, P, **opts):
        self.w, self.rank, self.P = w, rank, P
        self.q, self.Q = w.q, w.q + 1
        self.opts = mg.Options(omega_s=w.omega_s, **opts)
        self.H = mg.Hierarchy(mesh.Mesh(w.n, w.node_coords()), w.sigma, w.nu, w.tau, w.q, self.opts)
        L = len(self.H.levels)
        nd = 0
        while nd < L and self.H.levels[nd].S >= P and self.H.levels[nd].S % P == 0:
            nd += 1
        self.g0 = nd - 1 if P > 1 else L - 1
        self.loc = []
        for l in range(self.g0 + 1):
            G = self.H.levels[l]
            cnt = G.S // P
            lv = sto.Level(G.mesh, G.sigma, G.nu, G.tau[rank * cnt:(rank + 1) * cnt], w.q, M=G.M, K=G.K, Kn=G.Kn)
            lv.slab0 = rank * cnt
            self.loc.append(lv)
        self.bufs = {}
        self._Y = {}
        self.g = np.linalg.inv(time_dg.time_matrices(w.q)[0])[:, 0]

    # -- structure ---------------------------------------------------------
    def n_levels(self, set_):
        return len(self.loc) if set_ == 0 else len(self.H.levels) - self.g0

    def gathered_is_coarsest(self):
        return self.g0 == len(self.H.levels) - 1

    def _shape(self, set_, l):
        lv = self.loc[l] if set_ == 0 else self.H.levels[self.g0 + l]
        return (lv.n, self.Q, lv.S)

    def _buf(self, set_, l, which):
        key = (set_, l, which)
        if key not in self.bufs:
            self.bufs[key] = torch.zeros(self._shape(set_, l), dtype=torch.float64)
        return self.bufs[key]

    def level_vectors(self, l):
        return self._buf(0, l, "x"), self._buf(0, l, "f")

    def gathered_vector(self, l, which):
        return self._buf(1, l, which)

    def _prev(self, l, prev):
        if prev is None:
            return None
        blk = np.zeros((self.Q, self.loc[l].n))
        blk[self.q] = prev.numpy()
        return blk

    # -- arithmetic (oracle functions on the rank's slab block) ---------------
    def end_values(self, l, x):
        return x[:, self.q, -1].clone()

    def _res(self, l, x, f, prev):
        return _np(f) - sto.apply_L(self.loc[l], _np(x), self._prev(l, prev))

    def smooth_S(self, l, x, f, prev):
        X = _np(x)
        _put(x, X + self.opts.omega * sto.apply_B(self.loc[l], self._res(l, x, f, prev), self.opts))

    def correct_local(self, l, x, f, prev):
        lv = self.loc[l]
        W = lv.spatial(lv.G.T.tocsr(), self._res(l, x, f, prev))
        Y = sto.sigma_t(lv, sto.Kn_inverse(lv, W, self.opts))      # block scan from a zero end value
        self._Y[l] = Y
        return torch.from_numpy(Y[-1, self.q].copy())

    def correct_apply(self, l, x, carry):
        lv = self.loc[l]
        Y = self._Y.pop(l)
        if carry is not None:
            Y = Y + self.g[None, :, None] * carry.numpy()[None, None, :]
        _put(x, _np(x) + lv.spatial(lv.G, Y))

    def residual(self, l, x, f, prev):
        r = self._buf(0, l, "r")
        _put(r, self._res(l, x, f, prev))
        return r

    def residual_norm2(self, l, x, f, prev):
        return float(np.sum(self._res(l, x, f, prev) ** 2))

    def _theta(self, set_, l):
        lv = self.loc[l] if set_ == 0 else self.H.levels[self.g0 + l]
        return lv.tau[0::2] / (lv.tau[0::2] + lv.tau[1::2])

    def restrict(self, set_, l, r, fc):
        gl = l if set_ == 0 else self.g0 + l
        R = _np(r)
        th = self._theta(set_, l)
        S, Q, n = R.shape
        Fc = np.zeros((S // 2, Q, n))
        for K in range(S // 2):
            Fc[K] = time_dg.prolongation(self.q, th[K]).T @ R[2 * K:2 * K + 2].reshape(2 * Q, n)
        Pe = self.H.P_edge[gl]
        if Pe is not None:
            Fc = self.H.levels[gl].spatial(Pe.T.tocsr(), Fc)
        _put(fc, Fc)

    def prolong(self, set_, l, xc, x):
        gl = l if set_ == 0 else self.g0 + l
        Xc = _np(xc)
        Pe = self.H.P_edge[gl]
        if Pe is not None:
            Xc = self.H.levels[gl].spatial(Pe, Xc)
        th = self._theta(set_, l)
        Sc, Q, n = Xc.shape
        Xf = np.zeros((2 * Sc, Q, n))
        for K in range(Sc):
            Xf[2 * K:2 * K + 2] = (time_dg.prolongation(self.q, th[K]) @ Xc[K]).reshape(2, Q, n)
        _put(x, _np(x) + Xf)

    def vcycle_set(self, set_, l, x, f):
        gl = l if set_ == 0 else self.g0 + l
        X = _np(x) if gl < len(self.H.levels) - 1 else np.zeros(_np(f).shape)
        _put(x, mg.vcycle(self.H, gl, X, _np(f)))

    def zero(self, t):
        t.zero_()

    def add(self, x, c):
        x += c

    def carry(self, tots, rank):
        out = tots[0].clone()
        for t in tots[1:rank]:
            out += t
        return out

    def norm2(self, v):
        return float((v * v).sum())

    def assign(self, x, c):
        x.copy_(c)

    def join_slabs(self, parts):
        out = self._buf(1, 0, "f")
        ns = parts[0].shape[2]
        for r, p in enumerate(parts):
            out[:, :, r * ns:(r + 1) * ns] = p
        return out

    def split_slabs(self, vg, P):
        ns = vg.shape[2] // P
        return [vg[:, :, r * ns:(r + 1) * ns].contiguous() for r in range(P)]
