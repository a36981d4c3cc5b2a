"""The multi-rank driver (paper_1911_09548_b200.distributed) with the CUDA level operations.

P = 1: the driver sequences the same kernels as st_vcycle -> bitwise equal result.
P = 2: two processes on the one GPU of this box with gloo messages staged through host memory
(no kernel ever waits on another process); each builds a multi-rank handle (its slab block,
rank 0 also the gathered coarse levels) and the gathered result must equal the single-process
V-cycle to rounding."""
import os
import socket

import numpy as np
import pytest
import torch

import workloads

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(w, seed=5):
    rng = np.random.default_rng(seed)
    F = workloads.from_oracle(rng.uniform(-1, 1, (w.S, w.q + 1, w.n_edges)))
    X0 = workloads.from_oracle(rng.uniform(-1, 1, (w.S, w.q + 1, w.n_edges)))
    return X0, F


@pytest.mark.parametrize("name", ["c1", "c5", "c2"])
def test_driver_single_rank_bitwise(name):
    import paper_1911_09548_b200 as p
    from paper_1911_09548_b200.distributed import DistributedVCycle, GpuOps, LocalComm
    from paper_1911_09548_b200 import build as _b
    _b.build()
    w = workloads.small(name)
    X0, F = _inputs(w)
    s = p.Solver.from_workload(w)
    xa = torch.from_numpy(X0).cuda()
    f = torch.from_numpy(F).cuda()
    xb = xa.clone()
    s.vcycle(xa, f)
    DistributedVCycle(GpuOps(s), LocalComm()).vcycle(xb, f)
    torch.cuda.synchronize()
    assert torch.equal(xa, xb)


def _worker(rank, P, port, name, out, opts=None):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        import paper_1911_09548_b200 as p
        from paper_1911_09548_b200.distributed import DistributedVCycle, GpuOps, TorchComm
        torch.cuda.set_device(0)
        w = workloads.small(name)
        X0, F = _inputs(w)
        s = p.Solver.from_workload(w, rank=rank, nranks=P, **(opts or {}))
        cnt = w.S // P
        x = torch.from_numpy(np.ascontiguousarray(X0[:, :, rank * cnt:(rank + 1) * cnt])).cuda()
        f = torch.from_numpy(np.ascontiguousarray(F[:, :, rank * cnt:(rank + 1) * cnt])).cuda()
        drv = DistributedVCycle(GpuOps(s), TorchComm())
        drv.vcycle(x, f)
        torch.cuda.synchronize()
        parts = drv.comm.gather_to_root(x)
        x.zero_()
        it, hist = drv.solve(x, f, tol=1e-10, maxit=5)
        variants = p.kernel_variants()
        gathered = [None] * P
        dist.all_gather_object(gathered, sorted(variants))
        if rank == 0:
            out.put((torch.cat([q.cpu() for q in parts], dim=2).numpy(), hist, gathered))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,P,opts", [("c1", 2, {}), ("c4", 2, {}), ("c5", 2, {}), ("c1", 4, {}),
                                         ("c4", 2, {"inner": "mg"}),
                                         # 32 slabs per rank: the stencil march with the previous
                                         # rank's end values as the upwind coupling of slab 0
                                         ("c4_s64", 2, {})])
def test_two_ranks_one_gpu(name, P, opts):
    import torch.multiprocessing as mp
    import paper_1911_09548_b200 as p
    from paper_1911_09548_b200 import build as _b
    _b.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, name, q, opts)) for r in range(P)]
    for pr in procs:
        pr.start()
    Xd, hist, variants = q.get(timeout=600)
    if name == "c4_s64":
        # rank 1 ran the stencil residual with rank 0's end values as its upwind coupling
        assert "stencil/residual" in variants[1] and "coupling/prev" in variants[1], variants
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    w = workloads.small(name)
    X0, F = _inputs(w)
    s = p.Solver.from_workload(w, **opts)
    x = torch.from_numpy(X0).cuda()
    f = torch.from_numpy(F).cuda()
    s.vcycle(x, f)
    Xs = x.cpu().numpy()
    tol = 1e-11 if name == "c5" else 1e-12          # same kernels, the halo only moves a trace
    assert np.linalg.norm(Xd - Xs) <= tol * np.linalg.norm(Xs)
    x.zero_()
    it, h1 = s.solve(x, f, tol=1e-10, maxit=5)
    np.testing.assert_allclose(hist, h1, rtol=1e-10, atol=1e-14)


def test_bench_two_ranks_one_gpu_gloo():
    # the N > 1 path of bench.py (DistributedVCycle timing, max over ranks, e2e) with two ranks on
    # one GPU: gloo instead of NCCL (ST_BENCH_BACKEND); rank 0 prints the JSON line
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, ST_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--slabs", "16", "--cells", "8", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0 and d["e2e"]["value"] > 0
