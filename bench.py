"""bench.py — space-time dof-updates/s per V-cycle of the B200 space-time multigrid.

Contract: `python bench.py --gpus N --steps K --warmup W`
(N > 1 under torchrun, one rank per GPU).  A step is one V-cycle of the whole
hot path (all rows of DESIGN.md §0(a)) over the rank's slab block of the
BASELINE.json config 4 workload (64^3 hex mesh, 811,200 edges, dG(1),
tau = 1/4096, 512 slabs per GPU).  `--impl reference` times the CPU oracle on a
bounded sample of the same workload.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "space-time dof-updates/s per V-cycle"
UNIT = "dof-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--slabs", type=int, default=512, help="slabs per GPU (weak scaling)")
    ap.add_argument("--cells", type=int, default=64, help="cells per direction")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-out", default=None, help="write per-kernel event stats (json)")
    ap.add_argument("--kernel-path", type=int, default=0, help="0: assembled ELL (default), 1: matrix-free march")
    ap.add_argument("--inner", default="jacobi", choices=["jacobi", "mg"],
                    help="A_k^{-1} inside S: block-Jacobi sweeps (default) or the inner spatial V-cycle (R13)")
    return ap.parse_args()


def workload(args):
    return workloads.c4(n=args.cells, S=args.slabs, tau=1.0 / 4096)


def workload_name(args):
    return (f"c4: unit cube {args.cells}^3 hex, lowest-order Nedelec, dG(1), tau=1/4096, sigma=nu=1, "
            f"{args.slabs} slabs per GPU, f ~ U(-1,1) seed 3"
            + ("" if args.inner == "jacobi" else ", inner spatial V-cycle for A_k^{-1} (R13)"))


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(family):
    """(dram__bytes_read.sum + dram__bytes_write.sum, source) of the finest-level launch of the
    family's kernel in the committed `ncu --set full` capture of the bench command
    (profiles/r02_ncu_kernels.json, scripts/ncu_summary.py), or (None, why) when the capture was
    taken from other kernel sources than the ones built now (its source hash differs)."""
    sys.path.insert(0, os.path.join(ROOT, "scripts"))
    from srchash import srchash
    p = os.path.join(ROOT, "profiles", "r02_ncu_kernels.json")
    if not os.path.exists(p):
        return None, "no capture"
    cap = json.load(open(p))
    if cap.get("source_hash") != srchash():
        return None, f"capture {os.path.basename(p)} is of other kernel sources ({cap.get('source_hash')} vs {srchash()})"
    tags = {"residual": ("k_st_residual<", "k_residual<"), "sweep_update": ("k_st_sweep<", "k_sweep<"),
            "node_scan": ("k_sn_scan<", "k_node_scan<"), "gt": ("k_gt<",)}.get(family, ())

    def gb(v):
        val, unit = v.split()[:2]
        return float(val) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}.get(unit, 1.0)
    for d in cap["launches"]:
        if any(t in d["kernel"] for t in tags):
            return (gb(d["dram__bytes_read.sum"]) + gb(d["dram__bytes_write.sum"]),
                    f"{os.path.basename(p)} (source hash {cap['source_hash']}): {d['kernel'][:60]}, finest level")
    return None, "family not in the capture"


def link_bandwidth(torch, host, dev, stream, host2=None, dev2=None):
    """Pinned host <-> device copy bandwidth of this box per direction (GB/s), the bound of the
    e2e number: one full-vector copy each way alone, then both directions at once; CUDA events."""
    out = {}
    with torch.cuda.stream(stream):
        for name, dst, src in (("h2d", dev, host), ("d2h", host, dev)):
            dst.copy_(src, non_blocking=True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dst.copy_(src, non_blocking=True)
            e1.record(stream)
            stream.synchronize()
            out[name] = host.numel() * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9
    if host2 is not None:
        # both directions at once (what the pipelined e2e steps do): H2D host -> dev on one stream,
        # D2H dev2 -> host2 on another, each timed by its own events
        sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        stream.synchronize()
        for _ in range(2):                       # the second pass is the timed one
            with torch.cuda.stream(sa):
                ev[0].record(sa)
                dev.copy_(host, non_blocking=True)
                ev[1].record(sa)
            with torch.cuda.stream(sb):
                ev[2].record(sb)
                host2.copy_(dev2, non_blocking=True)
                ev[3].record(sb)
            sa.synchronize()
            sb.synchronize()
        out["h2d_both"] = host.numel() * 8 / (ev[0].elapsed_time(ev[1]) * 1e-3) / 1e9
        out["d2h_both"] = host.numel() * 8 / (ev[2].elapsed_time(ev[3]) * 1e-3) / 1e9
    return out


# ------------------------------------------------------------- CPU oracle
def oracle_sample(n=32, S=8):
    """Bounded sample of the c4 workload for the CPU oracle: n^3 cells, S slabs, same lambda = 1."""
    from oracle import mesh, multigrid as mg
    w = workloads.c4(n=n, S=S, tau=1.0 / (n * n))
    H = mg.Hierarchy(mesh.Mesh(w.n, w.node_coords()), w.sigma, w.nu, w.tau, w.q, mg.Options())
    F = workloads.to_oracle(w.rhs())
    return w, H, F


def time_oracle_vcycle(H, F, X):
    from oracle import multigrid as mg
    t = time.perf_counter()
    X = mg.vcycle(H, 0, X, F)
    return time.perf_counter() - t, X


def cpu_baseline():
    w, H, F = oracle_sample()
    dt, _ = time_oracle_vcycle(H, F, np.zeros_like(F))
    return {"value": F.size / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"one oracle V-cycle (numpy/scipy fp64, single-threaded sparse products) on the c4 recipe "
                      f"at {w.n[0]}^3 cells x {w.S} slabs (lambda = tau/h^2 = 1 as in c4), {F.size} dofs, "
                      f"{dt:.2f} s"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    w, H, F = oracle_sample()
    X = np.zeros_like(F)
    for _ in range(args.warmup):
        _, X = time_oracle_vcycle(H, F, X)
    ts = []
    for _ in range(args.steps):
        dt, X = time_oracle_vcycle(H, F, X)
        ts.append(dt)
    T = float(np.sum(ts))
    val = F.size * args.steps / T
    sample = (f"oracle V-cycle on the c4 recipe at {w.n[0]}^3 cells x {w.S} slabs (lambda = 1), "
              f"{F.size} dofs per step")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": sample},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


# ------------------------------------------------------------------- ours
def run_ours(args, rank, world, local_rank):
    import torch
    import paper_1911_09548_b200 as p
    torch.cuda.set_device(local_rank % torch.cuda.device_count())
    dist = None
    red_dev = "cuda"
    if world > 1:
        import torch.distributed as dist
        red_dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    # weak scaling: every rank owns `slabs` slabs of one global slab range (tau = 1/4096); with
    # N > 1 the V-cycle runs through paper_1911_09548_b200.distributed over NCCL (halo shift,
    # Sigma_t carries, coarse levels gathered on rank 0)
    w = workloads.c4(n=args.cells, S=args.slabs * world, tau=1.0 / 4096)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        s = p.Solver.from_workload(w, stream=stream, rank=rank, nranks=world, kernel_path=args.kernel_path,
                                   inner=args.inner)
        g = torch.Generator(device="cuda")
        g.manual_seed(3 + 1000 * rank)
        f = torch.empty(s.shape, dtype=torch.float64, device="cuda").uniform_(-1.0, 1.0, generator=g)
        x = torch.zeros_like(f)
        n_dofs = f.numel()
        if world > 1:
            from paper_1911_09548_b200.distributed import DistributedVCycle, GpuOps, TorchComm
            drv = DistributedVCycle(GpuOps(s), TorchComm())
            step = lambda: drv.vcycle(x, f)   # noqa: E731
        else:
            step = lambda: s.vcycle(x, f)     # noqa: E731
        for _ in range(args.warmup):
            step()
        stream.synchronize()
        if dist:
            dist.barrier()
        launches0 = s.info()["kernel_launches"]
        s.profile(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local_rank % torch.cuda.device_count()) as clk:
            stream.synchronize()
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
            stream.synchronize()
        ms = e0.elapsed_time(e1)
        kstats = s.profile_read()
        s.profile(False)
        launches = s.info()["kernel_launches"] - launches0
        t_max = ms
        if dist:
            t = torch.tensor([ms], device=red_dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_max = float(t.item())
        # end to end through the public API with host buffers: st_solve_host copies f and x in,
        # runs the V-cycle (+ its residual norms) and copies x back, all inside the call
        e2e = None
        if not args.no_e2e:
            fh = f.cpu().pin_memory()
            xh = torch.zeros(fh.shape, dtype=torch.float64).pin_memory()
            ke = max(1, min(args.steps, 3))
            if world == 1:
                # st_solve_many_host: per step (= problem) H2D f from pinned memory, x = 0, ||f||,
                # ||r||, one V-cycle, ||r||, D2H x; the copies of neighbouring steps overlap the solve
                xh2 = torch.zeros(fh.shape, dtype=torch.float64).pin_memory()
                s.solve_many_host([xh.numpy()], [fh.numpy()], tol=0.0, maxit=1, history=False)   # warm-up
                ke = max(20, args.steps)             # two pinned output buffers, reused alternately
                outs = [(xh if i % 2 == 0 else xh2).numpy() for i in range(ke)]
                t0 = time.perf_counter()
                s.solve_many_host(outs, [fh.numpy()] * ke, tol=0.0, maxit=1, history=False)
                te = (time.perf_counter() - t0) / ke
                note = (f"st_solve_many_host, {ke} steps in one call: per step H2D f from pinned memory, x = 0, "
                        "one V-cycle (tol = 0: no norms), D2H x; copies of neighbouring steps overlap the V-cycles "
                        "(the first H2D and the last D2H are not hidden and are included)")
            else:
                def e2e_step():
                    f.copy_(fh, non_blocking=True)
                    x.copy_(xh, non_blocking=True)
                    drv.vcycle(x, f)
                    xh.copy_(x, non_blocking=True)
                    stream.synchronize()
                e2e_step()
                dist.barrier()
                t0 = time.perf_counter()
                for _ in range(ke):
                    e2e_step()
                te = (time.perf_counter() - t0) / ke
                note = "per rank: H2D f,x from pinned memory, distributed V-cycle, D2H x"
            if dist:
                t = torch.tensor([te], device=red_dev, dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                te = float(t.item())
            link = link_bandwidth(torch, fh, f, stream, xh, x)
            h2d_b = (1 if world == 1 else 2) * f.numel() * 8
            d2h_b = f.numel() * 8
            # the copy bound of a fully pipelined step: the slower direction at the link speed measured
            # with both directions busy (the steady state of the pipeline)
            t_copy = max(h2d_b / (link["h2d_both"] * 1e9), d2h_b / (link["d2h_both"] * 1e9)) if link else None
            e2e = {"value": n_dofs * world / te, "unit": UNIT,
                   "h2d_bytes_per_step": h2d_b * world, "d2h_bytes_per_step": d2h_b * world, "note": note,
                   "link_GBps": link,
                   "copy_bound_value": (n_dofs * world / t_copy) if t_copy else None}
    info = s.info()
    s.close()
    torch.cuda.synchronize()
    if rank != 0:
        return
    peak, peak_src = measured_peak()
    fam, (nl, kms, kbytes) = max(kstats.items(), key=lambda kv: kv[1][1])
    traffic, traffic_src = ncu_traffic(fam) if (args.cells, args.slabs, world) == (64, 512, 1) else \
        (None, "capture is of the default 64^3 x 512-slab configuration")
    dur = kms / nl
    achieved = kbytes / nl / (dur * 1e-3) / 1e9
    total_bytes = sum(v[2] for v in kstats.values())
    value = n_dofs * world * args.steps / (t_max * 1e-3)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args), "rhs": "U(-1,1) drawn on the device (torch generator, seed 3 + 1000 rank)", "n_edges": s.n_edges, "slabs_per_gpu": args.slabs,
                   "dofs_per_gpu": n_dofs, "levels": info["n_levels"],
                   "matrix_free_levels": sum(info["level_matrix_free"]),
                   "l2": f"no flush: every space-time vector is {8 * n_dofs / 1e9:.2f} GB >> 126 MB L2",
                   "parallelism": f"time-slab blocks over {world} GPU(s) (NCCL halo/carry/norm collectives)"
                   if world > 1 else "single GPU"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_src, "kernel": fam, "peak_source": peak_src,
                     "kernel_share_of_step": kms / t_max,
                     "vcycle_algorithmic_GBps": total_bytes / (t_max * 1e-3) / 1e9},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "e2e": e2e,
        "kernels": {k: {"launches": v[0], "ms": v[1], "GBps": v[2] / (v[1] * 1e-3) / 1e9 if v[1] else None}
                    for k, v in kstats.items()},
    }
    if not args.no_cpu_baseline and world == 1:
        out["cpu_baseline"] = cpu_baseline()
    if args.profile_out:
        with open(args.profile_out, "w") as fh:
            json.dump(out, fh, indent=1)
    print(json.dumps(out), flush=True)


def spawn(args):
    """`--gpus N` outside torchrun: launch N ranks of this script with torch.distributed.run (one
    process per GPU, rendezvous on 127.0.0.1) and return their exit code."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch.distributed as dist
        # NCCL over NVLink; ST_BENCH_BACKEND=gloo only to exercise this path with several ranks
        # on one GPU (host-staged messages; not a measurement configuration)
        dist.init_process_group(os.environ.get("ST_BENCH_BACKEND", "nccl"))
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
