"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of a bench.py run:
per-kernel launches / device time / share over the timed V-cycles, next to bench.py's own
CUDA-event family shares from the plain run of the same command.

    python scripts/launch_summary.py launches.csv plain_bench.log steps > profiles/…txt
"""
import collections
import csv
import io
import json
import re
import sys


def main(csv_path, bench_log, steps):
    lines = [l for l in open(csv_path) if not l.startswith("==")]
    rows = [r for r in csv.DictReader(io.StringIO("".join(lines))) if r["Metric Name"] == "gpu__time_duration.sum"]
    ours = [r for r in rows if "st::" in r["Kernel Name"]]
    ends = [i for i, r in enumerate(ours) if "k_coarsest" in r["Kernel Name"]]   # last launch of a V-cycle
    timed = ours[ends[-steps - 1] + 1: ends[-1] + 1]
    agg = {}
    for r in timed:
        k = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "")[:60]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(r["Metric Value"]) / 1e6
    tot = sum(v[1] for v in agg.values())
    d = json.loads(open(bench_log).read().strip().splitlines()[-1])
    print(f"# ncu launch list of `bench.py --steps {steps} --warmup 3 --no-cpu-baseline --no-e2e`: the {steps} timed V-cycles, "
          f"{len(timed)} launches ({len(timed) // steps} per V-cycle; bench.py gpu_launches {d['gpu_launches']})")
    print("# cold-cache serialised per-launch times: compare SHARES with bench.py's live event shares")
    print("%-60s %9s %10s %6s" % ("kernel", "launches", "ms", "share"))
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print("%-60s %9d %10.3f %5.1f%%" % (k, v[0], v[1], 100 * v[1] / tot))
    print("total %.1f ms = %.1f ms / V-cycle serialised; bench.py (CUDA events, same command without ncu): %.1f ms / V-cycle"
          % (tot, tot / steps, d["ms_per_step"]))
    ev = sum(v["ms"] for v in d["kernels"].values())
    # launch_res_mass / launch_residual run their chunk-coupling pre-passes inside the family's events
    # (k_st_bslab, k_st_coupling: counted with the residual here, where most of them run)
    tags = {"residual": ("k_residual", "k_st_residual", "k_st_bslab", "k_st_coupling"),
            "sweep_update": ("k_sweep", "k_st_sweep"),
            "gtr_mass": ("k_res_mass", "k_st_res_mass", "k_gtr"), "node_scan": ("k_node_scan", "k_sn_scan", "k_sn_carry"),
            "gt": ("k_gt<",),
            "g_update": ("k_g_update",), "prolong": ("k_prolong",), "restrict": ("k_restrict",)}
    print("family shares, ncu / live events: " + ", ".join(
        "%s %.1f%% / %.1f%%" % (f, 100 * sum(v[1] for k, v in agg.items() if any(x in k for x in t)) / tot,
                                100 * d["kernels"][f]["ms"] / ev)
        for f, t in tags.items() if f in d["kernels"]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]))
