"""One-line-per-launch summary of `ncu --page raw --csv` exports: duration, DRAM bytes, achieved
DRAM GB/s, occupancy, issue / fp64 / LSU utilisation and the top stall reasons.

    python scripts/ncu_csv_summary.py raw1.csv [raw2.csv ...]
"""
import csv
import sys

KEYS = [("dur_ms", "gpu__time_duration.sum"), ("dram_rd", "dram__bytes_read.sum"), ("dram_wr", "dram__bytes_write.sum"),
        ("regs", "launch__registers_per_thread"), ("warps%", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("issue%", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        ("fp64%", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        ("lsu%", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
        ("dram%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"), ("grid", "launch__grid_size")]
SCALE = {"ms": 1.0, "us": 1e-3, "ns": 1e-6, "s": 1e3, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def main(paths):
    for p in paths:
        rows = list(csv.reader(open(p)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            d = {}
            for name, key in KEYS:
                if key in hdr:
                    i = hdr.index(key)
                    try:
                        d[name] = float(r[i]) * SCALE.get(units[i], 1.0)
                    except ValueError:
                        d[name] = r[i]
            ms = d["dur_ms"]
            gbs = (d["dram_rd"] + d["dram_wr"]) / (ms * 1e-3) / 1e9
            stalls = []
            for i, h in enumerate(hdr):
                if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                    try:
                        stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                    except ValueError:
                        pass
            stalls.sort(reverse=True)
            name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")[:48]
            print(f"{name:48s} {ms:7.3f} ms  DRAM {(d['dram_rd'] + d['dram_wr']) / 1e9:6.2f} GB = {gbs:6.0f} GB/s "
                  f"({d['dram%']:.0f}%)  regs {d['regs']:.0f} warps {d['warps%']:.0f}% issue {d['issue%']:.0f}% "
                  f"fp64 {d['fp64%']:.0f}% lsu {d['lsu%']:.0f}% | " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:4]))


if __name__ == "__main__":
    main(sys.argv[1:])
