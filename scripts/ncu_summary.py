"""Summarise an `ncu --set full` report into profiles/<name>.json: per captured launch the kernel,
grid, duration and DRAM bytes, plus the source hash of the kernels that produced it (bench.py only
quotes the capture's DRAM traffic when that hash equals the hash of the current csrc/ sources).

    python scripts/ncu_summary.py gpurun_out/x.ncu-rep <srchash> profiles/r02_ncu_kernels.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
           "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
           "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]


def main(rep, srchash, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    launches = []
    for row in rows[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = f"{row[i]} {units[i]}".strip()
        launches.append(d)
    json.dump({"source_hash": srchash, "report": rep, "launches": launches}, open(out, "w"), indent=1)
    print(out, len(launches), "launches")


if __name__ == "__main__":
    main(*sys.argv[1:4])
