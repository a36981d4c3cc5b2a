# One gpurun call that produces the round evidence under gpurun_out/ (copied to profiles/ afterwards):
# GPU tests, ncu --set full per kernel (reports stay in /tmp on the box: gpurun_out/ is capped at 64 MiB),
# plain bench + ncu launch list of the same command, final bench lines, smoke.
mkdir -p gpurun_out
H=$(python scripts/srchash.py)
echo "srchash $H"
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/f_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/f_pytest.log
# ncu --set full, one capture per kernel, first (finest-level) launch
for k in k_st_residual k_st_res_mass k_st_sweep k_sn_scan; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$k" -c 1 -f -o /tmp/f_full_$k \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/f_full_$k.log 2>&1; echo "ncu $k=$?"
  ncu -i /tmp/f_full_$k.ncu-rep --page raw --csv > gpurun_out/f_raw_$k.csv 2>/dev/null
done
python - <<EOF
import json, subprocess, sys
sys.path.insert(0, "scripts")
import ncu_summary as s
L = []
for k in "k_st_residual k_st_res_mass k_st_sweep k_sn_scan".split():
    try:
        s.main(f"/tmp/f_full_{k}.ncu-rep", "$H", f"gpurun_out/f_k_{k}.json")
        L += json.load(open(f"gpurun_out/f_k_{k}.json"))["launches"]
    except Exception as e:
        print("summary failed", k, e)
json.dump({"source_hash": "$H", "report": "f_full_<kernel>.ncu-rep (one capture per kernel, bench.py --steps 1 --warmup 0)", "launches": L}, open("gpurun_out/f_ncu_kernels.json", "w"), indent=1)
EOF
cp gpurun_out/f_ncu_kernels.json profiles/r02_ncu_kernels.json
python scripts/ncu_csv_summary.py gpurun_out/f_raw_*.csv > gpurun_out/f_ncu_summary.txt 2>&1
cat gpurun_out/f_ncu_summary.txt
# plain bench of the launch-list command, then the launch list
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_b2.json 2>gpurun_out/f_b2.err; echo b2=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/f_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_ncu_l.log 2>&1; echo launches=$?
python scripts/launch_summary.py gpurun_out/f_launches.csv gpurun_out/f_b2.json 2 > gpurun_out/f_launches.txt; tail -4 gpurun_out/f_launches.txt
# final bench lines
timeout 900 python bench.py > gpurun_out/f_bench.json 2>gpurun_out/f_bench.err; echo bench=$?
cat gpurun_out/f_bench.json | cut -c1-1800
timeout 600 python bench.py --impl reference > gpurun_out/f_bench_ref.json 2>gpurun_out/f_bench_ref.err; echo ref=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/f_smoke.log
cuobjdump -sass paper_1911_09548_b200/libst.so | grep -c UTMALDG > gpurun_out/f_utmaldg_count.txt
rm -f gpurun_out/q_src_* ; du -sh gpurun_out
