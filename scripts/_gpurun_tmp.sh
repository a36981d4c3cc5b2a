python scripts/srchash.py > gpurun_out/r2_l_srchash.txt
python bench.py > gpurun_out/r2_l_bench.json 2> gpurun_out/r2_l_bench.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_l_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_l_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_l_ncu1.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"k_st_" -c 2 -o gpurun_out/r2_l_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_l_ncu2.log 2>&1
du -sh gpurun_out
