mkdir -p gpurun_out
for k in k_st_residual_s k_st_residual; do
  v=7; [ $k = k_st_residual ] && v=0
  ST_SPLIT=$v timeout 600 ncu --set full --clock-control none -k regex:"^$k\$" -c 1 -f -o /tmp/p_$k \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/p_$k.log 2>&1; echo "ncu $k=$?"
  ncu -i /tmp/p_$k.ncu-rep --page raw --csv > gpurun_out/p_raw_$k.csv 2>/dev/null
  ncu -i /tmp/p_$k.ncu-rep --page details > gpurun_out/p_det_$k.txt 2>/dev/null
done
python scripts/ncu_csv_summary.py gpurun_out/p_raw_*.csv
