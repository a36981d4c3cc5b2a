for k in k_sn_scan k_prolong k_restrict k_g_update k_gt k_st_residual; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o /tmp/n_$k python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  ncu -i /tmp/n_$k.ncu-rep --page raw --csv > gpurun_out/s6_raw_$k.csv 2>&1
  ncu -i /tmp/n_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/s6_src_$k.csv 2>&1
done
ls -la gpurun_out/ | tail -14
