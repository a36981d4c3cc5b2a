timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/s10_bench.json 2> gpurun_out/s10_bench.err; echo bench_rc=$?
python -c "
import json;d=json.load(open('gpurun_out/s10_bench.json'));n=d['kernels']['coarsest']['launches'];print(d['ms_per_step'], d['value']/1e9, d['roofline']['achieved'], d['roofline']['frac']); print({k:round(v['ms']/n,2) for k,v in d['kernels'].items()})"
timeout 900 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_bench_paths.py tests/test_gpu_distributed.py -q -x -p no:cacheprovider > gpurun_out/s10_t.log 2>&1; echo t_rc=$?
tail -3 gpurun_out/s10_t.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_st_bslab|k_st_coupling" -c 14 --csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E "k_st_" | head -14
