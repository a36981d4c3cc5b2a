timeout 300 python bench.py --no-cpu-baseline > gpurun_out/s8_bench.json 2> gpurun_out/s8_bench.err; echo bench_rc=$?
python -c "
import json;d=json.load(open('gpurun_out/s8_bench.json'));n=d['kernels']['coarsest']['launches'];print(d['ms_per_step'], d['value']/1e9, d['roofline']['achieved'], d['roofline']['frac']); print({k:round(v['ms']/n,2) for k,v in d['kernels'].items()}); print(d['e2e'])"
timeout 1500 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_bench_paths.py tests/test_gpu_parity.py tests/test_gpu_edgecases.py tests/test_gpu_distributed.py tests/test_gpu_inner_mg.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > gpurun_out/s8_t.log 2>&1; echo t_rc=$?
tail -5 gpurun_out/s8_t.log
