mkdir -p gpurun_out
ST_NODAL_RES=3 timeout 900 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_bench_paths.py -x -q -p no:cacheprovider > gpurun_out/m_t.log 2>&1; echo t=$?
tail -5 gpurun_out/m_t.log
for v in 3 0 3 0; do ST_NODAL_RES=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/m_b$v.json 2>>gpurun_out/m_b.err; python -c "
import json;d=json.load(open('gpurun_out/m_b$v.json'));print('nodal_res=$v', round(d['ms_per_step'],2), {k:round(v['ms'],1) for k,v in d['kernels'].items()}, {k:round(v['GBps']) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"; done
