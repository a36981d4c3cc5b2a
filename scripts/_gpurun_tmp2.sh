mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stencil.py -x -q -p no:cacheprovider > gpurun_out/s_t.log 2>&1; echo t=$?
tail -15 gpurun_out/s_t.log
for v in 7 0 3 7 0; do ST_SPLIT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s_b$v.json 2>>gpurun_out/s_b.err; python -c "
import json;d=json.load(open('gpurun_out/s_b$v.json'));print('split=$v', round(d['ms_per_step'],2), {k:round(v['ms'],1) for k,v in d['kernels'].items()}, {k:round(v['GBps']) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"; done
tail -5 gpurun_out/s_b.err
