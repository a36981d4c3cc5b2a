for v in lib_cpl lib_zero lib_cpl lib_zero; do timeout 300 python scripts/variant_check.py variants_tmp/$v.so 5 >> gpurun_out/s14_var.log 2>&1; done
cat gpurun_out/s14_var.log
timeout 1500 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_bench_paths.py tests/test_gpu_distributed.py -q -x -p no:cacheprovider > gpurun_out/s14_t.log 2>&1; echo t_rc=$?
tail -3 gpurun_out/s14_t.log
