timeout 300 python scripts/variant_check.py paper_1911_09548_b200/libst.so 3 > gpurun_out/r2_n_variant.log 2>&1
timeout 900 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_bench_paths.py tests/test_gpu_distributed.py -q -x -p no:cacheprovider > gpurun_out/r2_n_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_n_tests.log
cat gpurun_out/r2_n_variant.log; tail -3 gpurun_out/r2_n_tests.log
