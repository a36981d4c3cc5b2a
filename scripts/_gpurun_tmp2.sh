mkdir -p gpurun_out
for i in 1 2; do
for l in paper_1911_09548_b200/libst.so variants_tmp/libst_m54.so variants_tmp/libst_m64.so; do
  timeout 300 python scripts/variant_check.py $l 5 2>&1 | tail -1
done; done | tee gpurun_out/v_mtiles.log
timeout 600 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_bench_paths.py -x -q -p no:cacheprovider 2>&1 | tail -3
