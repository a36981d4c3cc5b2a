timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r2_k_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2_k_pytest.log
tail -15 gpurun_out/r2_k_pytest.log
