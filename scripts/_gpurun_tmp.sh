for v in lib_side lib_1a1d lib_side lib_1a1d lib_side lib_1a1d; do timeout 300 python scripts/variant_check.py variants_tmp/$v.so 5 >> gpurun_out/s12_var.log 2>&1; done
cat gpurun_out/s12_var.log
