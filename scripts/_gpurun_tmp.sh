ST_STENCIL=1 python scripts/diag_precision.py > gpurun_out/r2_f_diag.log 2>&1
echo "--- ELL" >> gpurun_out/r2_f_diag.log
ST_STENCIL=0 python scripts/diag_precision.py >> gpurun_out/r2_f_diag.log 2>&1
cat gpurun_out/r2_f_diag.log
