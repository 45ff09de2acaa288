mkdir -p gpurun_out
O=gpurun_out/r02_ab16.txt
timeout 600 python scripts/step_ab.py "" "DDL_AG_EAGER=1" "" "DDL_AG_EAGER=1" > $O 2>&1
DDL_AG_EAGER=1 timeout 1200 python -m pytest tests/test_gpu_grouped.py tests/test_gpu_parity.py tests/test_gpu_inprocess.py tests/test_gpu_multiproc.py tests/test_gpu_edge.py -q -x --timeout 900 2>&1 | tail -2 >> $O
cat $O
