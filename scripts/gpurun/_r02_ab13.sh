mkdir -p gpurun_out
O=gpurun_out/r02_ab13.txt
timeout 600 python scripts/step_ab.py "" "DDL_RS_WS=1" "" "DDL_RS_WS=1" > $O 2>&1
DDL_RS_WS=1 timeout 900 python -m pytest tests/test_gpu_grouped.py tests/test_gpu_parity.py tests/test_gpu_inprocess.py -q -x --timeout 800 2>&1 | tail -2 >> $O
cat $O
