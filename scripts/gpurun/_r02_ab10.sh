mkdir -p gpurun_out
O=gpurun_out/r02_ab10.txt
echo "== ag default" > $O; timeout 300 python scripts/ag_bench.py >> $O 2>&1
echo "== ag deep copy (559)" >> $O; DDL_L2_HINTS=559 timeout 300 python scripts/ag_bench.py >> $O 2>&1
timeout 600 python scripts/step_ab.py "" "DDL_L2_HINTS=559" "DDL_L2_HINTS=559,DDL_GROUP_WAVE_MB=32" "DDL_L2_HINTS=559,DDL_CHANNELS=3" >> $O 2>&1
DDL_L2_HINTS=559 timeout 600 python -m pytest tests/test_gpu_grouped.py tests/test_gpu_parity.py -q -x -k "grouped or kernel_paths or reduce_scatter or config2" --timeout 500 2>&1 | tail -2 >> $O
cat $O
