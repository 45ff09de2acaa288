mkdir -p gpurun_out
O=gpurun_out/r02_ab11.txt
timeout 600 python scripts/step_ab.py "" "DDL_L2_HINTS=559" "" "DDL_L2_HINTS=559" "" "DDL_L2_HINTS=559" > $O 2>&1
cat $O
