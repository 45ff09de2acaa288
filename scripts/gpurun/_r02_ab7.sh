mkdir -p gpurun_out
O=gpurun_out/r02_ab7.txt
timeout 600 python scripts/step_ab.py "" "DDL_L2_HINTS=175" "DDL_L2_HINTS=303" "DDL_L2_HINTS=191" "DDL_L2_HINTS=63" "DDL_L2_HINTS=111" "DDL_L2_HINTS=239" > $O 2>&1
cat $O
