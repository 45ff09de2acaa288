mkdir -p gpurun_out
O=gpurun_out/r02_ab4.txt
timeout 600 python scripts/step_ab.py "DDL_L2_HINTS=47" "DDL_L2_HINTS=47,DDL_BALANCE=1" "DDL_L2_HINTS=47,DDL_BALANCE=2" "DDL_L2_HINTS=47,DDL_BALANCE=2,DDL_TRANSPOSE=0" "DDL_L2_HINTS=47,DDL_BALANCE=1,DDL_CHANNELS=3,DDL_GROUP_WAVE_MB=32" "DDL_L2_HINTS=47,DDL_BALANCE=2,DDL_GROUP_WAVE_MB=48" "DDL_BALANCE=2" > $O 2>&1
echo "== trace balance 2" >> $O
DDL_L2_HINTS=47 DDL_BALANCE=2 timeout 300 python scripts/trace_step.py --calls 2 >> $O 2>&1
cat $O
