mkdir -p gpurun_out
O=gpurun_out/r02_trace.txt
echo "== default" > $O; python scripts/trace_step.py >> $O 2>&1
echo "== hints47" >> $O; DDL_L2_HINTS=47 python scripts/trace_step.py >> $O 2>&1
echo "== hints47 waves32 ch3" >> $O; DDL_L2_HINTS=47 DDL_GROUP_WAVE_MB=32 DDL_CHANNELS=3 python scripts/trace_step.py >> $O 2>&1
cat $O
