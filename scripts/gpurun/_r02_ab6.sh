mkdir -p gpurun_out
O=gpurun_out/r02_ab6.txt
H=DDL_L2_HINTS=47
timeout 900 python scripts/step_ab.py "$H" "$H,DDL_GROUP_LOOKAHEAD=1" "$H,DDL_GROUP_LOOKAHEAD=1,DDL_GROUP_WAVE_MB=32" "$H,DDL_GROUP_LOOKAHEAD=1,DDL_GROUP_WAVE_MB=48" "$H,DDL_GROUP_LOOKAHEAD=1,DDL_GROUP_WAVE_MB=16" "$H,DDL_GROUP_LOOKAHEAD=1,DDL_CHANNELS=1" "$H,DDL_GROUP_LOOKAHEAD=1,DDL_CHANNELS=1,DDL_GROUP_WAVE_MB=32" "$H,DDL_GROUP_LOOKAHEAD=1,DDL_CHANNELS=1,DDL_GROUP_WAVE_MB=16" "$H,DDL_GROUP_LOOKAHEAD=1,DDL_CHANNELS=3,DDL_GROUP_WAVE_MB=32" "$H,DDL_GROUP_LOOKAHEAD=1,DDL_CHANNELS=1,DDL_GROUP_WAVES=4" > $O 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for cfg in "$H,DDL_GROUP_LOOKAHEAD=1" "$H,DDL_GROUP_LOOKAHEAD=1,DDL_GROUP_WAVE_MB=32"; do
  echo "== $cfg" >> $O
  ncu --metrics $M --clock-control none -k regex:ddl_multi -s 3 -c 1 python scripts/step_ab.py --ncu "$cfg" 2>&1 | grep -E "dram__|gpu__time" >> $O
done
cat $O
