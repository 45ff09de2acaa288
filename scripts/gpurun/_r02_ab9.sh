mkdir -p gpurun_out
O=gpurun_out/r02_ab9.txt
P=DDL_GROUP_PIPE=1
timeout 900 python scripts/step_ab.py "" "$P" "$P,DDL_GROUP_WAVE_MB=32" "$P,DDL_GROUP_WAVE_MB=16" "$P,DDL_GROUP_WAVES=2" "$P,DDL_GROUP_WAVES=4" "$P,DDL_CHANNELS=1" "$P,DDL_CHANNELS=1,DDL_GROUP_WAVES=2" "$P,DDL_CHANNELS=1,DDL_GROUP_WAVES=4" "$P,DDL_CHANNELS=3" "$P,DDL_CHANNELS=1,DDL_GROUP_WAVE_MB=32" > $O 2>&1
(cd build_variants/r1tree && timeout 300 python scripts/step_ab.py "") >> $O 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for cfg in "$P" "$P,DDL_GROUP_WAVES=2"; do
  echo "== $cfg" >> $O
  ncu --metrics $M --clock-control none -k regex:ddl_multi -s 3 -c 1 python scripts/step_ab.py --ncu "$cfg" 2>&1 | grep -E "dram__|gpu__time" >> $O
done
cat $O
