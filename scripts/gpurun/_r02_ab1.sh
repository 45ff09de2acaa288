mkdir -p gpurun_out
O=gpurun_out/r02_ab1.txt
python scripts/step_ab.py "" "DDL_GROUP_ORDER=1" "DDL_GROUP_WAVE_MB=64" "DDL_GROUP_WAVE_MB=48" "DDL_GROUP_WAVE_MB=32" "DDL_GROUP_WAVE_MB=24" "DDL_GROUP_WAVE_MB=16" "DDL_GROUP_WAVE_MB=32,DDL_GROUP_ORDER=1" "DDL_CHANNELS=3" "DDL_CHANNELS=3,DDL_GROUP_WAVE_MB=32" "DDL_CHANNELS=1" "DDL_CHANNELS=1,DDL_GROUP_WAVE_MB=32" "DDL_L2_HINTS=7" "DDL_L2_HINTS=31" "DDL_L2_HINTS=11" "DDL_L2_HINTS=13" > $O 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
for cfg in "" "DDL_GROUP_WAVE_MB=32" "DDL_GROUP_WAVE_MB=16" "DDL_CHANNELS=1"; do
  echo "== $cfg" >> $O
  ncu --metrics $M --clock-control none -k regex:ddl_multi -s 3 -c 1 python scripts/step_ab.py --ncu "$cfg" 2>&1 | grep -E "dram__|gpu__time|lts__" >> $O
done
cat $O
