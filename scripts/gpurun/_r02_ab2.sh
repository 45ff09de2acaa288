mkdir -p gpurun_out
O=gpurun_out/r02_ab2.txt
python scripts/step_ab.py "" "DDL_L2_HINTS=47" "DDL_L2_HINTS=111" "DDL_L2_HINTS=43" "DDL_L2_HINTS=47,DDL_CHANNELS=3" "DDL_L2_HINTS=47,DDL_CHANNELS=3,DDL_GROUP_WAVE_MB=32" "DDL_CHANNELS=3,DDL_GROUP_WAVE_MB=48" "DDL_CHANNELS=3,DDL_GROUP_WAVE_MB=64" "DDL_CHANNELS=4,DDL_GROUP_WAVE_MB=32" "DDL_CHANNELS=4" "DDL_L2_HINTS=47,DDL_GROUP_WAVE_MB=64" > $O 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
for cfg in "DDL_L2_HINTS=47" "DDL_L2_HINTS=111"; do
  echo "== $cfg" >> $O
  ncu --metrics $M --clock-control none -k regex:ddl_multi -s 3 -c 1 python scripts/step_ab.py --ncu "$cfg" 2>&1 | grep -E "dram__|gpu__time|lts__" >> $O
done
cat $O
