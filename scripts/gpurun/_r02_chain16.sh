mkdir -p gpurun_out
O=gpurun_out/r02_chain16.txt
: > $O
timeout 300 python scripts/step_ab.py "DDL_LB_CHAIN=0" "" >> $O 2>&1
for v in c384s2b c192s2 c320s2 c448s2 c128s2 c128s3; do
  echo "== $v" >> $O
  DDL_LIB=$PWD/build_variants/libddl_$v.so timeout 300 python scripts/step_ab.py "" "" >> $O 2>&1
done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_sector_hit_rate.pct
cat $O
cat $O
