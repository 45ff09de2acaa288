mkdir -p gpurun_out
O=gpurun_out/r02_chain15.txt
: > $O
timeout 300 python scripts/step_ab.py "DDL_LB_CHAIN=0" "DDL_CHAIN_TMA=0" "" "" >> $O 2>&1
for v in c256s2 c384s2 c640s2 c512s2r0 c256s3 c512s1; do
  echo "== $v" >> $O
  DDL_LIB=$PWD/build_variants/libddl_$v.so timeout 300 python scripts/step_ab.py "" "" >> $O 2>&1
done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_sector_hit_rate.pct
echo "== ncu default" >> $O
timeout 300 ncu --metrics $M --clock-control none -k regex:ddl_chain -s 3 -c 1 python scripts/step_ab.py --ncu "" 2>&1 | grep -E "dram__|gpu__time|lts__|sm__|l1tex" >> $O
cat $O
