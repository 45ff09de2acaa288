mkdir -p gpurun_out
O=gpurun_out/r02_chain4.txt
: > $O
timeout 300 python scripts/step_ab.py "DDL_LB_CHAIN=0" "" "" >> $O 2>&1
for v in pf0b3h2 pf1b2 pf1b2h2 pf0b2 lds; do
  echo "== $v" >> $O
  DDL_LIB=$PWD/build_variants/libddl_$v.so timeout 300 python scripts/step_ab.py "" "" >> $O 2>&1
done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed
echo "== ncu default" >> $O
timeout 300 ncu --metrics $M --clock-control none -k regex:ddl_chain -s 3 -c 1 python scripts/step_ab.py --ncu "" 2>&1 | grep -E "dram__|gpu__time|lts__|l1tex|sm__|smsp" >> $O
echo "== tests" >> $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_grouped.py -q -x -k "allreduce_parity or loopback_grouped_matches or randomized or config" --timeout 800 2>&1 | tail -5 >> $O
cat $O
