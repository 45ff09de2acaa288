mkdir -p gpurun_out
O=gpurun_out/r02_chain8.txt
: > $O
timeout 300 python scripts/step_ab.py "DDL_LB_CHAIN=0" "" "" >> $O 2>&1
for v in b3 b5 b6 b4r2 b5r2 noasync; do
  echo "== $v" >> $O
  DDL_LIB=$PWD/build_variants/libddl_$v.so timeout 300 python scripts/step_ab.py "" "" >> $O 2>&1
done
echo "== tests" >> $O
timeout 1200 python -m pytest tests/test_gpu_chain.py -q -x --timeout 1100 2>&1 | tail -5 >> $O
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed
echo "== ncu default" >> $O
timeout 300 ncu --metrics $M --clock-control none -k regex:ddl_chain -s 3 -c 1 python scripts/step_ab.py --ncu "" 2>&1 | grep -E "dram__|gpu__time|lts__|sm__" >> $O
cat $O
