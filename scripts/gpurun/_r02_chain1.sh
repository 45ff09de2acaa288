mkdir -p gpurun_out
O=gpurun_out/r02_chain1.txt
: > $O
timeout 600 python scripts/step_ab.py "DDL_LB_CHAIN=0" "" "DDL_CHAIN_HINTS=1" "DDL_CHAIN_HINTS=2" "DDL_CHAIN_HINTS=4" "DDL_CHAIN_HINTS=3" "DDL_CHAIN_HINTS=5" "DDL_CHAIN_HINTS=7" "DDL_LB_CHAIN=0" "" >> $O 2>&1
echo "== minb2" >> $O
DDL_LIB=$PWD/build_variants/libddl_chain_b2.so timeout 300 python scripts/step_ab.py "DDL_LB_CHAIN=0" "" "DDL_CHAIN_HINTS=2" "DDL_CHAIN_HINTS=5" >> $O 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum,l1tex__t_bytes.sum
for cfg in "" "DDL_CHAIN_HINTS=2" "DDL_CHAIN_HINTS=5"; do
  echo "== ncu $cfg" >> $O
  timeout 300 ncu --metrics $M --clock-control none -k regex:ddl_chain -s 3 -c 1 python scripts/step_ab.py --ncu "$cfg" 2>&1 | grep -E "dram__|gpu__time|lts__|l1tex" >> $O
done
echo "== tests" >> $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_grouped.py -q -x -k "allreduce_parity or loopback_grouped_matches or randomized or config" --timeout 800 2>&1 | tail -5 >> $O
cat $O
