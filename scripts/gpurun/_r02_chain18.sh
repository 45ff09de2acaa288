mkdir -p gpurun_out
O=gpurun_out/r02_chain18.txt
: > $O
timeout 300 python scripts/step_ab.py "DDL_LB_CHAIN=0" "" "" "DDL_CHAIN_TMA=0" >> $O 2>&1
for v in tm2 tm2c384 tm2c256; do
  echo "== $v" >> $O
  DDL_LIB=$PWD/build_variants/libddl_$v.so timeout 300 python scripts/step_ab.py "" "" >> $O 2>&1
done
echo "== tests" >> $O
timeout 1200 python -m pytest tests/test_gpu_chain.py -q -x --timeout 1100 2>&1 | tail -3 >> $O
cat $O
