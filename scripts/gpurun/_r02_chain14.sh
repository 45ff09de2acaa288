mkdir -p gpurun_out
O=gpurun_out/r02_chain14.txt
: > $O
timeout 300 python scripts/step_ab.py "DDL_LB_CHAIN=0" "" "DDL_CHAIN_TMA=1" "DDL_CHAIN_TMA=1" >> $O 2>&1
for v in c256s4 c768s2 c512s2 c384s3; do
  echo "== $v" >> $O
  DDL_LIB=$PWD/build_variants/libddl_$v.so timeout 300 python scripts/step_ab.py "DDL_CHAIN_TMA=1" "DDL_CHAIN_TMA=1" >> $O 2>&1
done
echo "== tests" >> $O
timeout 1200 python -m pytest tests/test_gpu_chain.py -q -x --timeout 1100 2>&1 | tail -5 >> $O
cat $O
