mkdir -p gpurun_out
O=gpurun_out/r02_chain6.txt
: > $O
timeout 300 python scripts/step_ab.py "DDL_LB_CHAIN=0" "" "DDL_CHAIN_GENERIC=1" >> $O 2>&1
for v in n1f2r2 n1f0r2 n1f1r2 n2f0r0 n2f2r2 n2f0r2 n4f0r2; do
  echo "== $v" >> $O
  DDL_LIB=$PWD/build_variants/libddl_$v.so timeout 300 python scripts/step_ab.py "" "" >> $O 2>&1
done
echo "== tests" >> $O
timeout 1200 python -m pytest tests/test_gpu_chain.py -q -x --timeout 1100 2>&1 | tail -5 >> $O
cat $O
