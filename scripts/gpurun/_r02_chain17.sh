mkdir -p gpurun_out
O=gpurun_out/r02_chain17.txt
: > $O
timeout 300 python scripts/step_ab.py "DDL_LB_CHAIN=0" "" "" >> $O 2>&1
for v in c288s2 c352s2 c320s3 c160s2; do
  echo "== $v" >> $O
  DDL_LIB=$PWD/build_variants/libddl_$v.so timeout 300 python scripts/step_ab.py "" "" >> $O 2>&1
done
echo "== tests" >> $O
timeout 1500 python -m pytest tests/test_gpu_chain.py tests/test_gpu_parity.py tests/test_gpu_grouped.py tests/test_gpu_edge.py -q -x --timeout 1400 2>&1 | tail -5 >> $O
cat $O
