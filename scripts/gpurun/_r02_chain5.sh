mkdir -p gpurun_out
O=gpurun_out/r02_chain5.txt
: > $O
timeout 300 python scripts/step_ab.py "DDL_LB_CHAIN=0" "" >> $O 2>&1
for v in v2 v2h2; do
  echo "== $v" >> $O
  DDL_LIB=$PWD/build_variants/libddl_$v.so timeout 300 python scripts/step_ab.py "" "" >> $O 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ddl_chain -s 3 -c 1 -o gpurun_out/r02_chain_default -f python scripts/step_ab.py --ncu "" > /dev/null 2>&1
DDL_LIB=$PWD/build_variants/libddl_v2.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:ddl_chain -s 3 -c 1 -o gpurun_out/r02_chain_v2 -f python scripts/step_ab.py --ncu "" > /dev/null 2>&1
ls -la gpurun_out >> $O
cat $O
