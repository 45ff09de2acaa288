mkdir -p gpurun_out
O=gpurun_out/r02_chain9.txt
: > $O
timeout 300 python scripts/step_ab.py "DDL_LB_CHAIN=0" "" >> $O 2>&1
for v in bmr2b3 bmr0b3 bmr2b4 rowr2b3; do
  echo "== $v" >> $O
  DDL_LIB=$PWD/build_variants/libddl_$v.so timeout 300 python scripts/step_ab.py "" "" >> $O 2>&1
done
DDL_LIB=$PWD/build_variants/libddl_bmr2b3.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:ddl_chain -s 3 -c 1 -o gpurun_out/r02_chain_bmr2b3 -f python scripts/step_ab.py --ncu "" > /dev/null 2>&1
DDL_LIB=$PWD/build_variants/libddl_rowr2b3.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:ddl_chain -s 3 -c 1 -o gpurun_out/r02_chain_rowr2b3 -f python scripts/step_ab.py --ncu "" > /dev/null 2>&1
cat $O
