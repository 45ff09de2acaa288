mkdir -p gpurun_out
O=gpurun_out/r02_ab14.txt
: > $O
timeout 300 python scripts/step_ab.py "" >> $O 2>&1
for S in 2 3 6; do echo "== rs stages $S" >> $O; DDL_LIB=$PWD/build_variants/libddl_rs$S.so timeout 300 python scripts/step_ab.py "DDL_RS_WS=1" >> $O 2>&1; done
cat $O
