mkdir -p gpurun_out
O=gpurun_out/r02_ab17.txt
: > $O
for i in 1 2; do
echo "== current (eager code, off)" >> $O; timeout 300 python scripts/step_ab.py "" >> $O 2>&1
echo "== previous commit" >> $O; DDL_LIB=$PWD/build_variants/libddl_prev.so timeout 300 python scripts/step_ab.py "" >> $O 2>&1
echo "== round 1" >> $O; (cd build_variants/r1tree && timeout 300 python scripts/step_ab.py "") >> $O 2>&1
done
cat $O
