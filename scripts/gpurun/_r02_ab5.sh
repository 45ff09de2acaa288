mkdir -p gpurun_out
O=gpurun_out/r02_ab5.txt
: > $O
for i in 1 2; do
echo "== current" >> $O
timeout 300 python scripts/step_ab.py "" "DDL_L2_HINTS=47" >> $O 2>&1
echo "== round-1 build" >> $O
(cd build_variants/r1tree && timeout 300 python scripts/step_ab.py "" "DDL_L2_HINTS=47") >> $O 2>&1
done
cat $O
