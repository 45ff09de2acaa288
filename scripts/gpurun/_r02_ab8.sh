mkdir -p gpurun_out
O=gpurun_out/r02_ab8.txt
: > $O
for i in 1 2; do
timeout 300 python scripts/step_ab.py "" "DDL_MULTI_GENERIC=1" >> $O 2>&1
(cd build_variants/r1tree && timeout 300 python scripts/step_ab.py "") >> $O 2>&1
done
cat $O
