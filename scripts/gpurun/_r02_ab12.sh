mkdir -p gpurun_out
O=gpurun_out/r02_ab12.txt
: > $O
for lib in paper_1811_12174_b200/libddl.so build_variants/libddl_cs8_lag1.so build_variants/libddl_cs8_lag4.so build_variants/libddl_cs16_lag4.so build_variants/libddl_cs4_lag1.so build_variants/libddl_cs16_lag8.so; do
  echo "== $lib" >> $O
  DDL_LIB=$PWD/$lib timeout 300 python scripts/step_ab.py "" >> $O 2>&1
done
echo "== again default" >> $O
timeout 300 python scripts/step_ab.py "" "DDL_DEEP_COPY=0" >> $O 2>&1
cat $O
