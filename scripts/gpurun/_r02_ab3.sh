mkdir -p gpurun_out
O=gpurun_out/r02_ab3.txt
: > $O
for lib in paper_1811_12174_b200/libddl.so build_variants/libddl_s2_k32_b3.so build_variants/libddl_s3_k32_b2.so build_variants/libddl_s4_k24_b2.so build_variants/libddl_s3_k24_b3.so build_variants/libddl_s2_k64_b1.so; do
  echo "== $lib" >> $O
  DDL_LIB=$PWD/$lib python scripts/step_ab.py "DDL_L2_HINTS=47" "DDL_L2_HINTS=47,DDL_GROUP_WAVE_MB=32" "DDL_L2_HINTS=47,DDL_CHANNELS=3,DDL_GROUP_WAVE_MB=32" "DDL_L2_HINTS=47,DDL_CHANNELS=3" >> $O 2>&1
done
cat $O
