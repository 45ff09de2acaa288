mkdir -p gpurun_out
O=gpurun_out/r02_chain7.txt
: > $O
echo "== default (n1f0r0)" >> $O; timeout 300 python scripts/chain_placement.py >> $O 2>&1
echo "== slice" >> $O; DDL_LB_CHAIN=0 timeout 300 python scripts/chain_placement.py >> $O 2>&1
echo "== n2f0r2" >> $O; DDL_LIB=$PWD/build_variants/libddl_n2f0r2.so timeout 300 python scripts/chain_placement.py >> $O 2>&1
cat $O
