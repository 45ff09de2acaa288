mkdir -p gpurun_out
O=gpurun_out/r02_san.txt
: > $O
timeout 300 python scripts/sanitize_check.py >> $O 2>&1; echo "plain rc=$?" >> $O
timeout 500 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_check.py > gpurun_out/r02_san_memcheck.txt 2>&1; echo "memcheck rc=$?" >> $O
tail -40 gpurun_out/r02_san_memcheck.txt >> $O
cat $O
