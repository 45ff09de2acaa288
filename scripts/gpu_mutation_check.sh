#!/bin/bash
# GPU mutation check: build libddl with a deliberate kernel mistake (DDL_MUTATE=1 descending
# fold order, 2 dropped 1/P scale, 3 copy phases drop their last chunk) and confirm the GPU
# parity tests FAIL on each, then that the unmutated build passes the same selection.
#   bash scripts/gpu_mutation_check.sh > gpurun_out/gpu_mutations.txt
cd "$(dirname "$0")/.."
mkdir -p build_variants
SEL='tests/test_gpu_parity.py::test_allreduce_parity tests/test_gpu_grouped.py::test_loopback_grouped_matches_oracle'
for m in 1 2 3; do
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -Xcompiler -fPIC -shared -cudart static \
    -Iinclude -Ipaper_1811_12174_b200/csrc -DDDL_MUTATE=$m paper_1811_12174_b200/csrc/ddl_host.cu \
    -o build_variants/libddl_mutate$m.so &
done
wait
for m in 1 2 3; do
  DDL_LIB=$PWD/build_variants/libddl_mutate$m.so timeout 900 python -m pytest $SEL -q -x -m gpu 2>&1 | tail -1 > /tmp/mut$m.txt
  if grep -q failed /tmp/mut$m.txt; then echo "mutation $m: CAUGHT ($(cat /tmp/mut$m.txt))"; else echo "mutation $m: NOT CAUGHT ($(cat /tmp/mut$m.txt))"; fi
done
timeout 900 python -m pytest $SEL -q -m gpu 2>&1 | tail -1 | sed 's/^/unmutated build: /'
