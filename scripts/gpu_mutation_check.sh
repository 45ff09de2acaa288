#!/bin/bash
# GPU mutation check: build libddl with a deliberate kernel mistake and confirm the GPU parity
# tests FAIL on each, then that the unmutated build passes the same selection.
#   slice kernels (ddl_device.cuh): 1 descending fold order, 2 dropped 1/P scale, 3 copy phases
#     drop their last chunk
#   column-chain kernels (ddl_chain.cuh): 4 descending fold order (CT kernels), 5 dropped 1/P
#     scale (CT kernels), 6 an innermost-dim allgather receiver skipped (CT kernels), 7 ranks 1 and
#     2's TMA ring segments swapped (TMA-fed kernel; 0 <-> 1 would be a no-op: fp add commutes), 8 dropped 1/P scale (generic kernel)
#   bash scripts/gpu_mutation_check.sh > gpurun_out/gpu_mutations.txt
cd "$(dirname "$0")/.."
mkdir -p build_variants
SEL_SLICE='tests/test_gpu_parity.py::test_allreduce_parity tests/test_gpu_grouped.py::test_loopback_grouped_matches_oracle'
SEL_CHAIN='tests/test_gpu_chain.py::test_chain_matches_oracle_edge_sizes tests/test_gpu_chain.py::test_chain_grouped_many_buckets'
MUTS=${MUTS:-"1 2 3 4 5 6 7 8"}
for m in $MUTS; do
  [ -f build_variants/libddl_mutate$m.so ] && continue
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -Xcompiler -fPIC -shared -cudart static \
    -Iinclude -Ipaper_1811_12174_b200/csrc -DDDL_MUTATE=$m paper_1811_12174_b200/csrc/ddl_host.cu \
    -o build_variants/libddl_mutate$m.so &
done
wait
for m in $MUTS; do
  if [ "$m" -le 3 ]; then SEL=$SEL_SLICE; else SEL=$SEL_CHAIN; fi
  DDL_LIB=$PWD/build_variants/libddl_mutate$m.so timeout 900 python -m pytest $SEL -q -x -m gpu 2>&1 | tail -1 > /tmp/mut$m.txt
  if grep -q failed /tmp/mut$m.txt; then echo "mutation $m: CAUGHT ($(cat /tmp/mut$m.txt))"; else echo "mutation $m: NOT CAUGHT ($(cat /tmp/mut$m.txt))"; fi
done
timeout 900 python -m pytest $SEL_SLICE $SEL_CHAIN -q -m gpu 2>&1 | tail -1 | sed 's/^/unmutated build: /'
