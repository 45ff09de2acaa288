#!/bin/bash
# libddl variants of the deep copy pipeline geometry (sub-stages : lag) into build_variants/.
set -e
cd "$(dirname "$0")/.."
mkdir -p build_variants
for cfg in "$@"; do
  IFS=: read S G <<< "$cfg"
  nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -fmad=false -Xcompiler -fPIC -shared \
    -cudart static -Iinclude -Ipaper_1811_12174_b200/csrc -DDDL_COPY_SUB=$S -DDDL_COPY_LAG=$G \
    paper_1811_12174_b200/csrc/ddl_host.cu -o build_variants/libddl_cs${S}_lag${G}.so &
done
wait
ls build_variants
