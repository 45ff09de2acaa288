#!/bin/bash
# Build libddl variants with different TMA pipeline parameters into build_variants/.
set -e
cd "$(dirname "$0")/.."
mkdir -p build_variants
for cfg in "$@"; do   # cfg = STAGES:STAGE_KB:MINBLOCKS
  IFS=: read S K B <<< "$cfg"
  nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -fmad=false -Xcompiler -fPIC -shared \
    -cudart static -Iinclude -Ipaper_1811_12174_b200/csrc -DDDL_TMA_STAGES=$S -DDDL_TMA_STAGE_KB=$K \
    -DDDL_TMA_MINBLOCKS=$B paper_1811_12174_b200/csrc/ddl_host.cu -o build_variants/libddl_s${S}_k${K}_b${B}.so &
done
wait
ls build_variants
