#!/bin/bash
# libddl variants into build_variants/: each argument is NAME=FLAG[,FLAG...], e.g.
#   pf0b3=DDL_CHAIN_PREFETCH=0,DDL_CHAIN_CT_MINB=3   ->  build_variants/libddl_pf0b3.so
set -e
cd "$(dirname "$0")/.."
mkdir -p build_variants
for cfg in "$@"; do
  name=${cfg%%=*}
  flags=""
  IFS=, read -ra defs <<< "${cfg#*=}"
  for d in "${defs[@]}"; do flags="$flags -D$d"; done
  nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -fmad=false -Xcompiler -fPIC -shared \
    -cudart static -Iinclude -Ipaper_1811_12174_b200/csrc $flags \
    paper_1811_12174_b200/csrc/ddl_host.cu -o build_variants/libddl_$name.so &
done
wait
ls build_variants
