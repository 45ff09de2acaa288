#!/bin/bash
# Build libddl.so for sm_100a (cross-compiles without a GPU).
set -euo pipefail
cd "$(dirname "$0")"
OUT=paper_1811_12174_b200/libddl.so
# DDL_EXPERIMENTAL=1: also compile the PATH 3 / PATH 4 experiment kernels
nvcc -std=c++17 -DDDL_EXPERIMENTAL=${DDL_EXPERIMENTAL:-0} -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a \
  -fmad=false -Xptxas -v -Xcompiler -fPIC,-Wall -shared -cudart static \
  -Iinclude -Ipaper_1811_12174_b200/csrc \
  paper_1811_12174_b200/csrc/ddl_host.cu -o "$OUT" "$@"
# the kernels' identity (SASS hash) for bench.py's roofline.traffic check; best effort
python -c "import bench; bench.source_hash()" > /dev/null 2>&1 || true
echo "built $OUT"
