#!/bin/bash
# Builds libmckg.so variants of detect.cu (kernel experiments) into
# build/variants/<name>/libmckg.so: each argument is "name:-DMACRO=V,-DMACRO=V".
set -e
cd "$(dirname "$0")/.."
NCCL=$(python -c "import __graft_entry__ as g; print(g._nccl_dir())")
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}; defs=${defs//,/ }
  out=build/variants/$name; mkdir -p $out
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -diag-suppress 20011 \
    -Iinclude -Ipaper_1211_6193_b200/host -Ipaper_1211_6193_b200/csrc -I$NCCL/include $defs \
    -c paper_1211_6193_b200/csrc/detect.cu -o $out/detect.cu.o -Xptxas -v 2>&1 | grep -A2 fast_kernel | grep -E "registers|spill" | sed "s/^/$name: /"
  objs=$(ls build/obj/*.o | grep -v detect.cu.o)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o $out/libmckg.so $out/detect.cu.o $objs \
    -L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL/lib
done
