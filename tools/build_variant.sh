#!/bin/bash
# Build an A/B variant of librbf.so with extra -D flags into tools/variants/<name>/ (debug
# and measurement only; the product library is paper_0909_5413_b200/librbf.so).
# Usage: build_variant.sh name -DFOO=1 ...
set -e
name=$1; shift
ND=$(python -c "import paper_0909_5413_b200.build as b; print(b.nccl_dir())")
out=/root/repo/tools/variants/$name
mkdir -p /tmp/variant_$name $out
objs=""
for src in /root/repo/paper_0909_5413_b200/csrc/*.cu; do
  o=/tmp/variant_$name/$(basename $src).o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC "$@" -I$ND/include -I/root/repo/include -c $src -o $o &
  objs="$objs $o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/librbf.so $objs -L$ND/lib -l:libnccl.so.2 -Xlinker -rpath=$ND/lib
echo $out/librbf.so
