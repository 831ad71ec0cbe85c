#!/bin/bash
# Build the phase-probe variant of librbf.so into tools/probe/ (debug only).
set -e
ND=/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl
mkdir -p /tmp/probe /root/repo/tools/probe
objs=""
for src in /root/repo/paper_0909_5413_b200/csrc/*.cu; do
  o=/tmp/probe/$(basename $src).o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -DRBF_PROBE -I$ND/include -I/root/repo/include -c $src -o $o &
  objs="$objs $o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /root/repo/tools/probe/librbf.so $objs -L$ND/lib -l:libnccl.so.2 -Xlinker -rpath=$ND/lib
echo ok
