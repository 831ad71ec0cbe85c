#!/bin/bash
# A/B builds of the LU path (tools/build_variant.sh) on the lu_ab.py cases; usage:
# lu_var_run.sh outdir variant [variant ...]
out=$1; shift
mkdir -p $out
rm -f gpurun_out/lu_var_*.pt
for v in "$@"; do
  timeout 900 python tools/lu_var.py tools/variants/$v/librbf.so $v lat2 lat3 clu256k >> $out/var.txt 2>&1
done
echo done >> $out/var.txt
