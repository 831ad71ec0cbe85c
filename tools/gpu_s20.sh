for cfg in 2 4; do
  timeout 300 python tools/trim_ab.py $cfg tools/ab/librbf_prev.so prev 2>&1 | tail -1
  timeout 300 python tools/trim_ab.py $cfg paper_0909_5413_b200/librbf.so new 2>&1 | tail -2
done
