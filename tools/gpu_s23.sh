O=gpurun_out/f5; mkdir -p $O
for cfg in 1 2 3 5; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg$cfg.log 2>&1; echo "rc=$?" >> $O/bench_cfg$cfg.log
done
