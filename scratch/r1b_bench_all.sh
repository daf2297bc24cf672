#!/bin/bash
# bench every config (fresh numbers) + ncu full capture of the estimate kernel on cfg2
mkdir -p gpurun_out
for c in cfg1 cfg2 cfg3 cfg5; do
  timeout 300 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c exit $?"; cut -c1-400 gpurun_out/bench_$c.json
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:estimate_kernel -s 3 -c 1 \
  -o gpurun_out/est_cfg2 -f python scratch/one_cfg.py cfg2 5 > gpurun_out/ncu_est.log 2>&1
echo "ncu exit $?"
