#!/bin/bash
# cfg3 count capture (the big-table shape), then every bench line (reads profiles/ncu_traffic.json)
S=gpurun_out/refresh_sum; mkdir -p $S
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:hash_count_big|emit_kernel' -s 6 -c 3 \
  -o gpurun_out/full_cfg3b -f python scratch/one_cfg.py cfg3 3 > $S/full_cfg3b.log 2>&1
python profiles/summarize_ncu.py full gpurun_out/full_cfg3b.ncu-rep cfg3 $S/r01_ncu_cfg3_full.json > $S/full_cfg3.txt 2>&1
python profiles/hotspots.py gpurun_out/full_cfg3b.ncu-rep hash_count_big 25 > $S/hotspots_cfg3_count.txt 2>&1
cp profiles/ncu_traffic.json $S/
for c in cfg4 cfg1 cfg2 cfg3 cfg5; do
  timeout 400 python bench.py --config $c > $S/r01_bench_$c.json 2> $S/r01_bench_$c.err; echo "bench $c $?"
done
timeout 400 python bench.py --config cfg4 --dtype int32 > $S/r01_bench_cfg4_int32.json 2> $S/r01_bench_cfg4_int32.err; echo "int32 $?"
timeout 400 python bench.py --impl reference > $S/r01_bench_reference_cfg4.json 2> $S/r01_bench_reference_cfg4.err; echo "ref $?"
python -c "import __graft_entry__ as g; g.smoke()" > $S/smoke.txt 2>&1; echo "smoke $?"
du -sh gpurun_out
