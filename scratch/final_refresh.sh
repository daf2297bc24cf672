#!/bin/bash
# final round-1 evidence: full GPU tests, smoke, bench lines for every config, reference arm,
# launch lists of the bench command, full captures of the working kernels (summarised here)
S=gpurun_out/final; mkdir -p $S
timeout 1200 python -m pytest tests -m gpu -q > $S/gpu_tests.log 2>&1; echo "tests $?"; tail -2 $S/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $S/smoke.txt 2>&1; echo "smoke $?"
O=gpurun_out/final_reps; mkdir -p $O
K='regex:estimate_kernel|tiny_count_kernel|hash_count|emit_kernel|compact_kernel|dense_pairs|small_sort'
for c in cfg4 cfg2 cfg1; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -s 14 -c 7 -o $O/full_$c -f \
    python scratch/one_cfg.py $c 3 > $O/full_$c.log 2>&1
  python profiles/summarize_ncu.py full $O/full_$c.ncu-rep $c $S/r01_ncu_${c}_full.json > $S/full_$c.txt 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -s 14 -c 7 -o $O/full_cfg4_int32 -f \
  python scratch/one_cfg.py cfg4 3 int32 > $O/full_cfg4_int32.log 2>&1
python profiles/summarize_ncu.py full $O/full_cfg4_int32.ncu-rep cfg4_int32 $S/r01_ncu_cfg4_int32_full.json > $S/full_cfg4_int32.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:hash_count_big|emit_kernel' -s 6 -c 3 \
  -o $O/full_cfg3 -f python scratch/one_cfg.py cfg3 3 > $O/full_cfg3.log 2>&1
python profiles/summarize_ncu.py full $O/full_cfg3.ncu-rep cfg3 $S/r01_ncu_cfg3_full.json > $S/full_cfg3.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:msd_|bucket_' -s 10 -c 6 -o $O/full_cfg5 -f \
  python scratch/one_cfg.py cfg5 3 > $O/full_cfg5.log 2>&1
python profiles/summarize_ncu.py full $O/full_cfg5.ncu-rep cfg5 $S/r01_ncu_cfg5_full.json > $S/full_cfg5.txt 2>&1
python profiles/hotspots.py $O/full_cfg4.ncu-rep hash_count 25 > $S/r01_hotspots_cfg4_count.txt 2>&1
python profiles/hotspots.py $O/full_cfg3.ncu-rep hash_count_big 25 > $S/r01_hotspots_cfg3_count.txt 2>&1
cp profiles/ncu_traffic.json $S/
for c in cfg4 cfg1 cfg2 cfg3 cfg5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $S/r01_ncu_${c}_launches.csv \
    python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > /dev/null 2>&1
  python profiles/summarize_ncu.py launches $S/r01_ncu_${c}_launches.csv $S/r01_ncu_${c}_launches.txt > /dev/null 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $S/r01_ncu_cfg4_int32_launches.csv \
  python bench.py --config cfg4 --dtype int32 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > /dev/null 2>&1
python profiles/summarize_ncu.py launches $S/r01_ncu_cfg4_int32_launches.csv $S/r01_ncu_cfg4_int32_launches.txt > /dev/null 2>&1
rm -rf $O
for c in cfg4 cfg1 cfg2 cfg3 cfg5; do
  timeout 400 python bench.py --config $c > $S/r01_bench_$c.json 2> $S/r01_bench_$c.err; echo "bench $c $?"
done
timeout 400 python bench.py --config cfg4 --dtype int32 > $S/r01_bench_cfg4_int32.json 2> $S/r01_bench_cfg4_int32.err; echo "int32 $?"
timeout 400 python bench.py --impl reference > $S/r01_bench_reference_cfg4.json 2> $S/r01_bench_reference_cfg4.err; echo "ref $?"
timeout 400 python bench.py --sharded > $S/r01_bench_cfg4_sharded.json 2> $S/r01_bench_cfg4_sharded.err; echo "sharded $?"
du -sh gpurun_out
