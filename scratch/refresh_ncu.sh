#!/bin/bash
# ncu evidence for profiles/: launch lists of the bench command, full captures of the working kernels
O=gpurun_out/refresh; mkdir -p $O
for c in cfg4 cfg1 cfg2 cfg3 cfg5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_$c.csv \
    python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > $O/launch_$c.out 2>&1
  echo "launch $c exit $?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_cfg4_int32.csv \
  python bench.py --config cfg4 --dtype int32 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > $O/launch_cfg4_int32.out 2>&1
echo "launch cfg4_int32 exit $?"
# full captures: the 3rd sort's pipeline kernels (skip the first two sorts' launches)
K='regex:estimate_kernel|tiny_count_kernel|hash_count|emit_kernel|compact_kernel|dense_pairs|small_sort'
for c in cfg4 cfg2 cfg3 cfg1; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -s 14 -c 7 -o $O/full_$c -f \
    python scratch/one_cfg.py $c 3 > $O/full_$c.log 2>&1
  echo "full $c exit $?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -s 14 -c 7 -o $O/full_cfg4_int32 -f \
  python scratch/one_cfg.py cfg4 3 int32 > $O/full_cfg4_int32.log 2>&1
echo "full cfg4_int32 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:msd_|bucket_' -s 10 -c 6 -o $O/full_cfg5 -f \
  python scratch/one_cfg.py cfg5 3 > $O/full_cfg5.log 2>&1
echo "full cfg5 exit $?"
ls -la $O
# summaries here (the reports are too big to bring back): profiles/ layout
S=gpurun_out/refresh_sum; mkdir -p $S
for c in cfg4 cfg1 cfg2 cfg3 cfg5 cfg4_int32; do
  python profiles/summarize_ncu.py full $O/full_$c.ncu-rep $c $S/r01_ncu_${c}_full.json > $S/full_$c.txt 2>&1
  cp $O/launch_$c.csv $S/r01_ncu_${c}_launches.csv
  python profiles/summarize_ncu.py launches $O/launch_$c.csv $S/r01_ncu_${c}_launches.txt > /dev/null 2>&1
done
cp profiles/ncu_traffic.json $S/
python profiles/hotspots.py $O/full_cfg4.ncu-rep hash_count 25 > $S/hotspots_cfg4_count.txt 2>&1
python profiles/hotspots.py $O/full_cfg3.ncu-rep hash_count_big 25 > $S/hotspots_cfg3_count.txt 2>&1
mkdir -p gpurun_out/keep; mv $O/full_cfg4.ncu-rep $O/full_cfg3.ncu-rep gpurun_out/keep/
rm -rf $O
du -sh gpurun_out
