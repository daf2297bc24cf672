# Regenerate the round-2 evidence under gpurun_out/ (one gpurun call, ~15 min):
#   bench lines of every config, launch lists (ncu gpu__time_duration), and one
#   `ncu --set full` capture of each config's pipeline kernels.
# Then, in the build container:  python profiles/summarize_ncu.py ...  (see README)
set -x
O=gpurun_out
for c in cfg4 cfg1 cfg2 cfg3 cfg5 cfg4r; do
  timeout 900 python bench.py --config $c > $O/r02_bench_$c.json 2> $O/r02_bench_$c.err
done
timeout 600 python bench.py --dtype int32 > $O/r02_bench_cfg4_int32.json 2> $O/r02_bench_cfg4_int32.err
timeout 600 python bench.py --sharded > $O/r02_bench_cfg4_sharded.json 2> $O/r02_bench_cfg4_sharded.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/r02_bench_reference_cfg4.json 2> $O/r02_bench_reference_cfg4.err
for c in cfg4 cfg1 cfg2 cfg3 cfg5 cfg4r; do
  args="--config $c --steps 1 --warmup 1 --no-cpu --e2e-steps 0"
  python bench.py $args > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/r02_ncu_${c}_launches.csv python bench.py $args > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on \
      -k regex:"estimate_kernel|tiny_count|hash_count|hp_|compact_kernel|dense_pairs|small_sort|emit_kernel|emit_map|msd_|bucket_|onesweep|radix_" \
      -c 40 -o $O/r02_ncu_${c}_full python bench.py $args \
      > $O/r02_ncu_${c}_full.log 2>&1
done
# per-call device time at the per-rank shard sizes of an 8-GPU split, single-GPU
# entry point and the native sharded one at one NCCL rank (profiles/percall.py)
: > $O/r02_percall.txt
for a in "cfg4 134217728" "cfg4 1073741824" "cfg2 3750000" "cfg3 3750000" "cfg4r 134217728"; do
  python profiles/percall.py $a 30 2>&1 | tail -1 >> $O/r02_percall.txt
  python profiles/percall.py $a 30 sharded 2>&1 | tail -1 >> $O/r02_percall.txt
done
echo done
# summaries (the .ncu-rep files are too large to bring back): written next to
# the launch lists, plus the DRAM-traffic table bench.py reads
cp profiles/ncu_traffic.json $O/ncu_traffic.json
for c in cfg4 cfg1 cfg2 cfg3 cfg5 cfg4r; do
  python profiles/summarize_ncu.py full $O/r02_ncu_${c}_full.ncu-rep $c $O/r02_ncu_${c}_full.json > /dev/null 2>&1
  python profiles/summarize_ncu.py launches $O/r02_ncu_${c}_launches.csv $O/r02_ncu_${c}_launches.txt > /dev/null 2>&1
done
cp profiles/ncu_traffic.json $O/ncu_traffic.json
rm -f $O/*.ncu-rep
echo summarized
