# Per-kernel device times of one config (ncu launch list; cold-cache, serialised):
#   gpurun -- 'bash profiles/kt.sh cfg3 [extra bench args]'
c=$1; shift
args="--config $c --steps 2 --warmup 1 --no-cpu --e2e-steps 0 $*"
python bench.py $args > /dev/null 2>&1 || { echo "bench failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/kt_$c.csv python bench.py $args > /dev/null 2>&1
python profiles/summarize_ncu.py launches gpurun_out/kt_$c.csv gpurun_out/kt_$c.txt > /dev/null 2>&1
grep -v "^#" gpurun_out/kt_$c.txt | grep -v "at::\|gen_" | head -${KT_LINES:-14}
