#!/bin/bash
# quick per-config bench summary: bash scratch/quick_bench.sh cfg1 cfg2 ...
for c in "$@"; do
  timeout 300 python bench.py --config $c --no-cpu --e2e-steps 0 > gpurun_out/qb_$c.json 2> gpurun_out/qb_$c.err
  python3 -c "
import json; d=json.loads(open('gpurun_out/qb_$c.json').read().splitlines()[-1])
k=d['roofline']['kernels'] if d.get('roofline') else {}
print('$c', round(d['value'],2), 'Gkeys/s step', round(d['ms_per_step']*1e3,1), 'us', {n: round(v['avg_ms']*1e3,1) for n,v in k.items()}, d['correct'])" || tail -5 gpurun_out/qb_$c.err
done
