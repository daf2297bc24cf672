#!/bin/bash
# cfg4 count-kernel shape sweep (TMA ring depth vs shared table size)
for s in 2 5 6 7 2; do
  CAFS_HC_SHAPE=$s timeout 300 python bench.py --no-cpu --e2e-steps 0 > gpurun_out/hc_shape_$s.json 2>&1
  python3 -c "
import json,sys; d=json.loads(open('gpurun_out/hc_shape_$s.json').read().splitlines()[-1])
k=d['roofline']['kernels']; print('shape $s', round(d['value'],1), 'count', round(k['count']['avg_ms']*1e3,1), 'us', round(k['count']['GB/s']), 'emit', round(k['emit']['avg_ms']*1e3,1), d['correct'])"
done
