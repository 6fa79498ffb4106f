#!/bin/bash
# A/B of the fused leaf level (QVTS_FUSED_LEAF=1, default) against materialised leaf parents (=0).
for rep in 1 2; do
  for f in 0 1; do
    QVTS_FUSED_LEAF=$f timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline > gpurun_out/ab_fused$f.log 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/ab_fused$f.log').read().strip().splitlines()[-1])
print('fused=$f', round(d['ms_per_step'],2), round(d['value']/1e6,1), 'M upd/s', {k: round(v/4,2) for k,v in d['kernel_ms'].items() if v > 0.5})"
  done
done
