#!/bin/bash
# A/B of runtime tuning knobs: each argument is "NAME:ENV=VAL ENV2=VAL2"
for rep in 1 2; do
  for spec in "$@"; do
    n=${spec%%:*}; envs=${spec#*:}
    env $envs timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline > gpurun_out/ab_$n.log 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/ab_$n.log').read().strip().splitlines()[-1])
print('$n', round(d['ms_per_step'],2), {k: round(v/4,2) for k,v in d['kernel_ms'].items() if v > 0.5})"
  done
done
