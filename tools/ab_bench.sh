#!/bin/bash
# A/B timing of library variants (variants/libqvts_*.so): bench.py kernel times per variant, twice.
for rep in 1 2 3; do
  for f in variants/libqvts_*.so; do
    n=$(basename $f .so)
    QVTS_LIB=$PWD/$f timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline > gpurun_out/ab_$n.log 2>&1
    python -c "
import json,sys; d=json.loads(open('gpurun_out/ab_$n.log').read().strip().splitlines()[-1])
print('$n', round(d['ms_per_step'],2), {k: round(v/4,2) for k,v in d['kernel_ms'].items() if v > 0.5})"
  done
done
