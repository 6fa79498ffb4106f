#!/bin/bash
# ncu --set full of the leaf kernel at C4 (tools/prof_plan.py: 2 plan steps; the 2nd leaf launch)
# usage (under gpurun): bash tools/ncu_leaf.sh <tag> [kernel-regex]
tag=${1:-leaf}; kre=${2:-k_leaf}
python tools/prof_plan.py C4 > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$kre -s 1 -c 1 \
    -o gpurun_out/prof_$tag python tools/prof_plan.py C4 > gpurun_out/ncu_$tag.log 2>&1
echo "ncu_rc=$?"
