#!/bin/bash
# ncu --set full of one kernel of the C4 plan step (tools/prof_plan.py runs 2 plan steps)
# usage (under gpurun): bash tools/ncu_kernel.sh <tag> <kernel-regex> <skip-launches> <count> [cfg]
tag=$1; kre=$2; skip=${3:-0}; cnt=${4:-1}; cfg=${5:-C4}
python tools/prof_plan.py $cfg > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c $cnt \
    -o gpurun_out/prof_$tag python tools/prof_plan.py $cfg > gpurun_out/ncu_$tag.log 2>&1
echo "ncu_rc=$?"
