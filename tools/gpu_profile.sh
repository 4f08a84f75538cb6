#!/bin/bash
# Profiling pass on the GPU box (run under gpurun). Writes into gpurun_out/.
# usage: tools/gpu_profile.sh <tag> [bench args...]
set -u
TAG=${1:-prof}; shift || true
ARGS="${*:---steps 3 --warmup 3 --no-cpu-baseline}"
mkdir -p gpurun_out
CMD="python bench.py $ARGS"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pole_kernel -s 2 -c 1 \
    -o gpurun_out/${TAG}_pole $CMD > gpurun_out/${TAG}_ncu2.log 2>&1
echo "profile rc=$?"
