#!/bin/bash
# Run on the GPU box (gpurun): plain bench run, then the ncu launch list and one
# --set full capture of the scan kernel for the same command (B200_PROFILING.md).
#   tools/profile_bench.sh <config> <tag>
set -u
CFG=${1:-c4}
TAG=${2:-r01}
CMD="python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu --no-e2e"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_${CFG}.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'icq_|lut_build' \
    --csv --log-file gpurun_out/launches_${CFG}_${TAG}.csv $CMD > gpurun_out/ncu_launches_${CFG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:icq_scan -s 1 -c 1 \
    -o gpurun_out/full_${CFG}_${TAG} $CMD > gpurun_out/ncu_full_${CFG}.log 2>&1
echo done
