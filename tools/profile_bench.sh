#!/bin/bash
# Run on the GPU box (gpurun): plain bench run, then the ncu launch list and one
# --set full capture per pipeline kernel for the same command (B200_PROFILING.md).
#   tools/profile_bench.sh <config> <tag> [kernels regex list]
set -u
CFG=${1:-c4}
TAG=${2:-r01}
KERNELS=${3:-"icq_filter icq_replay icq_prologue"}
CMD="python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu --no-e2e --no-sweep"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_${CFG}.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'icq_|lut_build' \
    --csv --log-file gpurun_out/launches_${CFG}_${TAG}.csv $CMD > gpurun_out/ncu_launches_${CFG}.log 2>&1
for K in $KERNELS; do
  # (filter / refine / replay launch once per round, kMaxRounds = 4 per batch:
  # skip whole batches so the capture is a first-round launch)
  SKIP=3
  # second batch, second round: count-mode queries list the bulk of the
  # database in round 1 (round 0 is the dense prefix)
  # (ROUND_SKIP=4 for a config whose queries stay in list mode: round 0 is their filter)
  case $K in icq_filter|icq_refine|icq_replay|icq_cl_gather|icq_cl_scan) SKIP=${ROUND_SKIP:-5};; esac
  ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 \
      -o gpurun_out/full_${CFG}_${TAG}_${K} $CMD > gpurun_out/ncu_full_${CFG}_${K}.log 2>&1
done
echo done
