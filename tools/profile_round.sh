#!/bin/bash
# Profile evidence of the C5 step on the GPU box (run under gpurun, one GPU):
#   1. the bench itself (exits 0 without ncu first),
#   2. the launch list of one step (gpu__time_duration.sum),
#   3. one `ncu --set full` capture per hot kernel (first launch in the profiled step).
# Outputs under gpurun_out/prof/; summarise here with tools/ncu_*.py into profiles/<round>/.
set -u
O=gpurun_out/prof
mkdir -p $O
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --profile-step"
python bench.py > $O/bench.json 2> $O/bench.err || exit 1
$B > $O/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file $O/launches.csv $B > $O/ncu_launches.log 2>&1
for k in "$@"; do
  ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"^${k}" -c 1 \
      -o $O/$k $B > $O/ncu_$k.log 2>&1
done
