#!/bin/bash
# Round-2 evidence on one GPU (run under gpurun): the default bench line (no ncu), the launch list +
# per-kernel DRAM traffic and executed lane instructions of ONE bench step (metrics pass), then one
# --set full capture per hot kernel.  Outputs under gpurun_out/prof2/; summarise with
# tools/launches.py, tools/ncu_kernels_db.py, tools/ncu_summary.py, tools/ncu_stalls.py, tools/ncu_lines.py.
set -u
O=gpurun_out/prof2
mkdir -p $O
python bench.py > $O/bench.json 2> $O/bench.err || exit 1
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --profile-step"
$B > $O/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__thread_inst_executed.sum \
    --clock-control none --profile-from-start off --csv --log-file $O/step_metrics.csv $B > $O/ncu_metrics.log 2>&1
for k in "$@"; do
  ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"^${k}" -c 1 \
      -o $O/$k $B > $O/ncu_$k.log 2>&1
done
