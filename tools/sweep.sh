#!/bin/bash
# Build-knob sweep on the GPU box: for each flag set, rebuild liblinprim.so and run the C5 bench;
# prints the flag set, Mpx/s and the per-stage times.   usage: tools/sweep.sh "-DA=1" "-DA=2" ...
for f in "$@"; do
  LP_EXTRA_NVCC_FLAGS="$f" python -c "from paper_2501_16312_b200 import _build; _build.build(force=True)" > /dev/null 2>&1 || { echo "$f build failed"; continue; }
  python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['value'], {k: round(v,4) for k,v in d['stages_ms_per_view'].items()})"
done
