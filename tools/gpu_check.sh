#!/bin/bash
# One GPU iteration (run under gpurun): the GPU test suite, then the default bench line.
# Usage: tools/gpu_check.sh [tag] [pytest -k expr]
set -u
T=${1:-chk}
mkdir -p gpurun_out
if [ -n "${2:-}" ]; then K="-k $2"; else K=""; fi
python -m pytest tests -m gpu -q -x -p no:cacheprovider $K > gpurun_out/pytest_$T.log 2>&1
echo "pytest_rc=$?" >> gpurun_out/pytest_$T.log
tail -3 gpurun_out/pytest_$T.log
python bench.py --no-cpu-baseline > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
echo "bench_rc=$?"
python - "$T" <<'PY'
import json, sys
t = sys.argv[1]
d = json.loads(open(f"gpurun_out/bench_{t}.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"])
print({k: v for k, v in d["stages_ms_per_view"].items()})
PY
