#!/bin/bash
# time every paper_2501_16312_b200/liblinprim_v*.so (and _old) with tools/rbwd_time.py [cfg] [views]
mkdir -p gpurun_out
for l in paper_2501_16312_b200/liblinprim_old.so paper_2501_16312_b200/liblinprim_v*.so; do
  [ -f "$l" ] || continue
  LP_LIB=$PWD/$l timeout 300 python tools/rbwd_time.py "$@" 2>&1 | tail -1
done | tee gpurun_out/variants.txt
