#!/bin/bash
# A/B timing of env-selected kernel variants (run on the GPU box):
#   VARIANTS="DEFAULT=1 ERATO_GPU_WHEEL=210,ERATO_GPU_FAR_DIV=1" CFGS="5 4" bash tools/ab.sh   (comma = several vars)
# prints ms/step, the timed steps one by one and the per-kernel split of a short bench run per variant.
export PYTHONUNBUFFERED=1
for c in ${CFGS:-5}; do
  for v in ${VARIANTS:-DEFAULT=1}; do
    env $(echo "$v" | tr "," " ") timeout 300 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-table-e2e \
      --no-file-e2e --no-cfg4 2>/dev/null | CFG=$c VAR=$v python -c '
import json, os, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print("cfg" + os.environ["CFG"], os.environ["VAR"], round(d["ms_per_step"], 3), "ms", d.get("step_ms"),
      d["roofline_run"]["kernel_split_ms"], "clk", d["clocks"]["sm_mhz"])'
  done
done
