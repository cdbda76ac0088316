#!/bin/bash
# The sanitizer substitute (compute-sanitizer is closed on the GPU pool): the
# GPU parity tests against the EG_DEBUG build, whose device-side bounds checks
# (tile offsets of hit records, hit-list / bucket indices against their
# allocations, medium start offsets, wheel/mod-7 state) trap on any violation.
#   bash tools/debug_checks.sh   (on the GPU box; writes gpurun_out/debug_checks.log)
mkdir -p gpurun_out
python -c "from paper_1111_3297_b200.build import build; build(debug=True)" > /dev/null
ERATO_GPU_SO=paper_1111_3297_b200/liberato_gpu_debug.so timeout 1500 python -m pytest tests/test_gpu_parity.py \
  tests/test_gpu_output_multi.py -q -p no:cacheprovider \
  -k "small or random or f0 or overlap or invariants or inject or mod210 or stream or overflow or genbin or near_2p64 or edge or rebase" \
  > gpurun_out/debug_checks.log 2>&1
tail -3 gpurun_out/debug_checks.log
