#!/bin/bash
# ncu evidence for the wave kernels (run on the GPU box via gpurun):
#   1. the plain bench line (must exit 0 before any ncu pass),
#   2. the launch list (gpu__time_duration.sum, --clock-control none),
#   3. one `--set full --import-source on` capture of k_tile / k_ml_walk / k_wave_sort (three
#      consecutive waves in the middle of the run) and of one k_far_walk launch,
#      so `ncu -i --page source` maps to the CUDA lines.
# env: CFG (default 5), TAG (file suffix), SKIP (kernel-filtered launch index of the capture, default 300)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
CFG=${CFG:-5}
TAG=${TAG:-cur}
ARGS="--config $CFG --no-cpu-baseline --no-table-e2e --no-file-e2e --no-cfg4"
timeout 300 python bench.py $ARGS --steps 5 --warmup 3 > gpurun_out/prof_plain_$TAG.json 2> gpurun_out/prof_plain_$TAG.err || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/launches_cfg${CFG}_$TAG.csv \
  python bench.py $ARGS --steps 1 --warmup 0 > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_tile|k_ml_walk|k_scatter|k_wave_sort" \
  --launch-skip ${SKIP:-300} --launch-count 3 -o gpurun_out/full_cfg${CFG}_$TAG -f \
  python bench.py $ARGS --steps 1 --warmup 0 > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_far_walk" \
  --launch-skip 1 --launch-count 1 -o gpurun_out/full_walk_cfg${CFG}_$TAG -f \
  python bench.py $ARGS --steps 1 --warmup 0 > gpurun_out/ncu_walk_$TAG.log 2>&1
echo prof done
