# one ncu --set full capture (with source) of kernels matching $K at cfg ${CFG:-5}
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
CFG=${CFG:-5}; TAG=${TAG:-cur}; K=${K:-k_scatter_ml}
timeout 300 python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-table-e2e > gpurun_out/prof_plain_$TAG.json 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$K" --launch-skip ${SKIP:-100} --launch-count ${CNT:-1} \
  -o gpurun_out/full_${TAG} -f python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu-baseline --no-table-e2e > gpurun_out/ncu_full_$TAG.log 2>&1
echo prof done
