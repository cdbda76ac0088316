# A/B an env knob: ENVAB="NAME=val1 NAME=val2" CFGS="5 4"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python tools/dev/quick_gpu_check.py > gpurun_out/quick_check.log 2>&1; tail -1 gpurun_out/quick_check.log
for c in ${CFGS:-5}; do
  for kv in $ENVAB; do
    echo -n "$kv "
    env $kv timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-table-e2e 2>&1 | python tools/dev/bsum.py
  done
done
