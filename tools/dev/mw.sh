export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python tools/dev/quick_gpu_check.py > gpurun_out/quick_check.log 2>&1; tail -1 gpurun_out/quick_check.log
timeout 900 python -m pytest tests -m gpu -x -q -k "pins or genbin or fresh or random or shard or rebase" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for c in 5 4; do for mw in 2 1; do
  echo -n "MW=$mw "; ERATO_GPU_ML_WINDOW=$mw timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-table-e2e 2>&1 | python tools/dev/bsum.py
done; done
