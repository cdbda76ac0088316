export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python tools/dev/quick_gpu_check.py > gpurun_out/quick_check.log 2>&1; tail -1 gpurun_out/quick_check.log
timeout 900 python -m pytest tests -m gpu -x -q -k "pins or invariant or genbin or random" 2>&1 | tail -1
echo -n "ML_BINS=0 "; ERATO_GPU_ML_BINS=0 timeout 300 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-table-e2e 2>&1 | python tools/dev/bsum.py
CFGS="5 4" bash tools/dev/var_nocheck.sh
