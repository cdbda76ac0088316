export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python tools/dev/quick_gpu_check.py > gpurun_out/quick_check.log 2>&1; tail -2 gpurun_out/quick_check.log
for c in ${CFGS:-5 4 3 2}; do
timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-table-e2e 2>&1 | python tools/dev/bsum.py
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
