export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python tools/dev/quick_gpu_check.py > gpurun_out/quick_check.log 2>&1; tail -2 gpurun_out/quick_check.log
timeout 1200 python -m pytest tests -m gpu -x -q ${PYK:+-k "$PYK"} > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
CFGS="${CFGS:-5 4 3 2}" bash tools/dev/var.sh 2>&1 | grep -v ALL_OK | grep -v "count="
