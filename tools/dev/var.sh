# parity probe on the default build, then cfg benches for each variant in build_var/
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python tools/dev/quick_gpu_check.py > gpurun_out/quick_check.log 2>&1; tail -2 gpurun_out/quick_check.log
CFGS=${CFGS:-5} bash tools/dev/run_var.sh
