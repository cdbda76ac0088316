set -x
export PYTHONUNBUFFERED=1
ERATO_GPU_SO=paper_1111_3297_b200/liberato_gpu_debug.so timeout 600 python tools/dev/quick_gpu_check.py > gpurun_out/qc_dbg.log 2>&1; tail -3 gpurun_out/qc_dbg.log
timeout 600 python tools/dev/quick_gpu_check.py > gpurun_out/qc.log 2>&1; tail -3 gpurun_out/qc.log
for c in 5 4 3; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-table-e2e 2>/dev/null | python tools/dev/bsum.py; done
for c in 5 4; do ERATO_GPU_SCATTER=fused timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-table-e2e 2>/dev/null | python tools/dev/bsum.py; done
