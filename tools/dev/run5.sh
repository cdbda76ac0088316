export PYTHONUNBUFFERED=1
ERATO_GPU_SO=paper_1111_3297_b200/liberato_gpu_debug.so timeout 600 python tools/dev/quick_gpu_check.py > gpurun_out/qc_dbg.log 2>&1; tail -1 gpurun_out/qc_dbg.log
CFGS="5" bash tools/dev/run_var.sh 2>&1
