export PYTHONUNBUFFERED=1
timeout 300 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-table-e2e > gpurun_out/b5.log 2>&1; tail -5 gpurun_out/b5.log | cut -c1-600
