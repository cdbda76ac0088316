export PYTHONUNBUFFERED=1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_scatter_ml|k_scatter_far|k_tile" --launch-skip 300 --launch-count 3 -o gpurun_out/prof_r1m -f python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-table-e2e > gpurun_out/ncu_r1m.log 2>&1
tail -2 gpurun_out/ncu_r1m.log
