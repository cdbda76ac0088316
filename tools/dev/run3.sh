export PYTHONUNBUFFERED=1
CFGS=5 bash tools/dev/run_var.sh > gpurun_out/var2.log 2>&1
ERATO_GPU_SO=build_var/liberato_gpu_G.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_scatter_ml|k_scatter_far" --launch-skip 200 --launch-count 2 -o gpurun_out/prof_split -f python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-table-e2e > gpurun_out/ncu_split.log 2>&1
cat gpurun_out/var2.log
