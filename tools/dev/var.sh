# parity probe on the default build, then cfg benches for each variant in build_var/
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python tools/dev/quick_gpu_check.py > gpurun_out/quick_check.log 2>&1; tail -2 gpurun_out/quick_check.log
for so in build_var/liberato_gpu_*.so; do
  for c in ${CFGS:-5}; do
    echo -n "$(basename $so) "
    ERATO_GPU_SO=$so timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-table-e2e > gpurun_out/var_out.txt 2>&1; python tools/dev/bsum.py < gpurun_out/var_out.txt; tail -2 gpurun_out/var_out.txt | grep -iv "^{" | head -2
  done
done
