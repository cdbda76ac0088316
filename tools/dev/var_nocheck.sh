export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
: > gpurun_out/var_summary.txt
for so in build_var/liberato_gpu_*.so; do
  for c in ${CFGS:-5}; do
    ERATO_GPU_SO=$so timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-table-e2e > gpurun_out/var_out.txt 2>&1
    echo "$(basename $so) $(python tools/dev/bsum.py < gpurun_out/var_out.txt) $(grep -i error gpurun_out/var_out.txt | head -1)" >> gpurun_out/var_summary.txt
  done
done
cat gpurun_out/var_summary.txt
