# run cfg5/cfg4 bench for each built variant (tools/dev/build_variants.sh)
export PYTHONUNBUFFERED=1
for so in build_var/liberato_gpu_*.so; do
  for c in ${CFGS:-5 4}; do
    echo -n "$(basename $so) "
    ERATO_GPU_SO=$so timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-table-e2e 2>&1 | python tools/dev/bsum.py
  done
done
