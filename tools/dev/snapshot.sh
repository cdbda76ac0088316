# Round snapshot: bench lines (all configs; cfg5 with CPU baseline), reference arm, ncu launch list + full capture.
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/snap
O=gpurun_out/snap
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 600 python bench.py --config 5 --steps 10 --warmup 3 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
for c in 4 3 2 1; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
timeout 600 python bench.py --impl reference --config 5 --steps 3 --warmup 1 > $O/bench_reference_cfg5.json 2> $O/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_cfg5.csv \
  python bench.py --config 5 --steps 1 --warmup 0 --no-cpu-baseline --no-table-e2e > $O/ncu_launch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file $O/launches_cfg4.csv \
  python bench.py --config 4 --steps 1 --warmup 0 --no-cpu-baseline --no-table-e2e > $O/ncu_launch4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_tile|k_scatter" --launch-skip 300 --launch-count 3 \
  -o $O/full_cfg5 -f python bench.py --config 5 --steps 1 --warmup 0 --no-cpu-baseline --no-table-e2e > $O/ncu_full.log 2>&1
echo snapshot done
