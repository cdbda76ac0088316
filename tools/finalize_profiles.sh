#!/bin/bash
# Round-end evidence (run on the GPU box via gpurun): the default bench line, the reference arm,
# the ncu launch lists + full captures of cfg5 and cfg4, the Table-1 curve.  Outputs under gpurun_out/;
# summarise here with tools/ncu_summarize.py / tools/ncu_lines.py and copy into profiles/.
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/final_bench_default.json 2> gpurun_out/final_bench_default.err
tail -c 600 gpurun_out/final_bench_default.json
timeout 900 python bench.py --impl reference > gpurun_out/final_bench_reference.json 2> gpurun_out/final_bench_reference.err
TAG=final bash tools/profile.sh
CFG=4 SKIP=100 TAG=final4 bash tools/profile.sh
timeout 900 python tools/table1.py --out gpurun_out/final_table1 > /dev/null 2> gpurun_out/final_table1.err
echo finalize done
