#!/bin/bash
# Round-2 evidence for the line-resident 1st-RF: config table, the C5 1st-RF bench line and its
# launch list, full ncu captures of the x and y kernels on all 100 levels.
set -o pipefail
tag=$1
mkdir -p gpurun_out
bash tools/config_table.sh > /dev/null 2>&1; cp gpurun_out/configs.jsonl gpurun_out/${tag}_configs.jsonl
timeout 600 python bench.py --order 1 --steps 10 --warmup 3 --no-extra > gpurun_out/${tag}_bench_rf1.json 2> gpurun_out/${tag}_bench_rf1.err
echo "bench rf1 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches_rf1.csv python bench.py --order 1 --steps 2 --warmup 1 --no-extra \
  --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_ncu_rf1.log 2>&1
echo "launch list rc=$?"
bash tools/dbg/rf1_line_ncu.sh ${tag}_rf1full 100 GX,GY f64
echo "full rc=$?"
