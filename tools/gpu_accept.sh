#!/bin/bash
# few-plane cases: acceptance 1024^2 (device), C3 level-0 CG iteration, and their launch lists
set -o pipefail
tag=$1
mkdir -p gpurun_out
timeout 300 python tools/bench_acceptance.py > gpurun_out/${tag}_accept.json 2> gpurun_out/${tag}_accept.err
echo "accept rc=$?"
timeout 300 python tools/bench_solve.py > gpurun_out/${tag}_solve.json 2> gpurun_out/${tag}_solve.err
echo "solve rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/${tag}_accept_launches.csv python tools/bench_acceptance.py --quick \
  > gpurun_out/${tag}_accept_ncu.log 2>&1
echo "ncu rc=$?"
