#!/bin/bash
# One GPU session: gpu tests, the driver's bench line, the reference arm (short),
# and the ncu launch list of the bench. Usage (on the box): tools/gpu_round.sh <tag> [pytest -k expr]
set -o pipefail
tag=$1; kexpr=${2:-}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
if [ -n "$kexpr" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$kexpr" > gpurun_out/${tag}_pytest.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest.log 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err
echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 --no-extra \
  --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/${tag}_pytest.log
