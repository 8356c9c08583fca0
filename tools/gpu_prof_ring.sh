#!/bin/bash
# full ncu captures of the two ring-sweep launches of one x+y application
# (x = first k_ring launch after warm-up, y = the next) -> raw/source CSVs
set -o pipefail
tag=$1; shift
python bench.py --no-cpu-baseline --no-extra --e2e-steps 0 --steps 1 --warmup 3 "$@" > gpurun_out/${tag}_plain.json || exit 1
for d in 0 1; do
  ncu --set full --import-source on --clock-control none -k regex:k_ring --launch-skip $((6 + d)) -c 1 -o gpurun_out/${tag}_d$d \
    python bench.py --no-cpu-baseline --no-extra --e2e-steps 0 --steps 1 --warmup 3 "$@" > gpurun_out/${tag}_d${d}_ncu.log 2>&1 || exit 1
  ncu -i gpurun_out/${tag}_d$d.ncu-rep --page raw --csv > gpurun_out/${tag}_d${d}_raw.csv 2>/dev/null
  ncu -i gpurun_out/${tag}_d$d.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_d${d}_src.csv 2>/dev/null
  ncu -i gpurun_out/${tag}_d$d.ncu-rep --page details --csv > gpurun_out/${tag}_d${d}_details.csv 2>/dev/null
  rm -f gpurun_out/${tag}_d$d.ncu-rep
done
echo done
