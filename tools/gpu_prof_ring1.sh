#!/bin/bash
# full ncu capture of one ring-sweep launch (d=0: x, d=1: y) -> raw/source CSVs
set -o pipefail
tag=$1; d=$2; shift 2
ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-k_ring} --launch-skip $((6 + d)) -c 1 -o gpurun_out/${tag}_d$d \
  python bench.py --no-cpu-baseline --no-extra --e2e-steps 0 --steps 1 --warmup 3 "$@" > gpurun_out/${tag}_d${d}_ncu.log 2>&1 || exit 1
ncu -i gpurun_out/${tag}_d$d.ncu-rep --page raw --csv > gpurun_out/${tag}_d${d}_raw.csv 2>/dev/null
ncu -i gpurun_out/${tag}_d$d.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_d${d}_src.csv 2>/dev/null
rm -f gpurun_out/${tag}_d$d.ncu-rep
echo done
