#!/bin/bash
# usage (on the GPU box): tools/gpu_prof.sh <kernel-regex> <name> [bench args...]
# full ncu capture of the first matching launch after warm-up + SASS source dump
set -o pipefail
re=$1; name=$2; shift 2
python bench.py --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 3 "$@" > gpurun_out/${name}_plain.json || exit 1
ncu --set full --import-source on --clock-control none -k regex:"$re" -c 1 -o gpurun_out/$name \
  python bench.py --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 3 "$@" > gpurun_out/${name}_ncu.log 2>&1 || exit 1
ncu -i gpurun_out/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/${name}_src.csv 2>/dev/null
ncu -i gpurun_out/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
rm -f gpurun_out/$name.ncu-rep
echo done
