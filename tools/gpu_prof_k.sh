#!/bin/bash
# full ncu capture of one launch of a kernel: tools/gpu_prof_k.sh <tag> <regex> <skip> [bench args]
set -o pipefail
tag=$1; re=$2; skip=$3; shift 3
ncu --set full --import-source on --clock-control none -k regex:$re --launch-skip $skip -c 1 -o gpurun_out/${tag} \
  python bench.py --no-cpu-baseline --no-extra --e2e-steps 0 --steps 1 --warmup 1 "$@" > gpurun_out/${tag}_ncu.log 2>&1 || exit 1
ncu -i gpurun_out/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i gpurun_out/${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_src.csv 2>/dev/null
rm -f gpurun_out/${tag}.ncu-rep
echo done
