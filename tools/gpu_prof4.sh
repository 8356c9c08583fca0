#!/bin/bash
# full ncu captures of the four checkpointed-sweep kernels (one launch each,
# after warm-up) -> raw CSVs + SASS source CSVs under gpurun_out/
set -o pipefail
tag=$1; shift
python bench.py --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 3 "$@" > gpurun_out/${tag}_plain.json || exit 1
for k in k_xck1 k_xck2 k_yck1 k_yck2; do
  ncu --set full --import-source on --clock-control none -k regex:"$k" -c 1 -o gpurun_out/${tag}_$k \
    python bench.py --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 3 "$@" > gpurun_out/${tag}_${k}_ncu.log 2>&1 || exit 1
  ncu -i gpurun_out/${tag}_$k.ncu-rep --page raw --csv > gpurun_out/${tag}_${k}_raw.csv 2>/dev/null
  ncu -i gpurun_out/${tag}_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_${k}_src.csv 2>/dev/null
  ncu -i gpurun_out/${tag}_$k.ncu-rep --page details --csv > gpurun_out/${tag}_${k}_details.csv 2>/dev/null
  rm -f gpurun_out/${tag}_$k.ncu-rep
done
echo done
