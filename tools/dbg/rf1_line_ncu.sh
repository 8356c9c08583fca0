#!/bin/bash
# full ncu capture of the line-resident 1st-RF kernels: tools/dbg/rf1_line_ncu.sh <tag> [nlev] [kinds] [dtype]
tag=$1; nlev=${2:-20}; kinds=${3:-GX,GY}; dt=${4:-f64}
nk=$(echo $kinds | tr "," "\n" | wc -l)
python tools/dbg/rf1_line_prof.py $nlev $kinds $dt > gpurun_out/${tag}_plain.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k "regex:k_rf1_res" --launch-skip $nk -c $nk -o gpurun_out/${tag} \
  python tools/dbg/rf1_line_prof.py $nlev $kinds $dt > gpurun_out/${tag}_ncu.log 2>&1 || exit 1
ncu -i gpurun_out/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i gpurun_out/${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_src.csv 2>/dev/null
rm -f gpurun_out/${tag}.ncu-rep
echo done
