#!/bin/bash
# one bench line per BASELINE config / dtype / filter -> gpurun_out/configs.jsonl
set -o pipefail
out=gpurun_out/configs.jsonl
: > $out
for c in C1 C2 C3 C4 C5; do
  for dt in f64 f32; do
    for o in 3 1; do
      line=$(python bench.py --config $c --dtype $dt --order $o --no-cpu-baseline --no-extra --e2e-steps 1 --steps 5 2>/dev/null | tail -1)
      echo "{\"cfg\": \"$c\", \"dtype\": \"$dt\", \"order\": $o, \"line\": $line}" >> $out
    done
  done
done
echo done
