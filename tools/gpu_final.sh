#!/bin/bash
# End-of-round evidence: GPU tests, bench lines (3rd-RF default, 1st-RF), reference arm, launch
# lists, full captures of the 1st-RF kernels, acceptance case and CG solve, config table.
set -o pipefail
tag=$1
bash tools/gpu_round.sh ${tag}
bash tools/gpu_accept.sh ${tag}
bash tools/gpu_rf1_final.sh ${tag}
