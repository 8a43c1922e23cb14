#!/bin/bash
# ncu evidence for round 1 (run under gpurun; outputs land in gpurun_out/)
set -x
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU="ncu --clock-control none"
# launch lists (every launch with its device time) of a short, basis-capped solve
$NCU --metrics gpu__time_duration.sum -s 700 -c 4000 --csv --log-file gpurun_out/launches_c2.csv python scripts/profile_target.py c2 12 > gpurun_out/launches_c2.log 2>&1
$NCU --metrics gpu__time_duration.sum -s 700 -c 4000 --csv --log-file gpurun_out/launches_c3.csv python scripts/profile_target.py c3 60 > gpurun_out/launches_c3.log 2>&1
# full-set captures of the top kernels
$NCU --set full --import-source on -k regex:clenshaw_step -s 200 -c 3 -o gpurun_out/prof_k1_c2 -f python scripts/profile_target.py c2 12 > gpurun_out/prof_k1_c2.log 2>&1
$NCU --set full --import-source on -k regex:clenshaw_step -s 200 -c 3 -o gpurun_out/prof_k1_c3 -f python scripts/profile_target.py c3 60 > gpurun_out/prof_k1_c3.log 2>&1
$NCU --set full --import-source on -k regex:gemm_tn_kernel -s 60 -c 2 -o gpurun_out/prof_tn_c3 -f python scripts/profile_target.py c3 60 > gpurun_out/prof_tn_c3.log 2>&1
$NCU --set full --import-source on -k regex:gemm_nn_kernel -s 60 -c 2 -o gpurun_out/prof_nn_c3 -f python scripts/profile_target.py c3 60 > gpurun_out/prof_nn_c3.log 2>&1
ls -la gpurun_out
