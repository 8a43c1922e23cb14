#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU="ncu --clock-control none"
$NCU --set full --import-source on -k regex:clenshaw_step_tasks -s 200 -c 2 -o gpurun_out/prof_k1t_c3 -f python scripts/profile_target.py c3 30 > gpurun_out/prof_k1t_c3.log 2>&1
$NCU --set full --import-source on -k regex:clenshaw_step_tasks -s 200 -c 2 -o gpurun_out/prof_k1t_c2 -f python scripts/profile_target.py c2 9 > gpurun_out/prof_k1t_c2.log 2>&1
tail -2 gpurun_out/prof_k1t_c3.log gpurun_out/prof_k1t_c2.log
