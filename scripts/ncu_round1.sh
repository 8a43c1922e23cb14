#!/bin/bash
# ncu evidence for round 1 (run under gpurun; outputs land in gpurun_out/)
set -x
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU="ncu --clock-control none"
# (1) launch list of the bench command itself: the launches of the first block steps of C2
$NCU --metrics gpu__time_duration.sum -s 300 -c 5000 --csv --log-file gpurun_out/launches_bench_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/launches_bench_c2.log 2>&1
# (2) launch lists of short, basis-capped solves: every phase (filter, orthogonalisation, recovery)
$NCU --metrics gpu__time_duration.sum -s 700 -c 4500 --csv --log-file gpurun_out/launches_c2.csv python scripts/profile_target.py c2 12 > gpurun_out/launches_c2.log 2>&1
$NCU --metrics gpu__time_duration.sum -s 700 -c 4500 --csv --log-file gpurun_out/launches_c3.csv python scripts/profile_target.py c3 60 > gpurun_out/launches_c3.log 2>&1
# (3) full-set captures of the top kernels
$NCU --set full --import-source on -k regex:clenshaw_step_ -s 200 -c 3 -o gpurun_out/prof_k1_c2 -f python scripts/profile_target.py c2 12 > gpurun_out/prof_k1_c2.log 2>&1
$NCU --set full --import-source on -k regex:clenshaw_step_ -s 200 -c 3 -o gpurun_out/prof_k1_c3 -f python scripts/profile_target.py c3 60 > gpurun_out/prof_k1_c3.log 2>&1
$NCU --set full --import-source on -k regex:clenshaw_step_ -s 200 -c 3 -o gpurun_out/prof_k1_c4 -f python scripts/profile_target.py c4 30 > gpurun_out/prof_k1_c4.log 2>&1
$NCU --set full --import-source on -k regex:gemm_tn_kernel -s 60 -c 2 -o gpurun_out/prof_tn_c3 -f python scripts/profile_target.py c3 60 > gpurun_out/prof_tn_c3.log 2>&1
$NCU --set full --import-source on -k regex:gemm_nn_kernel -s 60 -c 2 -o gpurun_out/prof_nn_c3 -f python scripts/profile_target.py c3 60 > gpurun_out/prof_nn_c3.log 2>&1
# (4) the same K1 launches with warm caches (no flush between replays): what the timed runs see
$NCU --cache-control none --section SpeedOfLight --section Occupancy --section MemoryWorkloadAnalysis --section LaunchStats -k regex:clenshaw_step_ -s 200 -c 2 python scripts/profile_target.py c2 12 > gpurun_out/k1_c2_warm.txt 2>&1
$NCU --cache-control none --section SpeedOfLight --section Occupancy --section MemoryWorkloadAnalysis --section LaunchStats -k regex:clenshaw_step_ -s 200 -c 2 python scripts/profile_target.py c3 60 > gpurun_out/k1_c3_warm.txt 2>&1
ls -la gpurun_out
