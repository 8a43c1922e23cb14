#!/bin/bash
# ncu evidence for round 2 (run under gpurun; outputs land in gpurun_out/).  Summaries are made
# here afterwards by scripts/refresh_profiles_r02.sh.
set -x
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU="ncu --clock-control none"
# (1) launch list of the bench command itself (headline c3, no extra workloads); SKIP_LIST=1 skips
[ -n "$SKIP_LIST" ] || $NCU --metrics gpu__time_duration.sum -s 200 -c 9000 --csv --log-file gpurun_out/r02_launches_bench_c3.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --extra '' > gpurun_out/r02_launches_bench_c3.log 2>&1
# (2) full-set captures of the K1 kernels: cold (default cache control) and warm
for w in c3 c4; do
  $NCU --set full --import-source on -k regex:"hybrid_" -s 200 -c 4 -o gpurun_out/r02_prof_k1_$w -f python scripts/profile_target.py $w 60 > gpurun_out/r02_prof_k1_$w.log 2>&1
  $NCU --cache-control none --set full -k regex:"hybrid_" -s 200 -c 4 -o gpurun_out/r02_prof_k1_${w}_warm -f python scripts/profile_target.py $w 60 > gpurun_out/r02_prof_k1_${w}_warm.log 2>&1
done
$NCU --set full --import-source on -k regex:clenshaw_step_ -s 200 -c 2 -o gpurun_out/r02_prof_k1_c2 -f python scripts/profile_target.py c2 12 > gpurun_out/r02_prof_k1_c2.log 2>&1
# (3) the dense kernels at full basis size and in the recovery of a COMPLETE c3 solve (630 basis
# vectors, 247 wanted pairs): K3 gemm_tn<1> / K4 gemm_nn<1,true> late in the factorization, K6
# lift gemm_nn<8,false>, K8 gemm_tn<4>, K9 rotation gemm_nn
$NCU --set full --kernel-name-base demangled -k regex:"gemm_tn_kernel<1>" -s 1500 -c 2 -o gpurun_out/r02_prof_k3_c3 -f python scripts/profile_target.py c3 0 > gpurun_out/r02_prof_k3_c3.log 2>&1
$NCU --set full --kernel-name-base demangled -k regex:"gemm_nn_kernel<1, *true>" -s 1500 -c 2 -o gpurun_out/r02_prof_k4_c3 -f python scripts/profile_target.py c3 0 > gpurun_out/r02_prof_k4_c3.log 2>&1
$NCU --set full --kernel-name-base demangled -k regex:"gemm_nn_kernel<8" -c 3 -o gpurun_out/r02_prof_k6_c3 -f python scripts/profile_target.py c3 0 > gpurun_out/r02_prof_k6_c3.log 2>&1
$NCU --set full --kernel-name-base demangled -k regex:"gemm_tn_kernel<4>" -c 3 -o gpurun_out/r02_prof_k8_c3 -f python scripts/profile_target.py c3 0 > gpurun_out/r02_prof_k8_c3.log 2>&1
ls -la gpurun_out
