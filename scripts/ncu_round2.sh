#!/bin/bash
# ncu evidence for round 2 (run under gpurun).  Every capture is exported to a raw-page CSV on
# the GPU box and the .ncu-rep is deleted there (gpurun brings back at most 64 MiB); the
# summaries under profiles/ are made here afterwards by scripts/refresh_profiles_r02.sh.
set -x
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU="ncu --clock-control none"
cap() {   # cap <name> <ncu args...> -- <python args...>
  local name=$1; shift
  local args=()
  while [ "$1" != "--" ]; do args+=("$1"); shift; done
  shift
  $NCU --set full "${args[@]}" -o gpurun_out/$name -f python "$@" > gpurun_out/$name.log 2>&1
  ncu -i gpurun_out/$name.ncu-rep --page raw --csv > gpurun_out/$name.csv 2>/dev/null
  rm -f gpurun_out/$name.ncu-rep
}
# (1) launch list of the bench command itself (headline c3, no extra workloads); SKIP_LIST=1 skips
[ -n "$SKIP_LIST" ] || $NCU --metrics gpu__time_duration.sum -s 200 -c 9000 --csv --log-file gpurun_out/r02_launches_bench_c3.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --extra '' > gpurun_out/r02_launches_bench_c3.log 2>&1
# (2) full-set captures of the K1 kernels: cold (default cache control) and warm; SKIP_K1=1 skips
[ -n "$SKIP_K1" ] || for w in c3 c4; do
  cap r02_prof_k1_$w -k regex:hybrid_ -s 200 -c 4 -- scripts/profile_target.py $w 60
  cap r02_prof_k1_${w}_warm --cache-control none -k regex:hybrid_ -s 200 -c 4 -- scripts/profile_target.py $w 60
done
[ -n "$SKIP_K1" ] || cap r02_prof_k1_c2 -k regex:clenshaw_step_ -s 200 -c 2 -- scripts/profile_target.py c2 12
# (3) the dense kernels at full basis size and in the recovery of a COMPLETE c3 solve (630 basis
# vectors, 247 wanted pairs): K3 gemm_tn<1> / K4 gemm_nn<1,true> late in the factorization, K6
# lift gemm_nn<8,false>, K8 gemm_tn<4>, K9 rotation gemm_nn
cap r02_prof_k3_c3 --kernel-name-base demangled -k "regex:gemm_tn_kernel<.int.1>" -s 1200 -c 2 -- scripts/profile_target.py c3 0
cap r02_prof_k4_c3 --kernel-name-base demangled -k "regex:gemm_nn_kernel<.int.1, .bool.1>" -s 1200 -c 2 -- scripts/profile_target.py c3 0
cap r02_prof_k6_c3 --kernel-name-base demangled -k "regex:gemm_nn_kernel<.int.8" -c 3 -- scripts/profile_target.py c3 0
cap r02_prof_k8_c3 --kernel-name-base demangled -k "regex:gemm_tn_kernel<.int.4>" -c 3 -- scripts/profile_target.py c3 0
ls -la gpurun_out
