#!/bin/bash
# ncu evidence for the second half of round 2 (run under gpurun): the orthogonalization kernels
# at full basis size (orth microbench on a 110k x 630 basis, r = 3: the C3 shape), the
# overlapped hybrid kernels on C4, and the launch list of the bench command.
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
$NCU --metrics gpu__time_duration.sum -s 200 -c 9000 --csv --log-file gpurun_out/r02b_launches_bench_c3.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --extra '' > gpurun_out/r02b_launches_bench_c3.log 2>&1
cap r02b_prof_k3_tn_full -k regex:gemm_tn_kernel -s 400 -c 2 -- scripts/orth_bench.py c3
cap r02b_prof_k4_update_full -k regex:ts_update_kernel -s 400 -c 2 -- scripts/orth_bench.py c3
cap r02b_prof_qr -k regex:block_qr_kernel -s 200 -c 2 -- scripts/orth_bench.py c3
cap r02b_prof_k4_update_c1 -k regex:ts_update_kernel -s 3400 -c 1 -- scripts/orth_bench.py c1
cap r02b_prof_k1_c4 -k regex:hybrid_ -s 200 -c 4 -- scripts/profile_target.py c4 60
cap r02b_prof_k1_c4_warm --cache-control none -k regex:hybrid_ -s 200 -c 4 -- scripts/profile_target.py c4 60
ls -la gpurun_out | tail -20
