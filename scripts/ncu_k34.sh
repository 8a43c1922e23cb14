cd "$(dirname "$0")/.."
NCU="ncu --clock-control none"
cap() { local name=$1; shift; local args=(); while [ "$1" != "--" ]; do args+=("$1"); shift; done; shift
  $NCU --set full "${args[@]}" -o gpurun_out/$name -f python "$@" > gpurun_out/$name.log 2>&1
  ncu -i gpurun_out/$name.ncu-rep --page raw --csv > gpurun_out/$name.csv 2>/dev/null; rm -f gpurun_out/$name.ncu-rep; }
cap r02_prof_k3_c3 --kernel-name-base demangled -k "regex:gemm_tn_kernel<.int.1>" -s 1200 -c 2 -- scripts/profile_target.py c3 0
cap r02_prof_k4_c3 --kernel-name-base demangled -k "regex:gemm_nn_kernel<.int.1, .bool.1>" -s 1200 -c 2 -- scripts/profile_target.py c3 0
