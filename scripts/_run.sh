run() { echo "== split=$1 pgbase=$2 kernel=$3"; FLZ_SPLIT=$1 FLZ_K1_PG_BASE=$2 FLZ_K1_KERNEL=$3 timeout 300 python scripts/k1_bench.py all 2>&1 | sed -n '4p;5p;8p'; }
run 1 12 mixed; run 1 6 mixed; run 1 24 mixed; run 1 48 mixed
FLZ_SPLIT=1 FLZ_K1_PG_BASE=12 FLZ_K1_KERNEL=mixed ncu --cache-control none --clock-control none --section SpeedOfLight --section Occupancy --section LaunchStats -k regex:clenshaw_step_ug -s 20 -c 2 python scripts/k1_profile.py c3 3 12 > gpurun_out/ncu_c3_warm.txt 2>&1
