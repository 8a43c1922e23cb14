#!/bin/bash
# per-kernel durations of the hybrid kernels (cold cache, serialised): scripts/ncu_hy.sh c3 libflz.so [tag]
shape=$1; lib=$2; tag=${3:-x}
FLZ_LIB=$PWD/paper_2409_15053_b200/$lib ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.max,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__occupancy_limit_shared_mem,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,l1tex__t_sector_hit_rate.pct \
  --clock-control none -k regex:hybrid --launch-skip 40 -c 6 --csv --log-file gpurun_out/ncu_hy_${shape}_${tag}.csv python scripts/k1_one.py $shape 4 > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/ncu_hy_${shape}_${tag}.csv")) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); mi=h.index("Metric Name"); vi=h.index("Metric Value"); ii=h.index("ID")
out={}
for r in rows[1:]:
    out.setdefault((r[ii],r[ki][:40]),{})[r[mi]]=r[vi]
for k,v in out.items():
    print("${shape} ${tag}",k[1], " ".join("%s=%s"%(a.split("__")[-1][:28],b) for a,b in v.items()))
PY
