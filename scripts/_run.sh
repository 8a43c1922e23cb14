for lay in i planar; do
FLZ_K1_LAYOUT=$lay ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section SchedulerStats --section WarpStateStats --section Occupancy --cache-control none --clock-control none -k regex:clenshaw_step_ug_warp -s 20 -c 1 python scripts/k1_profile.py c2 3 12 > gpurun_out/lean_$lay.txt 2>&1
done
