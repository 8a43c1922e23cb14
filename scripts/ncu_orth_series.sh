#!/bin/bash
# duration of every big projection / update launch of the orth microbench as the basis grows
shape=${1:-c3}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"ts_update|gemm_tn_kernel|gemm_nn_kernel" --csv --log-file gpurun_out/orth_series_$shape.csv python scripts/orth_bench.py $shape > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/orth_series_$shape.csv")) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); mi=h.index("Metric Name"); vi=h.index("Metric Value"); ii=h.index("ID")
d={}
for r in rows[1:]:
    d.setdefault(int(r[ii]),[r[ki][:30],0,0])
    if "time" in r[mi]: d[int(r[ii])][1]=float(r[vi].replace(",",""))
    else: d[int(r[ii])][2]=float(r[vi].replace(",",""))
# keep launches that read > 20 MB
big=[(i,v) for i,v in sorted(d.items()) if v[2]>20e6 or v[2]>20 and v[2]<1e5]
print(len(d), len(big))
for i,v in big[::max(1,len(big)//60)]:
    mb=v[2]/1e6 if v[2]>1e5 else v[2]
    print(i, v[0], "%.1f MB %.1f us %.2f TB/s"%(mb, v[1]/1e3 if v[1]>1e3 else v[1], mb/ (v[1]/1e3 if v[1]>1e3 else v[1]) /1e6*1e6/1e6))
PY
