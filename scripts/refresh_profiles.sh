#!/bin/bash
# Turns the ncu outputs of scripts/ncu_round1.sh (gpurun_out/) into the tracked summaries
# under profiles/ (runs here, no GPU needed).
set -e
cd "$(dirname "$0")/.."
R=${1:-r01}
for f in bench_c2 c2 c3; do python scripts/ncu_summary.py launches gpurun_out/launches_$f.csv > profiles/${R}_launches_$f.txt; done
for f in k1_c2 k1_c3 k1_c4 tn_c3 nn_c3; do python scripts/ncu_summary.py raw gpurun_out/prof_$f.ncu-rep | grep -v "hmma\|imma\|ops_path\|mem_tensor" > profiles/${R}_prof_$f.txt; done
cp gpurun_out/k1_c2_warm.txt profiles/${R}_k1_c2_warm_sections.txt
cp gpurun_out/k1_c3_warm.txt profiles/${R}_k1_c3_warm_sections.txt
python - <<'PY'
import subprocess, csv, io, json
out = {}
for w in ("c2", "c3", "c4"):
    txt = subprocess.run(["ncu", "-i", f"gpurun_out/prof_k1_{w}.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    tb = lambda v, u: float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
    vals = [tb(r[ir], units[ir]) + tb(r[iw], units[iw]) for r in rows[2:]]
    out[w] = sum(vals) / len(vals)
json.dump(out, open("profiles/k1_traffic.json", "w"), indent=1)
print(out)
PY
