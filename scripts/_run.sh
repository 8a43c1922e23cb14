(timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3)
python scripts/sync_vs_overlap.py tiny c1 c3 c2 2>&1 | tail -4
python bench.py --workload c3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c3_b.json
python bench.py --workload c1 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c1_b.json
python bench.py --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c2_b.json
