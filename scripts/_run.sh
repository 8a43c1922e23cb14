(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3)
timeout 300 python scripts/k1_bench.py all 2>&1 | tail -8
python bench.py --workload c3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c3_b.json
