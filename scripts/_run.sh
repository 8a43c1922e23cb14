(timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3)
python bench.py --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c2_b.json
python bench.py --workload c3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c3_b.json
