(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3)
python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c4_b.json
cp profiles/block_steps.json gpurun_out/block_steps.json
