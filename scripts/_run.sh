(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3)
timeout 300 python scripts/k1_bench.py all 2>&1 | sed -n '4,5p;8p'
timeout 300 python scripts/k1_bench.py stencil 2>&1 | tail -2
