#!/bin/bash
# Sweep of the TMA-staged stencil kernel (run under gpurun): tile rows x producer warps x CTAs
# per SM x ring depth on the 100^3 Laplacian, 3 columns and 1 column (us per Clenshaw step).
# FLZ_ST_TILE=0 is the one-warp-per-slice kernel.  Results of round 1 are in DESIGN.md §4.
cd "$(dirname "$0")/.."
echo "--- warp kernel"; FLZ_ST_TILE=0 python scripts/k1_bench.py lap 2>&1 | tail -2 | grep -o "[0-9.]* us/step" | paste - -
for T in 128 256 512; do for P in 2 4 8; do for C in 1 2 3; do for ST in 2 3 4; do
  echo "--- T=$T prod=$P ctas=$C stages=$ST"
  FLZ_ST_TILE=$T FLZ_ST_STAGES=$ST FLZ_ST_CTAS=$C FLZ_ST_PRODUCERS=$P timeout 200 python scripts/k1_bench.py lap 2>&1 |
    tail -2 | grep -o "[0-9.]* us/step\|Error.*\|error.*" | paste - -
done; done; done; done
