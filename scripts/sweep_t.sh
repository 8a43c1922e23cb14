#!/bin/bash
# K1 on long ragged rows: entries-per-warp target (task granularity) x programmatic dependent launch
cd "$(dirname "$0")/.."
for pdl in 1 0; do
  for T in auto 16 24 32 48; do
    echo "=== PDL=$pdl T=$T"
    if [ $T = auto ]; then FLZ_K1_PDL=$pdl python scripts/k1_bench.py parsec 2>&1 | grep "us/step"
    else FLZ_K1_PDL=$pdl FLZ_K1_T=$T python scripts/k1_bench.py parsec 2>&1 | grep "us/step"; fi
  done
  echo "=== PDL=$pdl lap"; FLZ_K1_PDL=$pdl python scripts/k1_bench.py lap 2>&1 | grep "us/step"
done
