#!/bin/bash
# A/B timing of K1 on the bench shapes across builds of libflz: scripts/ab_k1.sh "c3 c4" libflz.so libflz_a.so ...
# (every build is run twice, interleaved, so that clock / thermal drift shows)
shapes="$1"; shift
for rep in 1 2; do
  for lib in "$@"; do
    for s in $shapes; do
      FLZ_LIB=$PWD/paper_2409_15053_b200/$lib python scripts/k1_one.py $s 8 2>&1 | tail -1
    done
  done
done
