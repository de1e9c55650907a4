#!/bin/bash
# A/B two library builds on the same box: ab/<name>.so files are swapped in
# for paper_2502_03000_b200/_lib/liblm_b200.so in turn, ROUNDS times.
#   CMD='python bench.py --config 3c --steps 10 --warmup 3 --no-cpu --no-e2e' bash tools/ab.sh a b
set -u
LIB=paper_2502_03000_b200/_lib/liblm_b200.so
ROUNDS=${ROUNDS:-2}
for r in $(seq $ROUNDS); do
  for v in "$@"; do
    cp ab/$v.so $LIB
    echo "== $v (round $r)"
    eval "$CMD"
  done
done
