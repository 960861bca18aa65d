#!/bin/bash
# A/B timing of two in-tree builds of the ABI (diagnostic): runs the given
# command alternately with RECMG_LIB=librecmg_a.so and librecmg.so.
#   bash scripts/ab.sh 2 "python scripts/tc_phases.py 4000000" "caching:|prefetch:"
REPS=${1:-2}; CMD=${2}; PAT=${3:-.}
for i in $(seq $REPS); do
  for L in librecmg_a.so librecmg.so; do
    echo "== $L"; RECMG_LIB=$L $CMD 2>&1 | grep -E "$PAT"
  done
done
