#!/bin/bash
# A/B/C... timing of in-tree library variants (diagnostic):
#   bash scripts/abn.sh 2 "python scripts/fwd_time.py 8000000 5" "median" librecmg_a.so librecmg.so ...
REPS=$1; CMD=$2; PAT=$3; shift 3
for i in $(seq $REPS); do
  for L in "$@"; do
    echo "== $L"; RECMG_LIB=$L $CMD 2>&1 | grep -E "$PAT"
  done
done
