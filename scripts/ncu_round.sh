#!/bin/bash
# Run under gpurun: the round's profile set for config 2 (25 M accesses).
#  1. launch list of one bench step (device time per kernel, --clock-control none)
#  2. --set full captures (with source) of the caching / prefetch forwards and
#     of one priority-replay and one LRU launch
# Numbers printed by runs under ncu are never bench values.
OUT=gpurun_out
mkdir -p $OUT
[ -n "$SKIP_LIST" ] || ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 0 \
    --no-cpu-baseline --no-e2e --no-rows > $OUT/launches_bench.log 2>&1
i=0
for K in "lstm_tc_kernel<.int.0" "lstm_tc_kernel<.int.1" "replay_smem_kernel<.int.0" "replay_smem_kernel<.int.1"; do
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$K" -c 1 \
      -o $OUT/prof_$i python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e \
      --no-rows > $OUT/prof_$i.log 2>&1
  i=$((i+1))
done
ls -la $OUT
