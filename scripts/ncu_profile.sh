#!/bin/bash
# Run under gpurun: launch list (every kernel of one bench step, device time)
# and a full ncu capture of the named kernels.  Numbers printed by a run
# under ncu are never bench values.
set -x
OUT=gpurun_out
mkdir -p $OUT
N=${N:-2000000}
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python bench.py --accesses $N --steps 1 --warmup 0 \
    --no-cpu-baseline --no-e2e > $OUT/launches_bench.log 2>&1
for K in ${KERNELS:-lstm_fwd replay_narrow_kernel}; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-0} -c ${COUNT:-1} \
      -o $OUT/prof_$K python bench.py --accesses $N --steps 1 --warmup 0 --no-cpu-baseline \
      --no-e2e > $OUT/prof_$K.log 2>&1
done
ls -la $OUT
