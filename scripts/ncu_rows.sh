#!/bin/bash
# Run under gpurun: ncu evidence for K5 (rows_refresh_kernel) and K6
# (embedding_bag_kernel) in the config-4 DLRM batch loop: PCIe read bytes
# (zero-copy host rows), DRAM bytes and duration per launch for a series of
# batches, plus one --set full capture of each.  Never a bench value.
OUT=gpurun_out
mkdir -p $OUT
M=gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum
ncu --metrics $M --clock-control none --csv -k "regex:rows_refresh|embedding_bag" -c 40 \
    --log-file $OUT/rows_metrics.csv python bench.py --config 4 --steps 1 --warmup 1 \
    > $OUT/rows_metrics_bench.log 2>&1
for K in rows_refresh embedding_bag; do
  ncu --set full --clock-control none --import-source on -k "regex:$K" -s 20 -c 1 \
      -o $OUT/prof_$K python bench.py --config 4 --steps 1 --warmup 1 > $OUT/prof_$K.log 2>&1
done
ls -la $OUT
