#!/bin/bash
# DRAM bytes / L2 hit rate of each tcgen05 kernel with caches NOT flushed by ncu (single-pass metrics):
# shows how much of the row stage's workspace the column stage still finds in L2.
mkdir -p gpurun_out
for cfg in "$@"; do
timeout 600 ncu --cache-control none --clock-control none -k regex:tc_ \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct,lts__t_sector_op_write_hit_rate.pct \
  --csv python scripts/profile_run.py $cfg 4 > gpurun_out/warm_$cfg.csv 2>gpurun_out/warm_$cfg.log
done
