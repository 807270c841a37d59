#!/bin/bash
mkdir -p gpurun_out
for c in sf3hw kv21_3hw; do timeout 120 python scripts/trace_tc.py $c > gpurun_out/trace_pair_$c.txt 2>&1; done
