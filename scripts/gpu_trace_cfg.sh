#!/bin/bash
# usage: gpu_trace_cfg.sh cfg...   (timelines of the traced build into gpurun_out/trace_<cfg>.txt)
mkdir -p gpurun_out
for c in "$@"; do timeout 120 python scripts/trace_tc.py $c > gpurun_out/trace_$c.txt 2>&1; done
