#!/bin/bash
# A/B of MBX_DBG variants, interleaved, 3 rounds: usage gpu_ab.sh "cfgargs" dbgA dbgB ...
cfg=$1; shift
: > gpurun_out/ab.txt
for r in 1 2 3; do
  for d in "$@"; do
    echo "$cfg dbg=$d $(MBX_DBG=$d timeout 300 python bench.py --steps 30 --warmup 5 $cfg --no-cpu --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], [(k["name"], k["ms_avg"]) for k in d["kernels"]])')" >> gpurun_out/ab.txt
  done
done
