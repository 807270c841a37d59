#!/bin/bash
# usage: OUT=file gpu_sweep_list.sh "args" ... -> gpurun_out/$OUT (one bench JSON line per args)
mkdir -p gpurun_out; OUT=${OUT:-sweep.jsonl}; : > gpurun_out/$OUT
for a in "$@"; do
  timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 $a --no-cpu --no-backward 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); d['args']='$a'; print(json.dumps(d))" >> gpurun_out/$OUT
done
