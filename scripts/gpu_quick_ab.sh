#!/bin/bash
# usage: gpu_quick_ab.sh "ENV ..." "bench args" ... : one bench line per (env, args), 2 rounds, into gpurun_out/qab.txt
mkdir -p gpurun_out; : > gpurun_out/qab.txt
ENVS=$1; shift
for r in 1 2; do
for args in "$@"; do
  IFS='|' read -ra EL <<< "$ENVS"
  for e in "${EL[@]}"; do
    echo "$args [$e] $(env $e timeout 300 python bench.py --steps 20 --warmup 5 $args --no-cpu --no-dense --no-backward 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], [(k["name"], k["ms_avg"]) for k in d["kernels"]])')" >> gpurun_out/qab.txt
  done
done; done
