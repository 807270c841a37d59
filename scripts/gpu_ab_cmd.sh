#!/bin/bash
# usage: gpu_ab_cmd.sh "ENV_A" "ENV_B" "bench args"...  -> gpurun_out/abcmd.txt (interleaved, 2 rounds)
mkdir -p gpurun_out; : > gpurun_out/abcmd.txt
A=$1; B=$2; shift 2
for r in 1 2; do
for args in "$@"; do
  for e in "$A" "$B"; do
    echo "$args [$e] $(env $e timeout 300 python bench.py --steps 20 --warmup 5 $args --no-cpu --no-dense --no-backward 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], [(k["name"], k["ms_avg"]) for k in d["kernels"]])')" >> gpurun_out/abcmd.txt
  done
done; done
