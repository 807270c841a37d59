#!/bin/bash
# usage: gpu_ab_env.sh "ENV_A" "ENV_B" cfg...  -> gpurun_out/abenv.txt (interleaved, 2 rounds)
mkdir -p gpurun_out
A=$1; B=$2; shift 2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/abenv_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/abenv_pytest.log
for r in 1 2; do
for cfg in "$@"; do
  for e in "$A" "$B"; do
    echo "$cfg [$e] $(env $e timeout 300 python bench.py --steps 20 --warmup 5 --config $cfg --no-cpu --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], [(k["name"], k["ms_avg"]) for k in d["kernels"]])')" >> gpurun_out/abenv.txt
  done
done
done
