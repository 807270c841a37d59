#!/bin/bash
# usage: gpu_ab_envs.sh cfg "ENV1" "ENV2" ...  -> gpurun_out/abenvs.txt (2 interleaved rounds) + gpu tests
mkdir -p gpurun_out; : > gpurun_out/abenvs.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/abenvs_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/abenvs_pytest.log
cfg=$1; shift
for r in 1 2; do
  for e in "$@"; do
    echo "$cfg [$e] $(env $e timeout 300 python bench.py --steps 20 --warmup 5 --config $cfg --no-cpu --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], [(k["name"], k["ms_avg"]) for k in d["kernels"]])')" >> gpurun_out/abenvs.txt
  done
done
