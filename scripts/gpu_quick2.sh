#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q2_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/q2_pytest.log
for a in "--config sf" "--config sf3hw" "--config kv21" "--config kv21_3hw" "--config n32k_3hw"; do
  echo "$a $(timeout 300 python bench.py --steps 10 --warmup 3 $a --no-cpu --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], [(k["name"], k["ms_avg"]) for k in d["kernels"]])')" >> gpurun_out/q2.txt
done
