#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q -k "wide or tensor_core_path" > gpurun_out/w_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/w_pytest.log
for a in "--config sf3hw" "--config sf"; do
  echo "$a $(timeout 300 python bench.py --steps 10 --warmup 3 $a --no-cpu 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d.get("dense_fa_best_ms"), d["config"].get("path"), [(k["name"], k["ms_avg"], k["launches_per_step"]) for k in d["kernels"]])')" >> gpurun_out/w.txt
done
