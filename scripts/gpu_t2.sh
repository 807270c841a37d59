#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q -k "tensor_core_path or self_forcing or chunked_kv or deterministic" > gpurun_out/t2_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/t2_pytest.log
for a in "--config kv21 --iters 2" "--config kv21 --iters 3" "--config sf --iters 2" "--config sf --iters 3" "--config sf"; do
  echo "$a $(timeout 300 python bench.py --steps 10 --warmup 3 $a --no-cpu --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("path"), [(k["name"], k["ms_avg"], k["launches_per_step"]) for k in d["kernels"]])')" >> gpurun_out/t2.txt
done
