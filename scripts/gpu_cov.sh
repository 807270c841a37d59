#!/bin/bash
# coverage timing: configs that fall back to the SIMT path
for a in "--config kv21 --iters 2" "--config kv21 --iters 3" "--config sf --iters 2" "--config sf3hw" "--config n32k" "--config c1"; do
  echo "$a $(timeout 300 python bench.py --steps 3 --warmup 3 $a --no-cpu --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("path"), [(k["name"], k["ms_avg"]) for k in d["kernels"]])')" >> gpurun_out/cov.txt
done
