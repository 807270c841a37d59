#!/bin/bash
# every bench config (dense baselines included), iteration sweep on the rollout shapes
mkdir -p gpurun_out
: > gpurun_out/sweep.jsonl
for a in "--config sf" "--config sf --iters 2" "--config sf --iters 3" "--config sf3hw" \
         "--config kv21" "--config kv21 --iters 2" "--config kv21 --iters 3" "--config kv21_3hw" "--config kv21_3hw --iters 2" \
         "--config n32k" "--config n32k_3hw" "--config n32k_fhw" "--config n32k_mis" "--config c1"; do
  timeout 600 python bench.py --steps 10 --warmup 3 $a --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); d['args']='$a'; print(json.dumps(d))" >> gpurun_out/sweep.jsonl
done
echo done
