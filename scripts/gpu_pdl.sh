#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/p_pytest.log
for cfg in "--config sf" "--config kv21" "--config sf --iters 3" "--config sf3hw"; do
for v in "MBX_PDL=0" "MBX_PDL=1"; do
  echo "$cfg $v $(env $v timeout 300 python bench.py --steps 30 --warmup 5 $cfg --no-cpu --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], [(k["name"], k["ms_avg"]) for k in d["kernels"]])')" >> gpurun_out/p.txt
done; done
