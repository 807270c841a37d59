#!/bin/bash
for cfg in sf kv21; do
for v in "MBX_WIDE=0" "MBX_WIDE=1"; do
  echo "$cfg $v $(env $v timeout 300 python bench.py --steps 20 --warmup 5 --config $cfg --no-cpu --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], [(k["name"], k["ms_avg"]) for k in d["kernels"]])')" >> gpurun_out/w2.txt
done; done
MBX_WIDE=1 timeout 300 python -m pytest tests -m gpu -x -q -k "tensor_core_path and 1-12-1 or self_forcing" > gpurun_out/w2_pytest.log 2>&1; echo "exit $?" >> gpurun_out/w2_pytest.log
