#!/bin/bash
# quick: gpu parity tests + SF/KV21 timing (two-launch) + trace
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/q_pytest.log
for cfg in sf kv21; do
  echo "$cfg $(timeout 300 python bench.py --steps 20 --warmup 5 --config $cfg --no-cpu --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], [(k["name"], k["ms_avg"]) for k in d["kernels"]])')" >> gpurun_out/q_sweep.txt
done
NCTA=1 timeout 120 python scripts/trace_tc.py sf > gpurun_out/q_trace_sf.txt 2>&1
echo done
