#!/bin/bash
# parity tests, then fused/two-launch timing with a row-CTA sweep (SF and KV21), traces
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/s_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/s_pytest.log
for cfg in sf kv21; do
  for v in "MBX_FUSED=0" "MBX_ROW_CTAS=64" "MBX_ROW_CTAS=74" "MBX_ROW_CTAS=81" "MBX_ROW_CTAS=90" "MBX_ROW_CTAS=100"; do
    echo "$cfg $v $(env $v timeout 300 python bench.py --steps 20 --warmup 5 --config $cfg --no-cpu --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], [(k["name"], k["ms_avg"]) for k in d["kernels"]])')" >> gpurun_out/s_sweep.txt
  done
done
NCTA=1 timeout 120 python scripts/trace_tc.py sf > gpurun_out/s_trace_sf.txt 2>&1
NCTA=1 timeout 120 python scripts/trace_tc.py kv21 > gpurun_out/s_trace_kv21.txt 2>&1
echo done
