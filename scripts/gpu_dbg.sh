#!/bin/bash
for d in 0 1024 558; do
  echo "dbg $d $(MBX_DBG=$d timeout 300 python bench.py --steps 20 --warmup 5 --config sf --no-cpu --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print([(k["name"], k["ms_avg"]) for k in d["kernels"]])')" >> gpurun_out/dbg.txt
done
NCTA=1 timeout 120 python scripts/trace_tc.py sf > gpurun_out/t0.txt 2>&1
