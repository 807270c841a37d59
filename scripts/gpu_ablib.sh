#!/bin/bash
# A/B of two builds (paper_2602_12271_b200/libmonarch_b200_{a,b}.so), interleaved, 3 rounds
: > gpurun_out/ablib.txt
for cfg in "--config sf" "--config kv21"; do
for r in 1 2 3; do
  for v in a b; do
    echo "$cfg $v $(MBX_LIB=$PWD/paper_2602_12271_b200/libmonarch_b200_$v.so timeout 300 python bench.py --steps 30 --warmup 5 $cfg --no-cpu --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], [(k["name"], k["ms_avg"]) for k in d["kernels"]])')" >> gpurun_out/ablib.txt
  done
done; done
MBX_LIB=$PWD/paper_2602_12271_b200/libmonarch_b200_b.so timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/ablib_pytest_b.log 2>&1; echo "exit $?" >> gpurun_out/ablib_pytest_b.log
