#!/bin/bash
# backward A/B of library variants: V="a b" -> gpurun_out/bwd_ab.txt (+ backward GPU tests on the last variant)
mkdir -p gpurun_out; : > gpurun_out/bwd_ab.txt
for v in $V; do
  MBX_LIB=$PWD/paper_2602_12271_b200/libmonarch_b200_$v.so timeout 600 python -m pytest tests/test_backward_gpu.py -x -q > gpurun_out/bwd_pytest_$v.log 2>&1; echo "exit $?" >> gpurun_out/bwd_pytest_$v.log
done
for r in 1 2; do for v in $V; do
  echo "$v $(MBX_LIB=$PWD/paper_2602_12271_b200/libmonarch_b200_$v.so timeout 300 python bench.py --steps 5 --warmup 3 --config ${CFG:-sf} --no-cpu --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); b=d["backward"]; print(b["ms"], b["kernels_ms"])')" >> gpurun_out/bwd_ab.txt
done; done
