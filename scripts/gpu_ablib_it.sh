#!/bin/bash
# A/B of two builds at a refinement count: usage gpu_ablib_it.sh iters cfg...
mkdir -p gpurun_out; : > gpurun_out/ablib.txt
it=$1; shift
MBX_LIB=$PWD/paper_2602_12271_b200/libmonarch_b200_b.so timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/ablib_pytest_b.log 2>&1; echo "exit $?" >> gpurun_out/ablib_pytest_b.log
for r in 1 2; do
for cfg in "$@"; do
  for v in a b; do
    echo "$cfg T=$it $v $(MBX_LIB=$PWD/paper_2602_12271_b200/libmonarch_b200_$v.so timeout 300 python bench.py --steps 20 --warmup 5 --config $cfg --iters $it --no-cpu --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], [(k["name"], k["ms_avg"]) for k in d["kernels"]])')" >> gpurun_out/ablib.txt
  done
done; done
