#!/bin/bash
# A/B/... of builds paper_2602_12271_b200/libmonarch_b200_<v>.so, interleaved, 2 rounds
# usage: V="a b c" TESTV=b gpu_ablib.sh cfg...   (TESTV: variant the GPU tests run against first)
mkdir -p gpurun_out; : > gpurun_out/ablib.txt
V=${V:-"a b"}
for tv in ${TESTV:-b}; do
  MBX_LIB=$PWD/paper_2602_12271_b200/libmonarch_b200_$tv.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ablib_pytest_$tv.log 2>&1; echo "exit $?" >> gpurun_out/ablib_pytest_$tv.log
done
for r in 1 2; do
for cfg in "$@"; do
  for v in $V; do
    echo "$cfg $v $(MBX_LIB=$PWD/paper_2602_12271_b200/libmonarch_b200_$v.so timeout 300 python bench.py --steps 20 --warmup 5 --config $cfg --no-cpu --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], [(k["name"], k["ms_avg"]) for k in d["kernels"]])')" >> gpurun_out/ablib.txt
  done
done; done
