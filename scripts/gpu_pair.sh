#!/bin/bash
# A/B of the paired-rows row stage (MBX_PAIR=1, default) against the 128-row row stage (MBX_PAIR=0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pair_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/pair_pytest.log
for cfg in sf kv21 sf3hw kv21_3hw n32k_3hw n32k_mis; do
  for it in 1 2; do
    for p in 0 1; do
      echo "$cfg iters=$it pair=$p $(MBX_PAIR=$p timeout 300 python bench.py --steps 10 --warmup 3 --config $cfg --iters $it --no-cpu --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], [(k["name"], k["ms_avg"]) for k in d["kernels"]])')" >> gpurun_out/pair.txt
    done
  done
done
