mkdir -p gpurun_out; : > gpurun_out/qab_l2.txt
for r in 1 2 3; do
for args in "--config sf" "--config sf3hw" "--config kv21"; do
  for e in MBX_L2HINT=3 MBX_L2HINT=2 MBX_L2HINT=1 MBX_L2HINT=0; do
    echo "$args [$e] $(env $e timeout 300 python bench.py --steps 50 --warmup 5 $args --no-cpu --no-dense --no-backward 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], [(k["name"], k["ms_avg"]) for k in d["kernels"]])')" >> gpurun_out/qab_l2.txt
  done
done; done
