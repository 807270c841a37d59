mkdir -p gpurun_out; : > gpurun_out/ab.txt
for r in 1 2; do for v in base noexp; do for dbg in 0 1 9; do
echo "$v dbg=$dbg $(MBX_DBG=$dbg MBX_LIB=$PWD/paper_2602_12271_b200/libmonarch_b200_$v.so timeout 300 python bench.py --steps 20 --warmup 5 --config sf --no-cpu --no-dense --no-backward 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], [(k["name"], k["ms_avg"]) for k in d["kernels"]])')" >> gpurun_out/ab.txt
done; done; done
