#!/bin/bash
# round evidence pass: tests, smoke, bench lines (default + reference arm + torchrun), config sweep,
# ncu launch lists + full captures of every tcgen05 kernel family
mkdir -p gpurun_out/ev
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ev/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/ev/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/ev/smoke.log
timeout 900 python bench.py > gpurun_out/ev/bench_default.json 2> gpurun_out/ev/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev/bench_reference.json 2> gpurun_out/ev/bench_reference.err
timeout 300 python scripts/bwd_profile.py > gpurun_out/ev/bwd_profile.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu > gpurun_out/ev/bench_torchrun1.json 2> gpurun_out/ev/bench_torchrun1.err
# two ranks sharing the box's one GPU (self-launched under torch.distributed.run; gloo barrier / max)
timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --no-backward > gpurun_out/ev/bench_gpus2.json 2> gpurun_out/ev/bench_gpus2.err
timeout 900 python bench.py --gpus 2 --config wan --steps 2 --warmup 3 --no-cpu --no-backward > gpurun_out/ev/bench_wan_gpus2.json 2> gpurun_out/ev/bench_wan_gpus2.err
: > gpurun_out/ev/sweep.jsonl
for a in "--config sf" "--config sf --iters 2" "--config sf --iters 3" "--config sf3hw" \
         "--config kv21" "--config kv21 --iters 2" "--config kv21 --iters 3" "--config kv21_3hw" \
         "--config kv21_3hw --iters 2" "--config kv21_3hw --iters 3" \
         "--config n32k" "--config n32k_3hw" "--config n32k_fhw" "--config n32k_mis" "--config n32k_f" "--config c1" \
         "--config sf720" "--config sf720_3hw" "--config kv21_720_3hw" "--config n75k_720_3hw" "--config wan --steps 2" \
         "--config wan_3hw --steps 2" "--config n32k_w" "--config n32k_hw" "--config n32k_fw" "--config n32k_h" \
         "--config n32k_fhw --iters 2" "--config n32k_mis --iters 2" "--config n32k_3hw --iters 2"; do
  timeout 900 python bench.py --steps 10 --warmup 3 $a --no-cpu --no-backward 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); d['args']='$a'; print(json.dumps(d))" >> gpurun_out/ev/sweep.jsonl
done
# spec: config, refinements, launches per forward (sf3hw T=2 = row, column statistics, alpha_R, row, column)
for spec in "sf 1 2" "sf3hw 1 2" "kv21 1 2" "sf 2 4" "sf3hw 2 5"; do
  set -- $spec; cfg=$1; it=$2; n=$3; tag=${TAG:-r1d}_${cfg}_t${it}
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_ --csv \
      --log-file gpurun_out/ev/${tag}_launches.csv python bench.py --config $cfg --iters $it --steps 5 --warmup 3 \
      --no-dense --no-cpu > gpurun_out/ev/${tag}_launches_bench.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_ -s $n -c $n \
      -o gpurun_out/ev/${tag} python scripts/profile_run.py $cfg 3 $it > gpurun_out/ev/${tag}_full.log 2>&1
done
echo done
