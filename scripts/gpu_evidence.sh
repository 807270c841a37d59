#!/bin/bash
# evidence pass: ncu launch lists + full captures of every tcgen05 kernel family
mkdir -p gpurun_out
for spec in "sf 1" "sf3hw 1" "kv21 1" "sf 2"; do
  set -- $spec; cfg=$1; it=$2; tag=r1b_${cfg}_t${it}
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_ --csv \
      --log-file gpurun_out/${tag}_launches.csv python bench.py --config $cfg --iters $it --steps 5 --warmup 3 \
      --no-dense --no-cpu > gpurun_out/${tag}_launches_bench.log 2>&1
  n=$((it == 1 ? 2 : 3))
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_ -s $n -c $n \
      -o gpurun_out/${tag} python scripts/profile_run.py $cfg 3 $it > gpurun_out/${tag}_full.log 2>&1
done
echo done
