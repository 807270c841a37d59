#!/bin/bash
# first GPU pass: parity tests, smoke, bench, L2 microbench, launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/a_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/a_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/a_smoke.log
timeout 120 python scripts/l2_bw.py > gpurun_out/a_l2.json 2>&1
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err
timeout 300 python bench.py --steps 10 --warmup 3 --config kv21 --no-cpu > gpurun_out/a_bench_kv21.json 2> gpurun_out/a_bench_kv21.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/a_launches.csv python bench.py --steps 3 --warmup 3 --no-dense --no-cpu > /dev/null 2>&1
echo done
