#!/bin/bash
# quick GPU pass: gpu tests, smoke, SF + KV21 bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/k_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/k_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/k_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/k_smoke.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/k_bench.json 2> gpurun_out/k_bench.err
timeout 600 python bench.py --steps 20 --warmup 3 --config kv21 --no-cpu > gpurun_out/k_bench_kv21.json 2> gpurun_out/k_bench_kv21.err
echo done
