#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "tensor_core" > gpurun_out/b_tc.log 2>&1; echo "exit $?" >> gpurun_out/b_tc.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/b_pytest.log 2>&1; echo "exit $?" >> gpurun_out/b_pytest.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err
timeout 300 python bench.py --steps 10 --warmup 3 --config kv21 --no-cpu --no-dense > gpurun_out/b_bench_kv21.json 2> gpurun_out/b_bench_kv21.err
echo done
