#!/bin/bash
# iteration pass: gpu parity tests, bench SF + KV21 (no CPU arm), trace spans
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/i_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/i_pytest.log
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --no-dense > gpurun_out/i_bench.json 2> gpurun_out/i_bench.err
timeout 300 python bench.py --steps 10 --warmup 3 --config kv21 --no-cpu --no-dense > gpurun_out/i_bench_kv21.json 2> gpurun_out/i_bench_kv21.err
NCTA=1 timeout 120 python scripts/trace_tc.py sf > gpurun_out/i_trace_sf.txt 2>&1
NCTA=1 timeout 120 python scripts/trace_tc.py kv21 > gpurun_out/i_trace_kv21.txt 2>&1
echo done
