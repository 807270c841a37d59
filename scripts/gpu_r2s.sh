mkdir -p gpurun_out/r2s
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2s/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r2s/smoke.log
timeout 900 python bench.py > gpurun_out/r2s/bench_default.json 2> gpurun_out/r2s/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2s/bench_reference.json 2> gpurun_out/r2s/bench_reference.err
