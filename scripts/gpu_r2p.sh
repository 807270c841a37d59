mkdir -p gpurun_out/r2p
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2p/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2p/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2p/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r2p/smoke.log
timeout 900 python bench.py > gpurun_out/r2p/bench_default.json 2> gpurun_out/r2p/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2p/bench_reference.json 2> gpurun_out/r2p/bench_reference.err
timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --no-backward > gpurun_out/r2p/bench_gpus2.json 2> gpurun_out/r2p/bench_gpus2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2p/bwd_launches.csv python scripts/bwd_profile.py 1 > gpurun_out/r2p/bwd_launches.log 2>&1
