#!/bin/bash
# full evidence pass: gpu tests, smoke, bench (default + kv21 + reference arm), ncu launch list + full capture
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/c_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/c_smoke.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err
timeout 600 python bench.py --steps 20 --warmup 3 --config kv21 --no-cpu > gpurun_out/c_bench_kv21.json 2> gpurun_out/c_bench_kv21.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/c_bench_ref.json 2> gpurun_out/c_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_ --csv --log-file gpurun_out/c_launches.csv python bench.py --steps 5 --warmup 3 --no-dense --no-cpu > gpurun_out/c_launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_ -s 2 -c 2 -o gpurun_out/c_prof_sf python scripts/profile_run.py sf 3 > gpurun_out/c_prof.log 2>&1
echo done
