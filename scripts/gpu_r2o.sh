mkdir -p gpurun_out/r2o
rm -f gpurun_out/r2o/*
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_backward_gpu.py -q -x -k "bf16_matches" > gpurun_out/r2o/memcheck.log 2>&1; echo "exit $?" >> gpurun_out/r2o/memcheck.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_backward_gpu.py -q -x -k "bf16_matches and (nb_tiled or raw)" > gpurun_out/r2o/racecheck.log 2>&1; echo "exit $?" >> gpurun_out/r2o/racecheck.log
