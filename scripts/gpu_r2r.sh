mkdir -p gpurun_out/r2r
rm -f gpurun_out/r2r/*
timeout 600 python -m pytest tests/test_backward_gpu.py tests/test_custom_op_gpu.py -q -x > gpurun_out/r2r/pytest_bwd.log 2>&1; echo "exit $?" >> gpurun_out/r2r/pytest_bwd.log
timeout 300 python scripts/bwd_profile.py > gpurun_out/r2r/bwd_profile.txt 2>&1
