mkdir -p gpurun_out/r2k
rm -f gpurun_out/r2k/*
timeout 600 python -m pytest tests/test_backward_gpu.py tests/test_custom_op_gpu.py -q -x > gpurun_out/r2k/pytest_bwd.log 2>&1; echo "exit $?" >> gpurun_out/r2k/pytest_bwd.log
timeout 300 python scripts/bwd_profile.py > gpurun_out/r2k/bwd_profile_hybrid.txt 2>&1
MBX_BWD_CUBLAS=none timeout 300 python scripts/bwd_profile.py > gpurun_out/r2k/bwd_profile_mma.txt 2>&1
