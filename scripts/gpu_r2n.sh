mkdir -p gpurun_out/r2n
rm -f gpurun_out/r2n/*
timeout 600 python -m pytest tests/test_backward_gpu.py -q -x > gpurun_out/r2n/pytest_bwd.log 2>&1; echo "exit $?" >> gpurun_out/r2n/pytest_bwd.log
for v in ""; do
  if [ -n "$v" ]; then export MBX_LIB=paper_2602_12271_b200/libmonarch_b200_$v.so; else unset MBX_LIB; fi
  echo "== variant ${v:-default}" >> gpurun_out/r2n/ab.txt
  timeout 300 python scripts/bwd_profile.py >> gpurun_out/r2n/ab.txt 2>&1
  MBX_BWD_CUBLAS=none timeout 300 python scripts/bwd_profile.py 2>&1 | tail -1 >> gpurun_out/r2n/ab.txt
done
