mkdir -p gpurun_out/r2l
rm -f gpurun_out/r2l/*
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_batched_tf32 -s 2 -c 1 -o gpurun_out/r2l/bwd_dl python scripts/bwd_profile.py 1 > gpurun_out/r2l/ncu.log 2>&1
