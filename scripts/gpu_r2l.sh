mkdir -p gpurun_out/r2l
rm -f gpurun_out/r2l/*
timeout 600 ncu --section SpeedOfLight --section Occupancy --section LaunchStats --section MemoryWorkloadAnalysis --clock-control none -k regex:gemm_batched_tf32 -s 13 -c 13 -o gpurun_out/r2l/bwd_mma2 python scripts/bwd_profile.py > gpurun_out/r2l/ncu.log 2>&1
