mkdir -p gpurun_out/r2q
rm -f gpurun_out/r2q/*
for r in 1; do
for v in ""; do
  if [ -n "$v" ]; then export MBX_LIB=paper_2602_12271_b200/libmonarch_b200_$v.so; else unset MBX_LIB; fi
  echo "== variant ${v:-default} round $r" >> gpurun_out/r2q/ab.txt
  timeout 300 python scripts/bwd_profile.py 2>&1 | tail -1 >> gpurun_out/r2q/ab.txt
done
done
