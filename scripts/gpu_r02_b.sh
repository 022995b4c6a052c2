# round 2, GPU call B: ncu --set full (with source) of select_kernel and attend128 at c3
set -x
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'select_kernel|attend128' -s 8 -c 2 \
  -o gpurun_out/r02b_c3 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02b_ncu.log 2>&1
echo "ncu rc=$?"
tail -5 gpurun_out/r02b_ncu.log
