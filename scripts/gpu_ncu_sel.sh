# ncu --set full of select_kernel at c3: $1 = tag
T=${1:-sel}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'select_kernel' -s 4 -c 1 \
  -o gpurun_out/${T}_sel python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
