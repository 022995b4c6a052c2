T=${1:-fz}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'fused_step' -s 3 -c 1 \
  -o gpurun_out/${T}_fused python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
