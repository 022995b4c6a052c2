# ncu --set full of the tc build kernels (probe, tc mode only): $1 = tag
T=${1:-nb}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'build_tc_(lists|theta)_kernel|build_tc_kernel' -c 3 \
  -o gpurun_out/${T}_build python scripts/build_tc_probe.py tc > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/${T}_ncu.log
