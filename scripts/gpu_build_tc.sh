# tcgen05 table build: tests, probe timing, launch list
T=${1:-bt}
timeout 900 python -m pytest tests/test_gpu_build_tc.py tests/test_gpu_parity.py tests/test_gpu_hardening.py -x -q > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/${T}_tests.log
timeout 300 python scripts/build_tc_probe.py > gpurun_out/${T}_probe.log 2>&1; echo "probe rc=$?"
cat gpurun_out/${T}_probe.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python scripts/build_tc_probe.py tc fp64 > /dev/null 2>&1; echo "ncu rc=$?"
grep -E "build|refill" gpurun_out/${T}_launches.csv | awk -F'","' '{print $5, $NF}' | head -30
