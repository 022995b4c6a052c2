# round-end evidence: full GPU suite, smoke, benches (c3 default with CPU baseline + parity, c2, c4, c5), launch list
T=${1:-fin}
timeout 2000 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/${T}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${T}_smoke.log
timeout 1200 python bench.py > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err; echo "c3 rc=$?"; python scripts/summ.py gpurun_out/${T}_bench_c3.json
timeout 600 python bench.py --config c2 > gpurun_out/${T}_bench_c2.json 2> /dev/null; echo "c2 rc=$?"; python scripts/summ.py gpurun_out/${T}_bench_c2.json
timeout 1500 python bench.py --config c4 --no-cpu-baseline > gpurun_out/${T}_bench_c4.json 2> /dev/null; echo "c4 rc=$?"; python scripts/summ.py gpurun_out/${T}_bench_c4.json
timeout 1500 python bench.py --config c5 --no-cpu-baseline > gpurun_out/${T}_bench_c5.json 2> /dev/null; echo "c5 rc=$?"; python scripts/summ.py gpurun_out/${T}_bench_c5.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
