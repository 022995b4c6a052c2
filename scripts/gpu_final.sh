# round-end evidence: GPU suites, facade, smoke, benches c2/c3 (+ cpu baseline), ncu c3
bash scripts/gpu_round.sh
CSATTN_UNION=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 600 -x -k union > gpurun_out/gpu_tests_union.log 2>&1
tail -1 gpurun_out/gpu_tests_union.log
bash scripts/gpu_ncu_c3.sh
python scripts/ncu_summary.py gpurun_out/prof_c3.ncu-rep > gpurun_out/ncu_c3_summary.txt 2>&1
