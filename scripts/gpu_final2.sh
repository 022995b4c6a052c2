# round evidence: all suites, facade, smoke, benches c2/c3/c4/c5/c2o, reference arm, ncu c3
FULL=1 bash scripts/gpu_round.sh
timeout 300 python bench.py --config c2o --steps 10 --warmup 3 > gpurun_out/bench_c2o.json 2> gpurun_out/bench_c2o.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_c3.json 2> gpurun_out/bench_ref_c3.err
tail -c 600 gpurun_out/bench_ref_c3.json
bash scripts/gpu_ncu_c3.sh
python scripts/ncu_summary.py gpurun_out/prof_c3.ncu-rep > gpurun_out/ncu_c3_summary.txt 2>&1
