# round 2, GPU call A: box facts, full GPU suite (incl. the scale parity tests),
# default bench (c3) + reference arm, sanitizers on a small workload
set -x
nproc; free -g | head -2; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r02a_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r02a_gpu_tests.log
timeout 900 python bench.py > gpurun_out/r02a_bench_c3.json 2> gpurun_out/r02a_bench_c3.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02a_bench_c3.json
timeout 900 python bench.py --impl reference > gpurun_out/r02a_ref_c3.json 2> gpurun_out/r02a_ref_c3.err; echo "ref rc=$?"
tail -c 1500 gpurun_out/r02a_ref_c3.json
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --log-file gpurun_out/r02a_sanitize_$t.log python scripts/sanitize_workload.py > gpurun_out/r02a_sanitize_$t.out 2>&1; echo "$t rc=$?"
  tail -3 gpurun_out/r02a_sanitize_$t.log
done
