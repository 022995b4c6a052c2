# select-kernel phase breakdown (diagnostic; numbers under CSATTN_PHASE_PROF are not bench values)
export CSATTN_PHASE_PROF=1
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/phase_c2.json 2> gpurun_out/phase_c2.err
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/phase_c3.json 2> gpurun_out/phase_c3.err
grep csattn gpurun_out/phase_c2.err gpurun_out/phase_c3.err
