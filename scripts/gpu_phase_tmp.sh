CSATTN_PHASE_PROF=1 timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/r02r_phase_c3.json 2> gpurun_out/r02r_phase_c3.err; echo "phase rc=$?"
grep -E "csattn|fin" gpurun_out/r02r_phase_c3.err | tail -4
CSATTN_PHASE_PROF=1 timeout 600 python bench.py --config c2 --no-cpu-baseline --steps 5 > gpurun_out/r02r_phase_c2.json 2> gpurun_out/r02r_phase_c2.err; echo "phase rc=$?"
grep -E "csattn|fin" gpurun_out/r02r_phase_c2.err | tail -4
