#!/bin/bash
mkdir -p gpurun_out
for sk in 0.7 0.8 0.9 0.95; do
  CSATTN_SPEC_KEEP=$sk timeout 600 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/spec_$sk.json 2> gpurun_out/spec_$sk.err
  CSATTN_SPEC_KEEP=$sk timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/spec_c2_$sk.json 2> gpurun_out/spec_c2_$sk.err
  CSATTN_SPEC_KEEP=$sk CSATTN_PHASE_PROF=1 timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/specp_$sk.err
done
for sk in 0.7 0.8 0.9 0.95; do python scripts/summ.py gpurun_out/spec_$sk.json gpurun_out/spec_c2_$sk.json; grep "retried\|logged" gpurun_out/specp_$sk.err; done
