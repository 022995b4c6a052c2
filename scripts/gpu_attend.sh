#!/bin/bash
# attend128 change: parity suite + c3/c2/c4 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x > gpurun_out/att_tests.log 2>&1
tail -2 gpurun_out/att_tests.log
for cfg in c3 c2; do
  timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/att_$cfg.json 2> gpurun_out/att_$cfg.err
done
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/att_c4.json 2> gpurun_out/att_c4.err
CSATTN_ATT_GR=4 timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/att4_c4.json 2> gpurun_out/att4_c4.err
python scripts/summ.py gpurun_out/att_c3.json gpurun_out/att_c2.json gpurun_out/att_c4.json gpurun_out/att4_c4.json
