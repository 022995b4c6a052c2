#!/bin/bash
# attend128 change: parity suite + c3/c2 bench, GR=4 and GR=8
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x > gpurun_out/att_tests.log 2>&1
tail -2 gpurun_out/att_tests.log
for cfg in c3 c2; do
  timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/att_$cfg.json 2> gpurun_out/att_$cfg.err
  CSATTN_ATT_GR8=1 timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/att8_$cfg.json 2> gpurun_out/att8_$cfg.err
done
python scripts/summ.py gpurun_out/att_c3.json gpurun_out/att8_c3.json gpurun_out/att_c2.json gpurun_out/att8_c2.json
