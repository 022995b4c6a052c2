#!/bin/bash
mkdir -p gpurun_out
for g in 4 48 8; do
  CSATTN_ATT_GR=$g timeout 600 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/occ_$g.json 2> gpurun_out/occ_$g.err
done
CSATTN_ATT_GR=48 timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/occ_c4_48.json 2> gpurun_out/occ_c4_48.err
python scripts/summ.py gpurun_out/occ_4.json gpurun_out/occ_48.json gpurun_out/occ_8.json gpurun_out/occ_c4_48.json
