#!/bin/bash
mkdir -p gpurun_out
for sp in 1 2 3 4 6; do
  CSATTN_FORCE_SPLIT=$sp timeout 600 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/split_$sp.json 2> gpurun_out/split_$sp.err
done
python scripts/summ.py gpurun_out/split_1.json gpurun_out/split_2.json gpurun_out/split_3.json gpurun_out/split_4.json gpurun_out/split_6.json
