#!/bin/bash
# suites + c3/c2 bench + c3 ncu (full capture of the 4 step kernels, launch list)
bash scripts/gpu_select.sh
bash scripts/gpu_ncu_c3.sh
python scripts/ncu_summary.py gpurun_out/prof_c3.ncu-rep > gpurun_out/ncu_c3_summary.txt 2>&1
tail -5 gpurun_out/ncu_c3_summary.txt
