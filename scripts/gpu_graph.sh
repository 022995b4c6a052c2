#!/bin/bash
# decode-run CUDA graph: parity tests + bench lines (c3, c2)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_graph.py -x -q > gpurun_out/graph_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/graph_tests.log
CSATTN_HOST_PROF=1 timeout 600 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/graph_c3.json 2> gpurun_out/graph_c3.err
CSATTN_HOST_PROF=1 timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/graph_c2.json 2> gpurun_out/graph_c2.err
tail -3 gpurun_out/graph_tests.log
