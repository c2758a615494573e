#!/bin/bash
# traversal microbenchmark (random and coherent camera rays) + one ncu capture of k_trace (diagnostics)
mkdir -p gpurun_out
python tools/trace_bench.py 3; python tools/trace_bench.py 4
COHERENT=1 python tools/trace_bench.py 3; COHERENT=1 python tools/trace_bench.py 4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_trace -c 1 \
    -o gpurun_out/prof_trace -f python tools/trace_bench.py 3 1048576 > gpurun_out/ncu.log 2>&1; echo "ncu exit $?"
