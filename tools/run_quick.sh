python tools/trace_bench.py 3; python tools/trace_bench.py 4
CFGS=1,2,3,4 bash tools/gpu_iter.sh
