#!/bin/bash
# GPU box: build, then pytest -m gpu (optionally a -k filter in $K), log under gpurun_out/
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt 2>&1
timeout ${TMO:-1500} python -m pytest tests -m gpu -q ${K:+-k "$K"} --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -30 gpurun_out/pytest_gpu.log
