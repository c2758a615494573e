#!/bin/bash
# GPU-box diagnostics: parity tests, per-config timing, one ncu --set full capture of the top kernel.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python tools/timing.py 1,2,3,4 > gpurun_out/timing.log 2>&1; echo "timing exit $?"
cat gpurun_out/timing.log
if [ "$1" != "noncu" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_residual_bidir -c 1 \
  -o gpurun_out/prof_t6_c4 -f python tools/profile_run.py 4 256 0x60 8 > gpurun_out/ncu_t6.log 2>&1; echo "ncu exit $?"
tail -3 gpurun_out/ncu_t6.log
fi
