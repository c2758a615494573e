#!/bin/bash
# quick GPU iteration: parity tests + per-config timing (+ optional ncu of one kernel)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 1200 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -8 gpurun_out/pytest_gpu.log
fi
timeout 900 python tools/timing.py ${CFGS:-1,2,3,4} > gpurun_out/timing.log 2>&1; echo "timing exit $?"
cat gpurun_out/timing.log
if [ -n "${NCU_MASK:-}" ]; then
  python tools/profile_run.py 4 256 $NCU_MASK 8 > gpurun_out/plain.log 2>&1 || { cat gpurun_out/plain.log; exit 1; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-k_residual_bidir} -c 1 \
    -o gpurun_out/prof_${NCU_TAG:-x} -f python tools/profile_run.py 4 256 $NCU_MASK 8 > gpurun_out/ncu.log 2>&1; echo "ncu exit $?"
fi
