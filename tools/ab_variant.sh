#!/bin/bash
# A/B of the default library against tuning variants (tools/variants.py): per-config render timings for each
# VARIANTS="name ..." (build/variants/<name>.so); optionally the GPU tests on the default build (TESTS=1)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for rep in 1 2; do
for v in default ${VARIANTS:-}; do
  echo "== $v (rep $rep)"
  if [ "$v" = default ]; then lib=""; else lib=build/variants/$v.so; fi
  RR_LIB_VARIANT=$lib timeout 900 python tools/timing.py ${CFGS:-3,4} 2>&1 | tee gpurun_out/timing_$v.$rep.log
done
done
if [ "${TESTS:-0}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x ${K:+-k "$K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
  tail -5 gpurun_out/pytest_gpu.log
fi
