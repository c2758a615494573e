#!/bin/bash
# A/B of the BVH leaf size (RR_LEAF_MAX at scene upload): per-config render timings for each value
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for L in ${LEAVES:-1 2 4 8}; do
  echo "== RR_LEAF_MAX=$L"
  RR_LEAF_MAX=$L timeout 900 python tools/timing.py ${CFGS:-3,4} 2>&1 | tee gpurun_out/timing_leaf$L.log
done
