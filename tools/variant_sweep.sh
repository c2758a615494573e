#!/bin/bash
# time every build/variants/*.so (diagnostics): traversal microbenchmark + per-config renders
mkdir -p gpurun_out
for v in ${VARIANTS:-build/variants/*.so}; do
  echo "== $v"
  if [ "${TRACE:-1}" = "1" ]; then
    RR_LIB_VARIANT=$v python tools/trace_bench.py 3; RR_LIB_VARIANT=$v python tools/trace_bench.py 4
  fi
  RR_LIB_VARIANT=$v timeout 600 python tools/timing.py ${CFGS:-3} 2>&1 | grep -v "^\s*$" | grep -v "per launch\|sched"
  if [ "${IDENT:-0}" = "1" ]; then RR_LIB_VARIANT=$v python tools/ident_check.py 2>&1 | grep -E "bad|nonzero" | tail -4; fi
done
