#!/bin/bash
# time every build/variants/*.so on the given configs (diagnostics); IDENT=1 also runs tools/ident_check.py
mkdir -p gpurun_out
for v in ${VARIANTS:-build/variants/*.so}; do
  echo "== $v"
  RR_LIB_VARIANT=$v timeout 600 python tools/timing.py ${CFGS:-3} 2>&1 | grep -v "^\s*$" | grep -v "per launch"
  if [ "${IDENT:-0}" = "1" ]; then RR_LIB_VARIANT=$v python tools/ident_check.py 2>&1 | grep -E "bad|nonzero" | tail -4; fi
done
