TRACE=1 CFGS=3,4 bash tools/variant_sweep.sh > gpurun_out/sweep.log 2>&1
RR_LIB_VARIANT=build/variants/unit.so timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_unit.log 2>&1; echo "pytest unit exit $?"; tail -3 gpurun_out/pytest_unit.log
