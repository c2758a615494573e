mkdir -p gpurun_out
for v in build/variants/lb*.so; do
for m in -8 -16 -32; do
  RR_LIB_VARIANT=$v RR_TRACE_MODE=$m python tools/trace_bench.py 3 | sed "s|^|$v mode $m: |"
  RR_LIB_VARIANT=$v RR_TRACE_MODE=$m python tools/trace_bench.py 4 | sed "s|^|$v mode $m: |"
done
done
RR_LIB_VARIANT=build/variants/lb8.so RR_TRACE_MODE=-16 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_trace -c 1 \
    -o gpurun_out/prof_trace_lb8 -f python tools/trace_bench.py 3 1048576 > gpurun_out/ncu.log 2>&1; echo "ncu exit $?"
