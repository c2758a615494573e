mkdir -p gpurun_out
export RR_LIB_VARIANT=build/variants/s28b48.so
python tools/profile_run.py 3 512 0x40 8 > gpurun_out/plain.log 2>&1 || { cat gpurun_out/plain.log; exit 1; }
cat gpurun_out/plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_residual_single -c 1 \
    -o gpurun_out/prof_c3t7_s28 -f python tools/profile_run.py 3 512 0x40 8 > gpurun_out/ncu.log 2>&1; echo "ncu exit $?"
