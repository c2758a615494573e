mkdir -p gpurun_out
python tools/profile_run.py 4 512 0x60 8 > gpurun_out/plain.log 2>&1 || { cat gpurun_out/plain.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_residual_bidir -c 1 \
  -o gpurun_out/prof_t6_inl -f python tools/profile_run.py 4 512 0x60 8 > gpurun_out/ncu_t6.log 2>&1; echo "ncu exit $?"
