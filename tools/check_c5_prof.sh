mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "full_size or config5" > gpurun_out/pytest_c5.log 2>&1; echo "pytest exit $?"; tail -4 gpurun_out/pytest_c5.log
python tools/profile_run.py 4 512 0x60 8 > gpurun_out/plain.log 2>&1 || { cat gpurun_out/plain.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_residual_bidir -c 1 \
  -o gpurun_out/prof_r1_t6_full -f python tools/profile_run.py 4 512 0x60 8 > gpurun_out/ncu_full.log 2>&1; echo "ncu exit $?"
