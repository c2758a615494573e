bash tools/gpu_tests.sh
timeout 1500 python tools/quality_r2.py gpurun_out/quality_r2.json > gpurun_out/quality_r2.log 2>&1; echo "quality exit $?"; tail -30 gpurun_out/quality_r2.log
