bash tools/gpu_tests.sh
timeout 900 python tools/quality_variants.py gpurun_out/quality_variants.json > gpurun_out/quality_variants.log 2>&1; tail -4 gpurun_out/quality_variants.log
