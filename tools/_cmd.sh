bash tools/gpu_tests.sh
python tools/timing.py 3,4 2>&1 | grep -v "^\s*$"
