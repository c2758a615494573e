bash tools/gpu_tests.sh
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 2>&1 | tail -1
