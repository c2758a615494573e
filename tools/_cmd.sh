python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
python tools/dump_gpu_records.py > gpurun_out/dump.log 2>&1; tail -3 gpurun_out/dump.log
python tools/timing.py 4 2>&1 | grep -v "^\s*$"
python tools/timing.py 4 2>&1 | grep -v "^\s*$"
