python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
python tools/wave_probe.py 4 > gpurun_out/probe.log 2>&1; python tools/wave_probe.py 3 >> gpurun_out/probe.log 2>&1; cat gpurun_out/probe.log
python tools/timing.py 3,4 2>&1 | grep -v "^\s*$"
