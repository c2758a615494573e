python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -k "stats_accounting or records_config1_full" > gpurun_out/pt.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/pt.log
python tools/timing.py 4 2>&1 | grep "config\|per launch"
python tools/zero_samples.py 4 2>&1 | tail -14
