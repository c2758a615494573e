python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -k "reconnect_bidir or records_config1 or records_full_size_configs or t6_toward or occluder" > gpurun_out/pt.log 2>&1; echo "pytest $?"; tail -5 gpurun_out/pt.log; grep -E "^E .*Assert" gpurun_out/pt.log | cut -c1-600 | head -8
python tools/timing.py 4 2>&1 | grep "config\|per launch"
