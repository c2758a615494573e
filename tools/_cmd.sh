python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -k "reconnect_bidir or invalid" > gpurun_out/pt.log 2>&1; echo "pytest $?"; tail -5 gpurun_out/pt.log; grep -E "^E .*Assert" gpurun_out/pt.log | cut -c1-900 | head -8
