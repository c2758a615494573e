python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -k "records or stats or checkpoint or albedo or identity" > gpurun_out/pt.log 2>&1; echo "pytest $?"; tail -4 gpurun_out/pt.log; grep -E "^E .*Assert" gpurun_out/pt.log | cut -c1-600 | head -8
