python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
python tools/timing.py 4 2>&1 | grep "config\|per launch"
for v in ncg tcg ntcg nlu; do echo "== $v"; RR_LIB_VARIANT=build/variants/$v.so python tools/timing.py 4 2>&1 | grep "config\|per launch"; done
