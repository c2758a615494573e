python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for v in b12 b10 b8; do echo "== $v"; RR_LIB_VARIANT=build/variants/$v.so python tools/timing.py 3,4 2>&1 | grep "config\|per launch"; done
