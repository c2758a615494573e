#!/bin/bash
# Round-end measurement on one B200: bench line, ncu launch list of the same command, one ncu --set full
# capture of the dominant kernel (T6 side N launch at the bench config).  Outputs in gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"; cat gpurun_out/bench.json
if [ "${NCU:-1}" = "1" ]; then
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
echo "ncu launch list exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_residual_bidir -c 1 \
  -o gpurun_out/prof_full_t6 -f python tools/profile_run.py 4 512 0x60 8 > gpurun_out/ncu_full.log 2>&1
echo "ncu full exit $?"
fi
