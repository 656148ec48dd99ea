python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CNTGW_ORDER=cluster timeout 1500 python tools/solve_bench.py c4 1048576 10 > gpurun_out/c4_cluster.log 2>&1
CNTGW_ORDER=cluster timeout 1200 python tools/f64s_trace.py 1048576 0 20 c4 > gpurun_out/f64s_trace_c4_cl0.log 2>&1
timeout 1200 python tools/f64s_trace.py 1048576 0 20 c4 > gpurun_out/f64s_trace_c4_mo0.log 2>&1
cat gpurun_out/c4_cluster.log; grep -E "sweep (1|2|3|8|9|20):" gpurun_out/f64s_trace_c4_cl0.log gpurun_out/f64s_trace_c4_mo0.log
