python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python tools/f64s_trace.py 262144 0 70 > gpurun_out/f64s_trace0.log 2>&1
timeout 1500 python tools/solve_bench.py c5 262144 2 > gpurun_out/c5_2step_d.log 2>&1
grep -E "sweep (1|2|3|4|5|7|8|9|15|16|17|31|32|33|63|64|65|70):" gpurun_out/f64s_trace0.log; tail -n 3 gpurun_out/c5_2step_d.log
