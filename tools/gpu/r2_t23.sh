python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python tools/f64s_trace.py 1048576 2 12 c4 > gpurun_out/f64s_trace_c4e.log 2>&1
timeout 1500 python tools/solve_bench.py c4 1048576 10 > gpurun_out/c4_part2.log 2>&1
timeout 1500 python tools/solve_bench.py c5 262144 10 > gpurun_out/c5_part2.log 2>&1
cat gpurun_out/f64s_trace_c4e.log gpurun_out/c4_part2.log gpurun_out/c5_part2.log
