timeout 1200 python tools/f64s_trace.py 1048576 2 70 c4 > gpurun_out/f64s_trace_c4.log 2>&1
grep -E "sweep (1|2|3|4|5|7|8|9|15|16|17|31|32|33|63|64|65|70):" gpurun_out/f64s_trace_c4.log; tail -3 gpurun_out/f64s_trace_c4.log
