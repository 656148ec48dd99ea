timeout 1200 python tools/f64s_trace.py 1048576 0 100 c4 > gpurun_out/f64s_trace_c4_g0.log 2>&1
grep -E "sweep (1|2|3|4|5|6|8|10|16|20|30|40|60|80|100):" gpurun_out/f64s_trace_c4_g0.log
