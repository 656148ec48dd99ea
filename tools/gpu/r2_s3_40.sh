# session 3: ncu --set full of the steady-state (Gamma != 0) F64S sparse sweep at C4 and C5 (summary only)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:softmin_f64s_kernel --launch-skip 330 --launch-count 1 -o /tmp/f64s_c4s python tools/f64s_trace.py 1048576 3 30 c4 > gpurun_out/s3_40_a.log 2>&1; echo "a rc=$?"
python tools/ncu_summary.py /tmp/f64s_c4s.ncu-rep > gpurun_out/r2_ncu_f64s_c4_steady.txt 2>&1; python tools/ncu_hot.py /tmp/f64s_c4s.ncu-rep 12 >> gpurun_out/r2_ncu_f64s_c4_steady.txt 2>/dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:softmin_f64s_kernel --launch-skip 330 --launch-count 1 -o /tmp/f64s_c5s python tools/f64s_trace.py 262144 3 30 c5 > gpurun_out/s3_40_b.log 2>&1; echo "b rc=$?"
python tools/ncu_summary.py /tmp/f64s_c5s.ncu-rep > gpurun_out/r2_ncu_f64s_c5_steady.txt 2>&1; python tools/ncu_hot.py /tmp/f64s_c5s.ncu-rep 12 >> gpurun_out/r2_ncu_f64s_c5_steady.txt 2>/dev/null
head -19 gpurun_out/r2_ncu_f64s_c4_steady.txt gpurun_out/r2_ncu_f64s_c5_steady.txt
