# session 3: final ncu evidence of the F64S kernels: sparse sweeps at C4 / C5, sparse K4 at C4, kernel shares of 2 outer steps
timeout 900 ncu --set full --import-source on --clock-control none -k regex:softmin_f64s_kernel --launch-skip 30 --launch-count 1 -o /tmp/f64s_c4 python tools/f64s_trace.py 1048576 3 20 c4 > gpurun_out/s3_31_a.log 2>&1; echo "a rc=$?"
python tools/ncu_summary.py /tmp/f64s_c4.ncu-rep > gpurun_out/r2_ncu_f64s_c4_sparse.txt 2>&1; python tools/ncu_hot.py /tmp/f64s_c4.ncu-rep 12 >> gpurun_out/r2_ncu_f64s_c4_sparse.txt 2>/dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:softmin_f64s_kernel --launch-skip 30 --launch-count 1 -o /tmp/f64s_c5 python tools/f64s_trace.py 262144 3 20 c5 > gpurun_out/s3_31_b.log 2>&1; echo "b rc=$?"
python tools/ncu_summary.py /tmp/f64s_c5.ncu-rep > gpurun_out/r2_ncu_f64s_c5_sparse.txt 2>&1; python tools/ncu_hot.py /tmp/f64s_c5.ncu-rep 12 >> gpurun_out/r2_ncu_f64s_c5_sparse.txt 2>/dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:plan_reduce --launch-skip 1 --launch-count 1 -o /tmp/k4_c4 python tools/solve_bench.py c4 1048576 2 > gpurun_out/s3_31_c.log 2>&1; echo "c rc=$?"
python tools/ncu_summary.py /tmp/k4_c4.ncu-rep > gpurun_out/r2_ncu_k4_sparse_c4.txt 2>&1; python tools/ncu_hot.py /tmp/k4_c4.ncu-rep 12 >> gpurun_out/r2_ncu_k4_sparse_c4.txt 2>/dev/null
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file /tmp/c4_2steps.csv python tools/solve_bench.py c4 1048576 2 > gpurun_out/s3_31_d.log 2>&1; echo "d rc=$?"
python tools/launch_shares.py /tmp/c4_2steps.csv 30 > gpurun_out/r2_c4_2step_launch_shares.txt 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file /tmp/c5_2steps.csv python tools/solve_bench.py c5 262144 2 > gpurun_out/s3_31_e.log 2>&1; echo "e rc=$?"
python tools/launch_shares.py /tmp/c5_2steps.csv 30 > gpurun_out/r2_c5_2step_launch_shares.txt 2>&1
head -20 gpurun_out/r2_ncu_f64s_c4_sparse.txt gpurun_out/r2_ncu_f64s_c5_sparse.txt gpurun_out/r2_ncu_k4_sparse_c4.txt; head -16 gpurun_out/r2_c4_2step_launch_shares.txt gpurun_out/r2_c5_2step_launch_shares.txt
