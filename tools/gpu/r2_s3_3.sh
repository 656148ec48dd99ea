# session 3: L2 chunk sweep of the tcgen05 kernel; ncu --set full of the round-2 kernels at the C4 law (sparse sweep, probe, sparse K4)
timeout 600 python tools/sweep_paths.py 1048576 5 "C2 K=16 prec=2" > gpurun_out/s3_sweep_l2.log 2>&1; cat gpurun_out/s3_sweep_l2.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:softmin_f64s_kernel --launch-skip 40 --launch-count 1 -o gpurun_out/r2_ncu_f64s_c4_sparse python tools/f64s_trace.py 1048576 1 24 c4 > gpurun_out/s3_ncu_a.log 2>&1; echo "ncu a rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:f64s_probe_kernel --launch-skip 0 --launch-count 1 -o gpurun_out/r2_ncu_f64s_c4_probe python tools/f64s_trace.py 1048576 0 2 c4 > gpurun_out/s3_ncu_b.log 2>&1; echo "ncu b rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:plan_reduce --launch-skip 0 --launch-count 1 -o gpurun_out/r2_ncu_k4_c4 python tools/solve_bench.py c4 1048576 1 > gpurun_out/s3_ncu_c.log 2>&1; echo "ncu c rc=$?"
for f in r2_ncu_f64s_c4_sparse r2_ncu_f64s_c4_probe r2_ncu_k4_c4; do python tools/ncu_summary.py gpurun_out/$f.ncu-rep > gpurun_out/$f.txt 2>&1; done
tail -n 25 gpurun_out/r2_ncu_f64s_c4_sparse.txt
